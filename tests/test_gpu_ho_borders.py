"""GPU parity of the higher-order border extension (hoc-fourier-d1 / -d3,
BASELINE configs 1 and 3 at degree 1 and 3) through the C ABI against the
oracle's HoTransform (oracle/fdoracle.py, pinned in tests/test_ho_borders.py).

Tolerances.  The degree-1 transform is well conditioned (cond(T) ~ 50 at
n = 4096): coefficients and round trips at 1e-12.  The degree-3 transform is
intrinsically ill conditioned -- cond(T) grows like n^2.5 whatever basis spans
the border columns (1.4e6 at n = 1024) -- so coefficient-level
checks on white noise scale with it (1e-15 cond).  Restorations, GCV choices and
matvecs of smooth scenes keep the north_star bar: best_k identical, mu and the
restoration within 1e-10."""
import numpy as np
import pytest
import torch

import fdoracle as O
import paper_0906_2704_b200 as P
from paper_0906_2704_b200 import workloads as W
from util import np_, onesided, gauss, rel

pytestmark = pytest.mark.gpu

HO = [O.HOC_FOURIER_D1, O.HOC_FOURIER_D3]
SM = {0: O.IDENTITY, 1: O.LAPLACIAN, 2: O.FIRST_DIFFERENCE}


def coeff_tol(bc, n):
    if bc == O.HOC_FOURIER_D1:
        return 1e-12
    cond = {8: 10, 33: 3e2, 64: 1.5e3, 257: 5e4, 1024: 1.5e6, 4096: 5e7}.get(n, 5e7)
    return max(1e-12, 1e-15 * cond * 10)


@pytest.mark.parametrize("bc", HO)
@pytest.mark.parametrize("n", [8, 33, 64, 257, 1024, 4096])
def test_analyze_synthesize(bc, n, rng):
    op = P.build_operator([1.0], n, bc)
    b = O.SpectralBasis(bc, n)
    for B in (1, 3):  # odd batch: two real lines per FFT plus a lone line
        x = rng.standard_normal((B, n))
        got = np_(op.analyze(torch.from_numpy(x)))
        want = b.analyze(x.astype(complex))
        assert rel(got, want) < coeff_tol(bc, n), (n, B, rel(got, want))
        c = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
        assert rel(np_(op.synthesize(torch.from_numpy(c))), b.synthesize(c)) < coeff_tol(bc, n)
        back = np_(op.synthesize(op.analyze(torch.from_numpy(x)))).real
        assert rel(back, x) < coeff_tol(bc, n)
        # complex input lines (the 2D row pass)
        z = x + 1j * rng.standard_normal((B, n))
        assert rel(np_(op.analyze(torch.from_numpy(z))), b.analyze(z)) < coeff_tol(bc, n)


@pytest.mark.parametrize("bc", HO)
@pytest.mark.parametrize("n", [33, 512, 4096])
def test_eigenvalues_matvec_polynomials(bc, n, rng):
    psf = onesided(15, 0.2)
    op = P.build_operator(psf, n, bc)
    oop = O.build_operator(O.make_psf(psf, normalize=True), n, bc)
    assert np.max(np.abs(np_(op.eigenvalues()) - oop.eigenvalues)) < 1e-14
    f = np.cumsum(rng.standard_normal((2, n)), axis=-1) / np.sqrt(n)
    got, res = P.blur_apply(op, torch.from_numpy(f))
    want, wres = oop.apply(f)
    assert rel(np_(got), want) < 1e-11
    assert np.all(np_(res) < 1e-9)
    # polynomials of degree <= d are eigenvectors with eigenvalue 1
    d = O.HO_BORDERS[bc][2]
    x = np.linspace(-1.0, 1.0, n)
    polys = np.stack([(x - 0.2) ** p for p in range(d + 1)])
    got, _ = P.blur_apply(op, torch.from_numpy(polys))
    assert np.max(np.abs(np_(got) - polys)) < (1e-12 if d == 1 else 1e-8)


def scenes(n, psf, B, seed):
    cfg = W.config(1)
    truth, _ = W.signals_1d(cfg, seed, B, n=n + len(psf) - 1, m=0)
    return W.add_noise(W.convolve_valid(truth, np.asarray(psf) / np.sum(psf)), 0.005,
                       W.item_key(seed, np.arange(B, dtype=np.uint64)))


@pytest.mark.parametrize("bc", HO)
@pytest.mark.parametrize("smoother", [0, 1, 2])
@pytest.mark.parametrize("n,B,search", [(512, 5, (1e-8, 1.0, 64)), (4096, 3, (1e-8, 1.0, 256)),
                                        (1024, 40, (1e-8, 1.0, 256))])
def test_deblur_matches_oracle(bc, smoother, n, B, search):
    psf = onesided(15, 0.2)
    op = P.build_operator(psf, n, bc)
    L = P.smoothing_eigenvalues(smoother, op)
    oop = O.build_operator(O.make_psf(psf, normalize=True), n, bc)
    s = O.smoothing_eigenvalues(SM[smoother], bc, n, oop.eigenvalues)
    assert np.max(np.abs(np_(L.eigenvalues()) - s)) < 1e-14
    g = scenes(n, psf, B, 41 + n)
    mu_min, mu_max, K = search
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True), want_curve=True,
                   search=P.GcvSearch(mu_min, mu_max, K))
    want = O.deblur(oop, s, g, True, mu_min=mu_min, mu_max=mu_max, count=K, want_curve=True)
    assert np.array_equal(np_(rep.best_k), want.best_k)
    assert np.max(np.abs(np_(rep.gcv_curve) / want.curves - 1)) < 1e-10
    assert np.max(np.abs(np_(rep.mu_used) / want.mu_used - 1)) < 1e-10
    assert rel(np_(rep.restored), want.restored) < 1e-10
    # the curve-free path (screens / moments) picks the same mu
    rep2 = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True),
                    search=P.GcvSearch(mu_min, mu_max, K))
    assert np.array_equal(np_(rep2.best_k), want.best_k)
    assert np.max(np.abs(np_(rep2.mu_used) / want.mu_used - 1)) < 1e-10
    assert rel(np_(rep2.restored), want.restored) < 1e-10


@pytest.mark.parametrize("bc", HO)
@pytest.mark.parametrize("separable", [True, False])
def test_2d(bc, separable, rng):
    n1, n2 = 96, 80
    a = onesided(6, 0.25)
    p2 = O.separable_psf2d(O.make_psf(a, True), O.make_psf(a, True))
    if separable:
        op = P.build_operator_2d_separable(a, a, n1, n2, bc)
    else:
        op = P.build_operator_2d(p2.weights, n1, n2, bc)
    oop = O.build_operator_2d(p2, n1, n2, bc, separable=separable)
    assert np.max(np.abs(np_(op.eigenvalues()) - oop.eigenvalues)) < 1e-13
    f = np.cumsum(np.cumsum(rng.standard_normal((2, n1, n2)), -1), -2) / n1
    got, _ = P.blur_apply(op, torch.from_numpy(f))
    assert rel(np_(got), oop.apply(f)[0]) < 1e-11
    for smoother in (0, 1):
        L = P.smoothing_eigenvalues(smoother, op)
        s = O.smoothing_eigenvalues_2d(SM[smoother], bc, n1, n2, oop.eigenvalues)
        g = got.cpu().numpy() + 0.01 * rng.standard_normal((2, n1, n2))
        rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True),
                       search=P.GcvSearch(1e-6, 1.0, 128))
        want = O.deblur_2d(oop, s, g, True, mu_min=1e-6, mu_max=1.0, count=128)
        assert np.array_equal(np_(rep.best_k), want.best_k)
        assert np.max(np.abs(np_(rep.mu_used) / want.mu_used - 1)) < 1e-10
        assert rel(np_(rep.restored), want.restored) < 1e-10


@pytest.mark.parametrize("bc,n", [(O.HOC_FOURIER_D1, 64), (O.HOC_FOURIER_D1, 1366),
                                  (O.HOC_FOURIER_D1, 4096), (O.HOC_FOURIER_D3, 64),
                                  (O.HOC_FOURIER_D3, 2314)])
@pytest.mark.parametrize("smoother", [0, 2])
def test_mixed_radix_pair_path(bc, n, smoother):
    """d = 1 interiors m = 63, 1365, 4095 factor into 3..13: the pair kernels
    run the direct mixed-radix DFT (fd_mixed.cuh); d = 3 interiors m = 61 and
    2311 are primes with m - 1 = 4*3*5, 2*3*5*7*11: Rader (fd_rader.cuh)."""
    psf = onesided(15, 0.2)
    op = P.build_operator(psf, n, bc)
    L = P.smoothing_eigenvalues(smoother, op)
    oop = O.build_operator(O.make_psf(psf, normalize=True), n, bc)
    s = O.smoothing_eigenvalues(SM[smoother], bc, n, oop.eigenvalues)
    g = scenes(n, psf, 37, 7 + n)
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True), want_curve=True,
                   search=P.GcvSearch(1e-8, 1.0, 256))
    want = O.deblur(oop, s, g, True, mu_min=1e-8, mu_max=1.0, count=256, want_curve=True)
    assert np.array_equal(np_(rep.best_k), want.best_k)
    assert np.max(np.abs(np_(rep.gcv_curve) / want.curves - 1)) < 1e-10
    assert np.max(np.abs(np_(rep.mu_used) / want.mu_used - 1)) < 1e-10
    assert rel(np_(rep.restored), want.restored) < 1e-10


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_deblur_host_multi_matches_device(dtype):
    """fd_deblur_host_multi: one upload per chunk, every operator restores it."""
    n, B = 1024, 70
    psf = onesided(15, 0.2)
    g = torch.from_numpy(scenes(n, psf, B, 3)).to(dtype)
    ops = [P.build_operator(psf, n, bc) for bc in HO]
    Ls = [P.smoothing_eigenvalues(2, op) for op in ops]
    search = P.GcvSearch(1e-8, 1.0, 256)
    res = P.deblur_host_multi(ops, Ls, g, P.MuChoice(True), search=search, chunk=16)
    for op, L, (f, mu, bk) in zip(ops, Ls, res):
        rep = P.deblur(op, L, g.cuda(), P.MuChoice(True), search=search)
        assert f.dtype == dtype
        assert np.array_equal(bk.numpy(), np_(rep.best_k))
        assert np.array_equal(mu.numpy(), np_(rep.mu_used))
        assert np.array_equal(f.numpy(), np_(rep.restored))
