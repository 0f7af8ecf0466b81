"""GPU parity of the filter + GCV path (regularize.hpp:42-81,
regularize.cpp:73-247, pipeline.cpp:120-155) against the numpy restatement:
restorations within 1e-10 relative, identical GCV grid index best_k, refined
mu within 1e-10 relative (north_star parity contract)."""
import numpy as np
import pytest
import torch

import fdoracle as O
import paper_0906_2704_b200 as P
from paper_0906_2704_b200 import workloads as W
from util import gauss, np_, onesided, rel

pytestmark = pytest.mark.gpu

SM = {0: O.IDENTITY, 1: O.LAPLACIAN, 2: O.FIRST_DIFFERENCE}


def setup(bc, psf, n, smoother):
    op = P.build_operator(psf, n, bc)
    L = P.smoothing_eigenvalues(smoother, op)
    oop = O.build_operator(O.make_psf(psf, normalize=True), n, bc)
    s = O.smoothing_eigenvalues(SM[smoother], bc, n, oop.eigenvalues)
    return op, L, oop, s


CASES = [(O.HOC_COSINE, gauss(10, 3.0)), (O.HOC_FOURIER, onesided(15, 0.2)),
         (O.ANTIREFLECTIVE, gauss(4, 1.5)), (O.REFLECTIVE, gauss(3, 1.5)),
         (O.PERIODIC, onesided(5, 0.5))]


@pytest.mark.parametrize("bc,psf", CASES)
@pytest.mark.parametrize("smoother", [0, 1, 2])
def test_smoother_tikhonov_gcv_value(bc, psf, smoother, rng):
    n = 256
    op, L, oop, s = setup(bc, psf, n, smoother)
    assert np.max(np.abs(np_(L.eigenvalues()) - s)) < 1e-14
    g = np.cumsum(rng.standard_normal((3, n)), axis=-1) / 10
    mu = np.array([1e-6, 1e-3, 0.5])
    f, res = P.tikhonov_solve(op, L, torch.from_numpy(g), torch.from_numpy(mu))
    for b in range(3):
        want, _ = O.tikhonov_solve(oop, s, g[b], mu[b])
        assert rel(np_(f[b]), want) < 1e-10
    for m in (1e-7, 1e-2):
        G = np_(P.gcv_value(op, L, torch.from_numpy(g), m))
        want = O.gcv_value(oop, s, g, m)
        assert np.max(np.abs(G / want - 1)) < 1e-11


@pytest.mark.parametrize("bc,psf", CASES)
@pytest.mark.parametrize("smoother", [0, 1])
@pytest.mark.parametrize("search", [(1e-8, 1.0, 64), (1e-12, 10.0, 200), (1e-6, 1.0, 7)])
def test_gcv_select_and_deblur(bc, psf, smoother, search, rng):
    n = 512
    op, L, oop, s = setup(bc, psf, n, smoother)
    cfg = W.config(0)
    # config-0 style scenes on the extended grid, blurred with this case's psf
    truth, _ = W.signals_1d(cfg, 0, 5, n=n + len(psf) - 1, m=0)
    g = W.add_noise(W.convolve_valid(truth, np.asarray(psf) / np.sum(psf)), 0.01,
                    W.item_key(99, np.arange(5, dtype=np.uint64)))
    mu_min, mu_max, K = search
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True), want_curve=True,
                   search=P.GcvSearch(mu_min, mu_max, K))
    want = O.deblur(oop, s, g, True, mu_min=mu_min, mu_max=mu_max, count=K, want_curve=True)
    assert np.array_equal(np_(rep.best_k), want.best_k)
    assert np.max(np.abs(np_(rep.gcv_curve) / want.curves - 1)) < 1e-11
    assert np.max(np.abs(np_(rep.mu_used) / want.mu_used - 1)) < 1e-10
    assert rel(np_(rep.restored), want.restored) < 1e-10
    sel = P.gcv_select(op, L, torch.from_numpy(g), P.GcvSearch(mu_min, mu_max, K))
    assert np.array_equal(np_(sel.mu), np_(rep.mu_used))


def test_gcv_constant_functional_tie_break(rng):
    """test_regularize.cpp:201-222: identity psf + identity smoother gives a
    constant G = ||ghat||^2/n^2 and the geometric midpoint of the grid."""
    n = 16
    op = P.build_operator([1.0], n, "reflective")
    L = P.smoothing_eigenvalues("identity", op)
    g = rng.uniform(-1, 1, n)
    ghat = O.cosine_apply(g)
    want = np.sum(ghat ** 2) / (n * n)
    for mu in (1e-10, 1e-4, 1.0, 9.9):
        assert abs(float(np_(P.gcv_value(op, L, torch.from_numpy(g), mu))) / want - 1) < 1e-12
    sel = P.gcv_select(op, L, torch.from_numpy(g), P.GcvSearch(1e-12, 10.0, 200))
    assert abs(float(np_(sel.mu)) / np.sqrt(1e-12 * 10.0) - 1) < 1e-9


def test_identity_tikhonov_is_g_over_one_plus_mu(rng):
    """test_regularize.cpp:41-50."""
    op = P.build_operator([1.0], 32, "reflective")
    L = P.smoothing_eigenvalues("identity", op)
    g = rng.uniform(-1, 1, 32)
    for mu in (1e-3, 0.5, 2.0):
        f, _ = P.tikhonov_solve(op, L, torch.from_numpy(g), mu)
        assert np.allclose(np_(f), g / (1 + mu), rtol=1e-12, atol=0)


def test_degenerate_gcv_raises(rng):
    """test_regularize.cpp:277-284: all smoother eigenvalues zero -> DegenerateError."""
    op = P.build_operator([1.0], 16, "reflective")
    L = P.smoother_from_eigenvalues(op, np.zeros(16))
    with pytest.raises(P.DegenerateError):
        P.gcv_value(op, L, torch.from_numpy(rng.uniform(-1, 1, 16)), 1e-3)


def test_parameter_errors(rng):
    """test_regularize.cpp:296-304."""
    op = P.build_operator([1.0], 16, "reflective")
    L = P.smoothing_eigenvalues("identity", op)
    g = torch.from_numpy(rng.uniform(-1, 1, 16))
    with pytest.raises(P.ValidationError):
        P.tikhonov_solve(op, L, g, 0.0)
    with pytest.raises(P.ValidationError):
        P.tikhonov_solve(op, L, g, -1.0)
    with pytest.raises(P.ValidationError):
        P.gcv_select(op, L, g, P.GcvSearch(0.0, 1.0, 10))
    with pytest.raises(P.ValidationError):
        P.gcv_select(op, L, g, P.GcvSearch(1e-3, 1e-6, 10))


def test_gcv_argmin_scale_invariance(rng):
    """test_regularize.cpp:224-244: power-of-two scaling keeps the argmin and
    scales G by c^2."""
    op = P.build_operator(gauss(4, 2.0), 64, "hoc-cosine")
    L = P.smoothing_eigenvalues("laplacian", op)
    g = rng.uniform(-1, 1, 64)
    r1 = P.gcv_select(op, L, torch.from_numpy(g), P.GcvSearch(1e-10, 1.0, 60))
    r4 = P.gcv_select(op, L, torch.from_numpy(4 * g), P.GcvSearch(1e-10, 1.0, 60))
    assert int(np_(r1.best_k)) == int(np_(r4.best_k))
    assert np.allclose(np_(r4.curve), 16 * np_(r1.curve), rtol=1e-12, atol=0)


@pytest.mark.parametrize("bc,psf,smoother,search", [
    (O.HOC_FOURIER, onesided(15, 0.2), 2, (1e-8, 1.0, 256)),
    (O.HOC_COSINE, gauss(10, 3.0), 0, (1e-6, 1.0, 64)),
    (O.HOC_COSINE, gauss(6, 2.0), 1, (1e-6, 1.0, 128)),
    (O.PERIODIC, onesided(5, 0.5), 1, (1e-10, 1.0, 300))])
def test_batched_gemm_gcv_path(bc, psf, smoother, search):
    """Batches of >= 32 signals take the GEMM-form GCV grid (k_gcv_gemm)."""
    n, B = 1024, 97
    op, L, oop, s = setup(bc, psf, n, smoother)
    cfg = W.config(1)
    truth, _ = W.signals_1d(cfg, 100, B, n=n + len(psf) - 1, m=0)
    g = W.add_noise(W.convolve_valid(truth, np.asarray(psf) / np.sum(psf)), 0.005,
                    W.item_key(98, np.arange(B, dtype=np.uint64)))
    mu_min, mu_max, K = search
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True), want_curve=True,
                   search=P.GcvSearch(mu_min, mu_max, K))
    want = O.deblur(oop, s, g, True, mu_min=mu_min, mu_max=mu_max, count=K, want_curve=True)
    assert np.array_equal(np_(rep.best_k), want.best_k)
    assert np.max(np.abs(np_(rep.gcv_curve) / want.curves - 1)) < 1e-11
    assert np.max(np.abs(np_(rep.mu_used) / want.mu_used - 1)) < 1e-10
    assert rel(np_(rep.restored), want.restored) < 1e-10


@pytest.mark.parametrize("bc", [O.HOC_FOURIER, O.PERIODIC])
def test_hermitian_packed_synthesis(bc, rng):
    """Real outputs of complex bases: two Hermitian-projected lines per FFT give
    Re(T c) of the exact one-line path."""
    n = 4096
    psf = onesided(15, 0.2)
    op, L, oop, s = setup(bc, psf, n, 1)
    g = np.cumsum(rng.standard_normal((5, n)), axis=-1) / 30
    mu = np.array([1e-6, 1e-4, 1e-3, 1e-2, 1.0])
    f_fast, r_fast = P.tikhonov_solve(op, L, torch.from_numpy(g), torch.from_numpy(mu))
    f_exact, r_exact = P.tikhonov_solve(op, L, torch.from_numpy(g), torch.from_numpy(mu),
                                        want_imag_residue=True)
    assert r_fast is None and np.all(np_(r_exact) < 1e-9)
    assert rel(np_(f_fast), np_(f_exact)) < 1e-13
    for b in range(5):
        assert rel(np_(f_fast[b]), O.tikhonov_solve(oop, s, g[b], mu[b])[0]) < 1e-10


@pytest.mark.parametrize("chunk", [0, 7, 1000])
def test_deblur_host_pipeline_matches_device(chunk):
    """fd_deblur_host (chunked H2D | deblur | D2H on three streams) equals the
    device-resident deblur item by item."""
    n, B = 512, 50
    op = P.build_operator(onesided(15, 0.2), n, "hoc-fourier")
    L = P.smoothing_eigenvalues("first-difference", op)
    _, g = W.signals_1d(W.config(1), 0, B, n=n, m=14)
    gh = torch.from_numpy(g).pin_memory()
    search = P.GcvSearch(1e-8, 1.0, 256)
    rest, mu, bk = P.deblur_host(op, L, gh, P.MuChoice(True), search=search, chunk=chunk)
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True), search=search)
    # small chunks take the non-GEMM GCV kernels: equal to rounding
    assert np.array_equal(bk.numpy(), np_(rep.best_k))
    assert np.max(np.abs(mu.numpy() / np_(rep.mu_used) - 1)) < 1e-12
    assert rel(rest.numpy(), np_(rep.restored)) < 1e-12


@pytest.mark.parametrize("bc,psf,smoother,search", [
    (O.HOC_FOURIER, onesided(15, 0.2), 2, (1e-8, 1.0, 256)),
    (O.HOC_COSINE, gauss(10, 3.0), 1, (1e-6, 1.0, 100)),
    (O.PERIODIC, onesided(5, 0.5), 1, (1e-10, 1.0, 64)),
    (O.REFLECTIVE, gauss(6, 2.0), 0, (1e-8, 10.0, 256))])
def test_tensor_core_gcv_screen(bc, psf, smoother, search, monkeypatch):
    """Batches without a requested curve take the tcgen05 TF32 screen + exact
    fp64 candidates (fd_tc.cuh): identical best_k and mu to the all-fp64 grid
    and to the oracle; an all-zero item falls back to the exact grid."""
    n, B = 1024, 300
    op, L, oop, s = setup(bc, psf, n, smoother)
    truth, _ = W.signals_1d(W.config(1), 500, B, n=n + len(psf) - 1, m=0)
    g = W.add_noise(W.convolve_valid(truth, np.asarray(psf) / np.sum(psf)), 0.005,
                    W.item_key(97, np.arange(B, dtype=np.uint64)))
    g[17] = 0.0
    mu_min, mu_max, K = search
    sr = P.GcvSearch(mu_min, mu_max, K)
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True), search=sr)
    monkeypatch.setenv("FASTDEBLUR_GCV_SCREEN", "0")
    ref = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True), search=sr)
    assert np.array_equal(np_(rep.best_k), np_(ref.best_k))
    assert np.max(np.abs(np_(rep.mu_used) / np_(ref.mu_used) - 1)) < 1e-12
    assert rel(np_(rep.restored), np_(ref.restored)) < 1e-12
    sel = [i for i in range(B) if i % 10 == 3] + [17]
    want = O.deblur(oop, s, g[sel], True, mu_min=mu_min, mu_max=mu_max, count=K)
    assert np.array_equal(np_(rep.best_k)[sel], want.best_k)
    assert np.max(np.abs(np_(rep.mu_used)[sel] / want.mu_used - 1)) < 1e-10


@pytest.mark.parametrize("bc,psf,smoother", [(O.HOC_COSINE, gauss(10, 3.0), 0),
                                             (O.HOC_FOURIER, onesided(15, 0.2), 2),
                                             (O.ANTIREFLECTIVE, gauss(4, 1.5), 1)])
def test_sweep_mu_matches_oracle(bc, psf, smoother):
    """sweep_mu (pipeline.cpp:55-115): G curve, RRE at every grid mu (one
    analysis, batched filtered syntheses), mu_opt, mu_gcv, rre_gcv."""
    n = 1024
    op, L, oop, s = setup(bc, psf, n, smoother)
    truth, _ = W.signals_1d(W.config(1), 11, 1, n=n + len(psf) - 1, m=0)
    m = len(psf) // 2
    g = W.add_noise(W.convolve_valid(truth, np.asarray(psf) / np.sum(psf)), 0.01, 5)[0]
    t = truth[0, m:m + n]
    sr = P.GcvSearch(1e-6, 1.0, 40)
    sw = P.sweep_mu(op, L, torch.from_numpy(g), torch.from_numpy(t), search=sr)
    mus, G, rr, summ = O.sweep_mu(oop, s, g, t, 1e-6, 1.0, 40)
    assert np.array_equal([p.mu for p in sw.curve], mus)
    assert np.max(np.abs(np.array([p.gcv for p in sw.curve]) / G - 1)) < 1e-11
    assert np.max(np.abs(np.array([p.rre for p in sw.curve]) / rr - 1)) < 1e-10
    assert sw.mu_opt == summ[1]
    assert abs(sw.min_rre / summ[0] - 1) < 1e-10
    assert abs(sw.mu_gcv / summ[2] - 1) < 1e-10
    assert abs(sw.rre_gcv / summ[3] - 1) < 1e-10
    nt = P.sweep_mu(op, L, torch.from_numpy(g), search=sr)
    assert np.isnan(nt.min_rre) and np.isnan(nt.curve[0].rre) and nt.mu_gcv == sw.mu_gcv
    with pytest.raises(P.ValidationError):
        P.sweep_mu(op, L, torch.from_numpy(g), torch.zeros(n, dtype=torch.float64), search=sr)


def test_sweep_mu_2d_consistent():
    """sweep_mu_2d: the RRE of every grid mu equals that of tikhonov_solve_2d."""
    n1, n2 = 96, 128
    psf = gauss(4, 1.5)
    op = P.build_operator_2d_separable(psf, psf, n1, n2, "hoc-cosine")
    L = P.smoothing_eigenvalues("laplacian", op)
    truth, g = W.image_2d(W.config(2), 1, n1, n2)
    sr = P.GcvSearch(1e-6, 1.0, 12)
    sw = P.sweep_mu(op, L, torch.from_numpy(g), torch.from_numpy(truth), search=sr)
    sel = P.gcv_select(op, L, torch.from_numpy(g), search=sr)
    for p in sw.curve:
        f, _ = P.tikhonov_solve(op, L, torch.from_numpy(g), p.mu)
        want = np.linalg.norm(truth - np_(f)) / np.linalg.norm(truth)
        assert abs(p.rre / want - 1) < 1e-12
    assert abs(sw.mu_gcv / float(np_(sel.mu)) - 1) < 1e-14
