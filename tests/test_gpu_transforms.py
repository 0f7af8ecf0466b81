"""GPU parity: T_X^{-1} / T_X (analyze / synthesize) and matvec through the
C ABI vs the numpy restatement of boundary.cpp / trig.cpp (oracle/fdoracle.py).

Tolerances: synthesize is well conditioned (<= 1e-12 relative).  Analyze of
the corrected bases goes through the 2x2 SMW solve whose capacitance
condition grows like n for hoc-fourier; two exact-to-rounding
implementations (the compiled reference and the numpy restatement) already
differ by ~1e-11 at n = 4096 (tests/test_oracle_pins.py), so analyze is
checked at 1e-12 up to n = 128 and 1e-9 beyond, and the round trip
synthesize(analyze(y)) = y at 1e-10 everywhere."""
import numpy as np
import pytest
import torch

import fdoracle as O
import paper_0906_2704_b200 as P
from util import np_, rel, gauss, onesided

pytestmark = pytest.mark.gpu

SIZES = [5, 6, 7, 8, 33, 64, 101, 128, 1024, 2049, 4096]


def _max_n(bc):
    return 4098


@pytest.mark.parametrize("bc", range(5))
@pytest.mark.parametrize("n", SIZES)
def test_analyze_synthesize(bc, n, rng):
    if n > _max_n(bc):
        pytest.skip("antireflective DST-I length limit of this build")
    op = P.build_operator([1.0], n, bc)
    b = O.SpectralBasis(bc, n)
    for B in (1, 3):  # odd batch exercises the two-lines-per-FFT packing
        x = rng.standard_normal((B, n))
        got = np_(op.analyze(torch.from_numpy(x)))
        want = b.analyze(x.astype(complex) if b.complex else x)
        tol = 1e-12 if n <= 128 else 1e-9
        assert rel(got, want) < tol, (bc, n, B, rel(got, want))
        c = rng.standard_normal((B, n)) + (1j * rng.standard_normal((B, n)) if b.complex else 0)
        got_s = op.synthesize(torch.from_numpy(c))
        got_s = np_(got_s if b.complex else got_s[0])
        assert rel(got_s, b.synthesize(c)) < 1e-12, (bc, n, B)
        back = op.synthesize(op.analyze(torch.from_numpy(x)))
        back = np_(back).real if b.complex else np_(back[0])
        assert rel(back, x) < 1e-10


@pytest.mark.parametrize("bc", [O.PERIODIC, O.HOC_FOURIER])
@pytest.mark.parametrize("n", [6, 64, 1024, 4096])
def test_complex_input_analyze(bc, n, rng):
    op = P.build_operator([1.0], n, bc)
    b = O.SpectralBasis(bc, n)
    x = rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n))
    got = np_(op.analyze(torch.from_numpy(x)))
    assert rel(got, b.analyze(x)) < (1e-12 if n <= 128 else 1e-9)


def test_real_synthesis_reports_imag_residue(rng):
    n = 64
    op = P.build_operator([1.0], n, "hoc-fourier")
    b = O.SpectralBasis(O.HOC_FOURIER, n)
    c = rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n))
    out, res = op.synthesize(torch.from_numpy(c), complex_out=False)
    want = b.synthesize(c)
    assert rel(np_(out), want.real) < 1e-12
    assert np.allclose(np_(res), np.sqrt(np.sum(want.imag ** 2, axis=-1)), rtol=1e-12)


CASES = [(O.PERIODIC, onesided(5, 0.5)), (O.REFLECTIVE, gauss(3, 1.5)),
         (O.ANTIREFLECTIVE, gauss(4, 2.0)), (O.HOC_COSINE, gauss(10, 3.0)),
         (O.HOC_FOURIER, onesided(15, 0.2))]


@pytest.mark.parametrize("bc,psf", CASES)
@pytest.mark.parametrize("n", [33, 256, 1024])
def test_eigenvalues_and_matvec(bc, psf, n, rng):
    op = P.build_operator(psf, n, bc)
    oop = O.build_operator(O.make_psf(psf, normalize=True), n, bc)
    d = np_(op.eigenvalues())
    assert np.max(np.abs(d - oop.eigenvalues)) < 1e-14
    if O.is_boundary_corrected(bc):
        assert d[0] == 1.0 and d[-1] == 1.0
    f = rng.standard_normal((3, n))
    got, res = op.apply(torch.from_numpy(f))
    want, wres = oop.apply(f)
    assert rel(np_(got), want) < 1e-11
    assert np.all(np_(res) < 1e-10)


def motion_psf(m):
    """psf.cpp:71-76: h_j ∝ m+1-j for j = 0..m, zero for j < 0."""
    w = np.zeros(2 * m + 1)
    w[m:] = m + 1 - np.arange(m + 1)
    return w / w.sum()


@pytest.mark.parametrize("bc,psf,degs,tol", [
    (O.ANTIREFLECTIVE, gauss(6, 2.0), (0, 1), 1e-10),
    (O.HOC_COSINE, gauss(6, 2.0), (0, 1, 2), 1e-8),
    (O.HOC_FOURIER, motion_psf(4), (0, 1, 2), 1e-8)])
def test_polynomial_preservation(bc, psf, degs, tol):
    """test_operators.cpp:162-197: sampled polynomials (x + 0.3)^deg on the
    extended grid are fixed points (AR: deg <= 1, hoc: deg <= 2)."""
    n = 64
    op = P.build_operator(psf, n, bc)
    basis = {O.ANTIREFLECTIVE: O.B_AR, O.HOC_COSINE: O.B_HC, O.HOC_FOURIER: O.B_HF}[bc]
    pts = O.extended_grid(basis, n)[2]
    for deg in degs:
        f = (pts + 0.3) ** deg
        got, res = op.apply(torch.from_numpy(f))
        assert rel(np_(got), f) < tol
        assert float(np_(res)) <= 1e-10 * (1.0 + np.linalg.norm(f))


@pytest.mark.parametrize("bc", [O.HOC_COSINE, O.REFLECTIVE, O.HOC_FOURIER, O.PERIODIC])
@pytest.mark.parametrize("n", [8194, 16384])
def test_split_convolution_lines(bc, n, rng):
    """Lines whose half-length Bluestein size exceeds shared memory (config 4:
    interior DCT length 16382 = 2 * 8191) run as two half convolutions."""
    psf = gauss(16, 4.0) if bc in (O.HOC_COSINE, O.REFLECTIVE) else onesided(15, 0.2)
    op = P.build_operator(psf, n, bc)
    oop = O.build_operator(O.make_psf(psf, True), n, bc)
    b = oop.basis
    x = np.cumsum(rng.standard_normal((2, n)), axis=-1) / 50
    got = np_(op.analyze(torch.from_numpy(x)))
    want = b.analyze(x.astype(complex) if b.complex else x)
    assert rel(got, want) < 1e-9
    L = P.smoothing_eigenvalues("laplacian", op)
    s = O.smoothing_eigenvalues(O.LAPLACIAN, bc, n, oop.eigenvalues)
    for mu in (1e-6, 1e-2):
        f, _ = P.tikhonov_solve(op, L, torch.from_numpy(x), mu)
        assert rel(np_(f), O.tikhonov_solve(oop, s, x, mu)[0]) < 1e-10
    if not b.complex:
        c = rng.standard_normal((3, n))
        assert rel(np_(op.synthesize(torch.from_numpy(c))[0]), b.synthesize(c)) < 1e-12


def test_split_convolution_2d_columns(rng):
    """2D operator whose column lines (n1 = 16384) need the split convolution."""
    n1, n2 = 16384, 40
    a, bb = gauss(16, 4.0), gauss(2, 1.0)
    op = P.build_operator_2d_separable(a, bb, n1, n2, "hoc-cosine")
    p = O.separable_psf2d(O.make_psf(a, True), O.make_psf(bb, True))
    oop = O.build_operator_2d(p, n1, n2, O.HOC_COSINE, separable=True)
    # Smooth field: on white noise the bordered (SMW-corrected) transforms of the
    # oracle and of the compiled reference already disagree by ~5e-11 at
    # n = 16384 (conditioning of T_X), so the 1e-10 bar is stated on the
    # regime it is meant for, as in test_split_convolution_lines.
    f = np.cumsum(np.cumsum(rng.standard_normal((n1, n2)), axis=0), axis=1) / 100
    got, _ = op.apply(torch.from_numpy(f))
    assert rel(np_(got), oop.apply(f)[0]) < 1e-10
    L = P.smoothing_eigenvalues("laplacian", op)
    s = O.smoothing_eigenvalues_2d(O.LAPLACIAN, O.HOC_COSINE, n1, n2)
    rep = P.deblur(op, L, torch.from_numpy(f), P.MuChoice(True), search=P.GcvSearch(1e-8, 1, 64))
    w = O.deblur_2d(oop, s, f, True, mu_min=1e-8, mu_max=1.0, count=64)
    assert int(np_(rep.best_k)) == int(w.best_k)
    assert rel(np_(rep.restored), w.restored) < 1e-10
