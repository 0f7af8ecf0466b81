"""Pin the numpy restatement (oracle/fdoracle.py) before trusting it:
  * the known answers the reference's own tests hold (file:line cited);
  * golden vectors produced by the reference itself (tests/golden, made by
    oracle/gen_golden.py from oracle/_ref);
  * the live reference library when it is built here (oracle/_ref).
CPU only."""
import math

import numpy as np
import pytest

import fdoracle as O
import reflib as R
from util import gauss, onesided, rel
from paper_0906_2704_b200 import workloads as W

PI = math.pi
G1 = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                        "golden_1d.npz"))
G2 = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                        "golden_2d.npz"))


# ---------------------------------------------------------------- known answers
def test_hoc_cosine_n6_grid_and_column():
    """test_boundary.cpp:55-73: q~ = pi^2 (25/16, 1, 9/16, 1/4, 1/16, 0)."""
    a, b, pts = O.extended_grid(O.B_HC, 6)
    assert abs(a + PI / 8) < 1e-15 and abs(b - 9 * PI / 8) < 1e-15
    assert np.allclose(pts, (2 * np.arange(6) - 1) * PI / 8, rtol=1e-15, atol=0)
    qt = PI * PI * np.array([25 / 16, 1, 9 / 16, 1 / 4, 1 / 16, 0])
    t = O.build_transform(O.B_HC, 6)
    assert np.allclose(t.q, qt / np.linalg.norm(qt), rtol=1e-13, atol=0)


def test_antireflective_column_n5():
    """test_boundary.cpp:36-53."""
    e = np.array([1, 0.75, 0.5, 0.25, 0])
    assert np.allclose(O.build_transform(O.B_AR, 5).q, e / np.linalg.norm(e), rtol=1e-14)


def test_fourier_grid_and_zero_last_entry():
    """test_boundary.cpp:75-84."""
    a, b, _ = O.extended_grid(O.B_HF, 6)
    assert abs(a + PI / 2) < 1e-15 and abs(b - 2 * PI) < 1e-15
    for n in (5, 9, 33, 128):
        assert O.build_transform(O.B_HF, n).q[-1] == 0.0


def test_cosine_rows_alternate_bitwise():
    """test_boundary.cpp:111-119."""
    t = O.build_transform(O.B_HC, 40)
    j = np.arange(38)
    assert np.array_equal(t.c_b[j % 2 == 0], t.c_a[j % 2 == 0])
    assert np.array_equal(t.c_b[j % 2 == 1], -t.c_a[j % 2 == 1])


def test_symbol_quarter_half_quarter():
    """test_operators.cpp:35-40."""
    p = O.make_psf([0.25, 0.5, 0.25])
    assert abs(O.symbol_eval(p, PI)) < 1e-15
    z = O.symbol_eval(p, PI / 2)
    assert abs(z.real - 0.5) < 1e-15 and z.imag == 0.0


def test_eigenvalue_grids():
    """test_operators.cpp:62-80."""
    assert np.allclose(O.eigenvalue_grid(O.HOC_COSINE, 6), [0, 0, PI / 4, PI / 2, 3 * PI / 4, 0])
    assert np.allclose(O.eigenvalue_grid(O.ANTIREFLECTIVE, 5), [0, PI / 4, PI / 2, 3 * PI / 4, 0])
    assert np.allclose(O.eigenvalue_grid(O.PERIODIC, 4), [0, PI / 2, PI, 3 * PI / 2])


def test_periodic_eigenvalues_quarter_half_quarter():
    """test_oracle.cpp:127-136: (1/4,1/2,1/4) periodic n=4 -> (1, 1/2, 0, 1/2)."""
    d = O.operator_eigenvalues(O.make_psf([0.25, 0.5, 0.25]), 4, O.PERIODIC)
    assert np.allclose(d, [1, 0.5, 0, 0.5], atol=1e-15)


def test_trig_identities():
    """test_trig.cpp:19-101: ones -> sqrt(m) e1; involution; round trips."""
    for m in (1, 2, 7, 64, 255, 4096):
        v = np.ones(m)
        f = O.fourier_apply(v.astype(complex))
        assert abs(f[0] - math.sqrt(m)) < 1e-12 and np.all(np.abs(f[1:]) < 1e-10)
        c = O.cosine_apply(v)
        assert abs(c[0] - math.sqrt(m)) < 1e-12 and np.all(np.abs(c[1:]) < 1e-10)
        x = np.random.default_rng(m).uniform(-1, 1, m)
        assert rel(O.cosine_apply(O.cosine_apply(x), forward=False), x) < 1e-12
        assert rel(O.sine_apply(O.sine_apply(x)), x) < 1e-12


def test_trig_vs_dense_matrices():
    """test_trig.cpp:103-125: entry-wise agreement with oracle.cpp:132-157."""
    for m in (1, 2, 5, 16, 33, 64):
        i, j = np.meshgrid(np.arange(1, m + 1), np.arange(1, m + 1), indexing="ij")
        F = np.exp(-2j * PI * (i - 1) * (j - 1) / m) / math.sqrt(m)
        Cm = np.sqrt(np.where(i == 1, 1.0, 2.0) / m) * np.cos((i - 1) * (2 * j - 1) * PI / (2 * m))
        Q = math.sqrt(2 / (m + 1)) * np.sin(i * j * PI / (m + 1))
        I = np.eye(m)
        assert np.max(np.abs(O.fourier_apply(I.astype(complex).T).T - F)) < 1e-13
        assert np.max(np.abs(O.cosine_apply(I.T).T - Cm)) < 1e-13
        assert np.max(np.abs(O.sine_apply(I.T).T - Q)) < 1e-13


def test_dense_transform_inverse():
    """test_boundary.cpp:182-223: fast inverse equals the dense LU inverse."""
    rng = np.random.default_rng(5)
    for basis in (O.B_AR, O.B_HC, O.B_HF):
        for n in (8, 33, 100):
            t = O.build_transform(basis, n)
            a, b, pts = O.extended_grid(basis, n)
            cols = np.arange(1, n - 1)
            if basis == O.B_AR:
                T = math.sqrt(2 / (n - 1)) * np.sin(np.outer(pts, cols))
            elif basis == O.B_HC:
                T = np.sqrt(np.where(cols == 1, 1.0, 2.0) / (n - 2)) * np.cos(np.outer(pts, cols - 1))
            else:
                T = np.exp(1j * np.outer(pts, cols - 1)) / math.sqrt(n - 2)
            D = np.zeros((n, n), dtype=complex)
            D[:, 0], D[:, n - 1], D[:, 1:n - 1] = t.q, t.q[::-1], T
            y = rng.uniform(-1, 1, n)
            assert rel(O.transform_apply_inverse(t, y), np.linalg.solve(D, y)) < 1e-9
            assert rel(O.transform_apply(t, y), D @ y) < 1e-12


def test_gcv_constant_and_tie():
    """test_regularize.cpp:201-222."""
    n = 16
    op = O.build_operator(O.make_psf([1.0]), n, O.REFLECTIVE)
    s = np.ones(n)
    g = np.random.default_rng(2024).uniform(-1, 1, n)
    want = np.sum(O.cosine_apply(g) ** 2) / n ** 2
    for mu in (1e-10, 1e-4, 1.0, 9.9):
        assert abs(O.gcv_value(op, s, g, mu) / want - 1) < 1e-12
    r = O.gcv_select(op, s, g, 1e-12, 10.0, 200)
    assert r.tied and abs(r.mu / math.sqrt(1e-11) - 1) < 1e-9


# ---------------------------------------------------------------- golden vectors
@pytest.mark.parametrize("bc", range(5))
@pytest.mark.parametrize("n", (6, 33, 64))
def test_golden_transforms(bc, n):
    k = f"bc{bc}_n{n}"
    b = O.SpectralBasis(bc, n)
    x, c = G1[k + "_x"], G1[k + "_c"]
    got = b.analyze(x.astype(complex) if b.complex else x)
    assert rel(got, G1[k + "_analyze"]) < 1e-12
    assert rel(b.synthesize(c), G1[k + "_synth"]) < 1e-12
    op = O.build_operator(O.make_psf(G1[k + "_psf"], True), n, bc)
    assert np.max(np.abs(op.eigenvalues - G1[k + "_eig"])) < 1e-14
    assert rel(op.apply(G1[k + "_f"])[0], G1[k + "_matvec"]) < 1e-12


def test_golden_config0():
    op = O.build_operator(O.make_psf(G1["c0_psf"], True), 1024, O.HOC_COSINE)
    s = np.ones(1024)
    r = O.deblur(op, s, G1["c0_g"], True, mu_min=1e-6, mu_max=1.0, count=64, want_curve=True)
    assert np.max(np.abs(r.curves / G1["c0_curve"] - 1)) < 1e-12
    assert abs(r.mu_used[0] / G1["c0_mu"][0] - 1) < 1e-12
    assert rel(r.restored, G1["c0_restored"]) < 1e-12


def test_golden_config1_slice():
    op = O.build_operator(O.make_psf(G1["c1_psf"], True), 4096, O.HOC_FOURIER)
    s = G1["c1_s"]
    assert np.max(np.abs(O.smoothing_eigenvalues(O.FIRST_DIFFERENCE, O.HOC_FOURIER, 4096) - s)) \
        < 1e-15
    r = O.deblur(op, s, G1["c1_g"], True, mu_min=1e-8, mu_max=1.0, count=256, want_curve=True)
    assert np.max(np.abs(r.curves / G1["c1_curve"] - 1)) < 1e-11
    assert np.max(np.abs(r.mu_used / G1["c1_mu"] - 1)) < 1e-10
    assert rel(r.restored, G1["c1_restored"]) < 1e-10


def test_golden_config2_slice():
    p = O.separable_psf2d(O.make_psf(G2["c2_psf"], True), O.make_psf(G2["c2_psf"], True))
    op = O.build_operator_2d(p, 256, 256, O.HOC_COSINE, separable=True)
    s = O.smoothing_eigenvalues_2d(O.LAPLACIAN, O.HOC_COSINE, 256, 256)
    r = O.deblur_2d(op, s, G2["c2_g"], True, mu_min=1e-6, mu_max=1.0, count=128,
                    want_curve=True)
    assert np.max(np.abs(r.curves / G2["c2_curve"] - 1)) < 1e-11
    assert abs(np.ravel(r.mu_used)[0] / G2["c2_mu"][0] - 1) < 1e-10
    assert rel(r.restored, G2["c2_restored"]) < 1e-10


@pytest.mark.parametrize("name,kind", [("identity", O.IDENTITY), ("laplacian", O.LAPLACIAN)])
def test_golden_config3_slice(name, kind):
    p = O.separable_psf2d(O.make_psf(G2["c3_psf"], True), O.make_psf(G2["c3_psf"], True))
    op = O.build_operator_2d(p, 96, 96, O.HOC_FOURIER, separable=True)
    s = O.smoothing_eigenvalues_2d(kind, O.HOC_FOURIER, 96, 96)
    r = O.deblur_2d(op, s, G2["c3_g"], True, mu_min=1e-6, mu_max=1.0, count=128,
                    want_curve=True)
    assert np.max(np.abs(r.curves / G2[f"c3_{name}_curve"] - 1)) < 1e-11
    assert np.max(np.abs(r.mu_used / G2[f"c3_{name}_mu"] - 1)) < 1e-10
    assert rel(r.restored, G2[f"c3_{name}_restored"]) < 1e-10


def test_golden_general_2d():
    p = O.make_psf2d(G2["disk_psf"], normalize=True)
    op = O.build_operator_2d(p, 16, 20, O.HOC_COSINE)
    assert np.max(np.abs(op.eigenvalues - G2["disk_eig"])) < 1e-13
    assert rel(op.apply(G2["disk_f"])[0], G2["disk_matvec"]) < 1e-11
    s = O.smoothing_eigenvalues_2d(O.LAPLACIAN, O.HOC_COSINE, 16, 20)
    r = O.deblur_2d(op, s, G2["disk_f"], True, mu_min=1e-6, mu_max=1.0, count=32)
    assert abs(np.ravel(r.mu_used)[0] / G2["disk_mu"][0] - 1) < 1e-10
    assert rel(r.restored, G2["disk_restored"]) < 1e-10


# ---------------------------------------------------------------- live reference
needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("bc", range(5))
def test_live_reference_deblur(bc):
    n = 200
    rng = np.random.default_rng(bc)
    psf = np.array([0.1, 0.2, 0.4, 0.2, 0.1]) if bc in (1, 2, 3) else \
        np.array([0.0, 0.0, 0.5, 0.3, 0.2])
    g = np.cumsum(rng.standard_normal((3, n)), axis=-1) / 10
    out, mu, curve, res = R.deblur_1d(psf, n, bc, 1, g, True, mu_min=1e-8, mu_max=1.0, count=50,
                                      want_curve=True)
    op = O.build_operator(O.make_psf(psf, True), n, bc)
    s = O.smoothing_eigenvalues(O.LAPLACIAN, bc, n, op.eigenvalues)
    r = O.deblur(op, s, g, True, mu_min=1e-8, mu_max=1.0, count=50, want_curve=True)
    assert np.max(np.abs(r.curves / curve - 1)) < 1e-11
    assert np.max(np.abs(r.mu_used / mu - 1)) < 1e-10
    assert rel(r.restored, out) < 1e-10


@needs_ref
def test_live_reference_gcv_minimize_paths():
    """gcv_minimize with analytic G: interior minimum, edge minimum, flat (tie)."""
    for G in (lambda m: (math.log(m) + 7.3) ** 2 + 1.0, lambda m: m, lambda m: 2.5):
        mu_ref, curve = R.gcv_minimize(G, 1e-9, 1.0, 40)
        r = O.gcv_minimize(G, 1e-9, 1.0, 40)
        assert abs(r.mu / mu_ref - 1) < 1e-14
        assert np.allclose(r.vals, curve, rtol=0, atol=0)


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("bc,smoother", [(O.HOC_COSINE, O.IDENTITY), (O.HOC_FOURIER, O.LAPLACIAN),
                                         (O.REFLECTIVE, O.LAPLACIAN)])
def test_sweep_mu_pins_reference(bc, smoother):
    """sweep_mu (pipeline.cpp:55-115): curve, RRE per grid mu, summary."""
    psf = gauss(10, 3.0) if bc != O.HOC_FOURIER else onesided(15, 0.2)
    n = 512
    truth, g = W.signals_1d(W.config(0), 3, 1, n=n, m=len(psf) // 2)
    g = W.add_noise(W.convolve_valid(np.pad(truth[0], len(psf) // 2, mode="edge"),
                                     np.asarray(psf) / np.sum(psf)), 0.01, 7)
    op = O.build_operator(O.make_psf(psf, True), n, bc)
    s = O.smoothing_eigenvalues(smoother, bc, n, op.eigenvalues)
    mus, G, rr, summ = O.sweep_mu(op, s, g, truth[0], 1e-6, 1.0, 24)
    rm, rG, rrr, rsumm = R.sweep_mu_1d(psf, n, bc, smoother, g, truth[0], 1e-6, 1.0, 24)
    assert np.array_equal(mus, rm)
    assert np.max(np.abs(G / rG - 1)) < 1e-12
    assert np.max(np.abs(rr / rrr - 1)) < 1e-11
    assert summ[1] == rsumm[1]  # mu_opt: identical grid point
    assert abs(summ[0] / rsumm[0] - 1) < 1e-11
    assert abs(summ[2] / rsumm[2] - 1) < 1e-10
    assert abs(summ[3] / rsumm[3] - 1) < 1e-10
    _, _, rr0, s0 = R.sweep_mu_1d(psf, n, bc, smoother, g, None, 1e-6, 1.0, 24)
    assert np.all(np.isnan(rr0)) and np.isnan(s0[0]) and np.isnan(s0[3])
