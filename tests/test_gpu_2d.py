"""GPU parity of the 2D path (multidim.cpp): tensor transforms, three-step
eigenvalues, separable fast path, matvec, Tikhonov and GCV restoration."""
import numpy as np
import pytest
import torch

import fdoracle as O
import paper_0906_2704_b200 as P
from paper_0906_2704_b200 import workloads as W
from util import gauss, np_, onesided, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bc", range(5))
@pytest.mark.parametrize("shape", [(12, 12), (14, 18), (33, 20), (64, 64)])
def test_tensor_transforms(bc, shape, rng):
    n1, n2 = shape
    op = P.build_operator_2d(np.ones((1, 1)), n1, n2, bc)
    r, c = O.SpectralBasis(bc, n1), O.SpectralBasis(bc, n2)
    x = rng.standard_normal((2, n1, n2))
    got = np_(op.analyze(torch.from_numpy(x)))
    want = O.tensor_apply(r, c, x.astype(complex) if r.complex else x, forward=False)
    assert rel(got, want) < 1e-11
    cc = rng.standard_normal((2, n1, n2)) + (1j * rng.standard_normal((2, n1, n2))
                                             if r.complex else 0)
    s = op.synthesize(torch.from_numpy(cc))
    s = np_(s if r.complex else s[0])
    assert rel(s, O.tensor_apply(r, c, cc, forward=True)) < 1e-12


def _disk(radius):
    j = np.arange(-radius, radius + 1)
    return (j[:, None] ** 2 + j[None, :] ** 2 <= radius * radius).astype(float)


@pytest.mark.parametrize("bc,psf2", [
    (O.HOC_COSINE, _disk(2)), (O.REFLECTIVE, _disk(3)), (O.ANTIREFLECTIVE, _disk(2)),
    (O.HOC_FOURIER, np.outer(onesided(3, 0.5), gauss(2, 1.0)) + 0.01),
    (O.PERIODIC, np.outer(onesided(3, 0.5), onesided(2, 0.3)))])
def test_general_2d_operator(bc, psf2, rng):
    n1, n2 = 14, 18
    op = P.build_operator_2d(psf2, n1, n2, bc)
    p = O.make_psf2d(psf2, normalize=True)
    oop = O.build_operator_2d(p, n1, n2, bc)
    assert np.max(np.abs(np_(op.eigenvalues()) - oop.eigenvalues)) < 1e-13
    f = rng.standard_normal((n1, n2))
    got, _ = op.apply(torch.from_numpy(f))
    want, _ = oop.apply(f)
    assert rel(np_(got), want) < 1e-11
    L = P.smoothing_eigenvalues("laplacian", op)
    s = O.smoothing_eigenvalues_2d(O.LAPLACIAN, bc, n1, n2, oop.eigenvalues)
    rep = P.deblur(op, L, torch.from_numpy(f), P.MuChoice(True),
                   search=P.GcvSearch(1e-6, 1.0, 32))
    w = O.deblur_2d(oop, s, f, True, mu_min=1e-6, mu_max=1.0, count=32)
    assert int(np_(rep.best_k)) == int(w.best_k)
    assert rel(np_(rep.restored), w.restored) < 1e-10


@pytest.mark.parametrize("bc,a,b", [(O.HOC_COSINE, gauss(3, 1.2), gauss(2, 1.0)),
                                    (O.HOC_FOURIER, onesided(4, 0.25), onesided(3, 0.5)),
                                    (O.REFLECTIVE, gauss(2, 1.0), gauss(2, 1.0))])
@pytest.mark.parametrize("smoother", ["identity", "laplacian"])
def test_separable_2d_pipeline(bc, a, b, smoother, rng):
    n1, n2 = 48, 40
    op = P.build_operator_2d_separable(a, b, n1, n2, bc)
    p = O.separable_psf2d(O.make_psf(a, True), O.make_psf(b, True))
    oop = O.build_operator_2d(p, n1, n2, bc, separable=True)
    assert np.max(np.abs(np_(op.eigenvalues()) - oop.eigenvalues)) < 1e-14
    # separable eigenvalues agree with the three-step direct scheme
    assert np.max(np.abs(oop.eigenvalues - O.eigenvalues_2d(p, n1, n2, bc))) < 1e-10
    f = rng.standard_normal((3, n1, n2))
    got, _ = op.apply(torch.from_numpy(f))
    want, _ = oop.apply(f)
    assert rel(np_(got), want) < 1e-11
    kind = O.IDENTITY if smoother == "identity" else O.LAPLACIAN
    L = P.smoothing_eigenvalues(smoother, op)
    s = O.smoothing_eigenvalues_2d(kind, bc, n1, n2, oop.eigenvalues)
    assert np.max(np.abs(np_(L.eigenvalues()) - s)) < 1e-14
    rep = P.deblur(op, L, torch.from_numpy(f), P.MuChoice(True), want_curve=True,
                   search=P.GcvSearch(1e-6, 1.0, 128))
    w = O.deblur_2d(oop, s, f, True, mu_min=1e-6, mu_max=1.0, count=128, want_curve=True)
    assert np.array_equal(np_(rep.best_k), w.best_k)
    assert np.max(np.abs(np_(rep.gcv_curve) / w.curves - 1)) < 1e-11
    assert np.max(np.abs(np_(rep.mu_used) / w.mu_used - 1)) < 1e-10
    assert rel(np_(rep.restored), w.restored) < 1e-10


def test_config2_scaled_image():
    """BASELINE config 2 family (hoc-cosine, Laplacian, 128 lambda) at 256^2."""
    cfg = W.config(2)
    truth, g = W.image_2d(cfg, 0, 256, 256)
    op = P.build_operator_2d_separable(cfg.psf, cfg.psf, 256, 256, cfg.bc)
    L = P.smoothing_eigenvalues("laplacian", op)
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True),
                   search=P.GcvSearch(cfg.mu_min, cfg.mu_max, cfg.count))
    p = O.separable_psf2d(O.make_psf(cfg.psf, True), O.make_psf(cfg.psf, True))
    oop = O.build_operator_2d(p, 256, 256, cfg.bc, separable=True)
    s = O.smoothing_eigenvalues_2d(O.LAPLACIAN, cfg.bc, 256, 256)
    w = O.deblur_2d(oop, s, g, True, mu_min=cfg.mu_min, mu_max=cfg.mu_max, count=cfg.count)
    assert int(np_(rep.best_k)) == int(w.best_k)
    assert rel(np_(rep.restored), w.restored) < 1e-10


@pytest.mark.parametrize("bc,smoother,search", [("hoc-cosine", "laplacian", (1e-8, 1.0, 512)),
                                                ("hoc-fourier", "identity", (1e-6, 1.0, 128)),
                                                ("reflective", "laplacian", (1e-6, 1.0, 7))])
def test_interval_screen_single_image(bc, smoother, search, monkeypatch):
    """Single large images (>= 2^20 coefficients) bound G on every grid point
    from an r-histogram and evaluate exactly only the possible minima: the
    same best_k, mu and restoration as the full fp64 grid."""
    import paper_0906_2704_b200 as PP
    n1, n2 = 1024, 1040
    psf = W.gaussian_weights(6, 2.0) if bc != "hoc-fourier" else W.onesided_exp_weights(7, 0.25)
    op = PP.build_operator_2d_separable(psf, psf, n1, n2, bc)
    L = PP.smoothing_eigenvalues(smoother, op)
    _, g = W.image_2d(W.config(2), 3, n1, n2)
    sr = PP.GcvSearch(*search)
    rep = PP.deblur(op, L, torch.from_numpy(g), PP.MuChoice(True), search=sr)
    monkeypatch.setenv("FASTDEBLUR_GCV_SCREEN", "0")
    ref = PP.deblur(op, L, torch.from_numpy(g), PP.MuChoice(True), search=sr)
    assert int(rep.best_k.cpu()) == int(ref.best_k.cpu())
    assert abs(float(rep.mu_used.cpu()) / float(ref.mu_used.cpu()) - 1) < 1e-12
    assert rel(rep.restored.cpu().numpy(), ref.restored.cpu().numpy()) < 1e-12


def test_deblur_smoothers_equals_separate_calls(rng):
    """fd_deblur_smoothers (one analysis, several smoothing norms) returns exactly
    what separate deblur calls return: 2D d = 3 batch (config-3 shape, fp64 and
    fp32 storage), a 1D hoc-fourier batch and a fixed mu."""
    from paper_0906_2704_b200 import workloads as W
    cfg = W.config(3)
    n, B = 96, 40
    g = np.stack([W.image_2d(cfg, i, n, n)[1] for i in range(B)])
    op = P.build_operator_2d_separable(cfg.psf, cfg.psf, n, n, W.HOC_FOURIER_D3)
    Ls = [P.smoothing_eigenvalues(k, op) for k in ("identity", "laplacian")]
    search = P.GcvSearch(1e-6, 1.0, 64)
    for dt in (torch.float64, torch.float32):
        gd = torch.from_numpy(g).to("cuda", dt)
        got = P.deblur_smoothers(op, Ls, gd, P.MuChoice(True), search=search)
        for L, r in zip(Ls, got):
            w = P.deblur(op, L, gd, P.MuChoice(True), search=search)
            assert torch.equal(r.best_k, w.best_k)
            assert torch.equal(r.mu_used, w.mu_used)
            assert torch.equal(r.restored, w.restored)
    op1 = P.build_operator(onesided(9, 0.3), 512, "hoc-fourier")
    L1 = [P.smoothing_eigenvalues(k, op1) for k in ("laplacian", "identity")]
    g1 = torch.from_numpy(rng.standard_normal((50, 512)) + 3.0).cuda()
    for mu in (P.MuChoice(True), P.MuChoice(False, 1e-3)):
        got = P.deblur_smoothers(op1, L1, g1, mu, search=search)
        for L, r in zip(L1, got):
            w = P.deblur(op1, L, g1, mu, search=search)
            assert torch.equal(r.mu_used, w.mu_used) and torch.equal(r.restored, w.restored)
