"""fp32 storage variant (BASELINE config 3 "fp32 and fp64"; include/fastdeblur_b200.h
fd_*_f32): float inputs / outputs, fp64 arithmetic.  Checked against the fp64
oracle run on the same fp32-rounded input: identical best_k, mu within 1e-10
and the restoration within fp32 output rounding -- far inside the north_star
fp32 bar (1e-4 relative)."""
import numpy as np
import pytest
import torch

import fdoracle as O
import paper_0906_2704_b200 as P
from paper_0906_2704_b200 import workloads as W
from util import np_, onesided, rel

pytestmark = pytest.mark.gpu
SM = {0: O.IDENTITY, 1: O.LAPLACIAN, 2: O.FIRST_DIFFERENCE}


@pytest.mark.parametrize("bc", [O.HOC_FOURIER_D3, O.HOC_FOURIER, O.HOC_COSINE])
@pytest.mark.parametrize("smoother", [0, 1])
def test_2d_deblur_f32(bc, smoother):
    cfg = W.config(3)
    n1, n2, B = 128, 96, 3
    a = cfg.psf if bc != O.HOC_COSINE else W.gaussian_weights(5, 1.5)
    g = np.stack([W.image_2d(cfg, i, n1, n2)[1] for i in range(B)]).astype(np.float32)
    op = P.build_operator_2d_separable(a, a, n1, n2, bc)
    L = P.smoothing_eigenvalues(smoother, op)
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True), want_curve=True,
                   search=P.GcvSearch(1e-6, 1.0, 128))
    assert rep.restored.dtype == torch.float32
    p2 = O.separable_psf2d(O.make_psf(a, True), O.make_psf(a, True))
    oop = O.build_operator_2d(p2, n1, n2, bc, separable=True)
    s = O.smoothing_eigenvalues_2d(SM[smoother], bc, n1, n2, oop.eigenvalues)
    want = O.deblur_2d(oop, s, g.astype(np.float64), True, mu_min=1e-6, mu_max=1.0, count=128,
                       want_curve=True)
    assert np.array_equal(np_(rep.best_k), want.best_k)
    assert np.max(np.abs(np_(rep.mu_used) / want.mu_used - 1)) < 1e-10
    assert np.max(np.abs(np_(rep.gcv_curve) / want.curves - 1)) < 1e-10
    assert rel(np_(rep.restored).astype(np.float64), want.restored) < 1e-6


@pytest.mark.parametrize("bc", [O.HOC_FOURIER_D1, O.HOC_FOURIER_D3, O.HOC_FOURIER,
                                O.HOC_COSINE])
def test_1d_deblur_matvec_f32(bc):
    n, B = 1024, 40
    psf = onesided(15, 0.2) if bc != O.HOC_COSINE else W.gaussian_weights(6, 2.0)
    truth, _ = W.signals_1d(W.config(1), 3, B, n=n + len(psf) - 1, m=0)
    g = W.add_noise(W.convolve_valid(truth, np.asarray(psf) / np.sum(psf)), 0.005,
                    W.item_key(5, np.arange(B, dtype=np.uint64))).astype(np.float32)
    op = P.build_operator(psf, n, bc)
    L = P.smoothing_eigenvalues(1, op)
    oop = O.build_operator(O.make_psf(psf, normalize=True), n, bc)
    s = O.smoothing_eigenvalues(O.LAPLACIAN, bc, n, oop.eigenvalues)
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True),
                   search=P.GcvSearch(1e-8, 1.0, 256))
    want = O.deblur(oop, s, g.astype(np.float64), True, mu_min=1e-8, mu_max=1.0, count=256)
    assert np.array_equal(np_(rep.best_k), want.best_k)
    assert np.max(np.abs(np_(rep.mu_used) / want.mu_used - 1)) < 1e-10
    assert rel(np_(rep.restored).astype(np.float64), want.restored) < 1e-6
    got, _ = P.blur_apply(op, torch.from_numpy(g))
    assert got.dtype == torch.float32
    assert rel(np_(got).astype(np.float64), oop.apply(g.astype(np.float64))[0]) < 1e-6
    # host-buffer pipeline, fp32
    r2, mu2, bk2 = P.deblur_host(op, L, torch.from_numpy(g), P.MuChoice(True),
                                 search=P.GcvSearch(1e-8, 1.0, 256), chunk=16)
    assert r2.dtype == torch.float32
    assert np.array_equal(bk2.numpy(), want.best_k)
    assert rel(r2.numpy().astype(np.float64), want.restored) < 1e-6
