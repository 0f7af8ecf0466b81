"""Full-size parity of every BASELINE configuration (VERDICT r1 "untested configs").

Each test runs the configuration at its BASELINE size on the GPU through the
C ABI, on the bench's own seeded inputs (paper_0906_2704_b200/workloads.py),
and compares with the CPU oracle on the same bytes:

* configs 2 and 4 (4096^2, 16384^2 hoc-cosine, Laplacian) against the
  reference itself (oracle/_ref: the unmodified sources compiled by
  oracle/Makefile; deblur_2d pipeline.cpp:157-165, gcv_minimize
  regularize.cpp:144-214, blur_apply_2d multidim.cpp:324-327);
* config 3 (512 x 1024^2 at d = 3, both smoothers, fp64 and fp32): the GPU
  restores the whole 512-image batch, four of its images are checked against
  the numpy HoTransform oracle (the reference has no d = 3);
* config 1 (65,536 x 4096 at d = 1 and d = 3): the GPU restores the whole
  batch, 64 items spread over it are checked against the oracle;
* single images with >= 2^20 coefficients whose GCV minimum is INTERIOR to the
  grid, through the interval screen (and the all-fp64 grid), against the
  reference, plus a 2D batch with interior minima.

Bar (north_star): best_k identical, mu and the restoration within 1e-10
relative in fp64 (1e-4 for the fp32 arm, best_k identical).
"""
import dataclasses
import os

import numpy as np
import pytest
import torch

import fdoracle as O
import paper_0906_2704_b200 as P
import reflib as R
from paper_0906_2704_b200 import workloads as W
from util import np_, rel

pytestmark = pytest.mark.gpu

CORES = len(os.sched_getaffinity(0))
SM_NAME = {0: "identity", 1: "laplacian", 2: "first-difference"}
SM_ORACLE = {0: O.IDENTITY, 1: O.LAPLACIAN, 2: O.FIRST_DIFFERENCE}
needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def _search(cfg):
    return P.GcvSearch(cfg.mu_min, cfg.mu_max, cfg.count)


def _check_single(got_f, got_mu, got_k, ref_f, ref_mu, ref_curve, tol=1e-10):
    want_k = int(np.argmin(ref_curve))
    assert got_k == want_k, (got_k, want_k)
    assert abs(got_mu / ref_mu - 1) < tol, (got_mu, ref_mu)
    assert rel(got_f, ref_f) < tol, rel(got_f, ref_f)


def _gpu_deblur_single(cfg, psf, g, smoother, search):
    op = P.build_operator_2d_separable(psf, psf, g.shape[0], g.shape[1], cfg.bc)
    L = P.smoothing_eigenvalues(SM_NAME[smoother], op)
    rep = P.deblur(op, L, torch.from_numpy(g).cuda(), P.MuChoice(True), search=search)
    torch.cuda.synchronize()
    return op, np_(rep.restored), float(rep.mu_used.cpu().reshape(-1)[0]), int(rep.best_k.cpu().reshape(-1)[0])


def _ref_deblur(cfg, psf, g, smoother, search):
    p2 = np.outer(psf, psf)
    p2 = p2 / float(np.sum(p2))
    out, mu, curve, _ = R.deblur_2d(p2, cfg.bc, smoother, g, True, mu_min=search.mu_min,
                                    mu_max=search.mu_max, count=search.count, eig_mode=1,
                                    threads=CORES, want_curve=True)
    return out[0], float(mu[0]), curve[0]


@needs_ref
def test_config2_full_size():
    """BASELINE config 2: 4096^2, hoc-cosine 2D, Laplacian, 128 lambda in [1e-6, 1]."""
    cfg = W.config(2)
    _, g = W.image_2d(cfg, 0)
    search = _search(cfg)
    _, f, mu, k = _gpu_deblur_single(cfg, cfg.psf, g, cfg.smoothers[0], search)
    rf, rmu, rc = _ref_deblur(cfg, cfg.psf, g, cfg.smoothers[0], search)
    _check_single(f, mu, k, rf, rmu, rc)


@needs_ref
def test_config4_full_size_with_matvec():
    """BASELINE config 4: 16384^2 hoc-cosine 2D, Laplacian, 512 lambda in
    [1e-8, 1]: the re-blur matvec and the GCV restoration (single image:
    interval screen + Taylor-moment golden section on the GPU)."""
    cfg = W.config(4)
    g = W.image_2d_large(4, 0, workers=CORES)
    search = _search(cfg)
    op, f, mu, k = _gpu_deblur_single(cfg, cfg.psf, g, cfg.smoothers[0], search)
    rf, rmu, rc = _ref_deblur(cfg, cfg.psf, g, cfg.smoothers[0], search)
    _check_single(f, mu, k, rf, rmu, rc)
    del f, rf
    # matvec (blur_apply_2d) of the restoration's input image
    got, _ = P.blur_apply(op, torch.from_numpy(g).cuda())
    torch.cuda.synchronize()
    want, _ = R.matvec_2d(cfg.psf2d(), cfg.bc, g, eig_mode=1)
    # T D T^-1 without the filter's damping: |T^-1| ~ n/2 per axis, 4x config
    # 2's (where the reference and its numpy restatement agree to 2.5e-11)
    assert rel(np_(got), want) < 1e-9


@pytest.mark.parametrize("sigma,lo,smoother", [(2.5, 1e-14, 1), (1.0, 1e-14, 1),
                                                (2.5, 1e-18, 0)])
@needs_ref
def test_single_image_interior_minimum(sigma, lo, smoother, monkeypatch):
    """A >= 2^20-coefficient image (1024^2) whose GCV minimum lies strictly
    inside the grid, through the interval screen (single-image path: r
    histogram bounds + exact fp64 candidates) and, with
    FASTDEBLUR_GCV_SCREEN=0, through the all-fp64 grid."""
    cfg = dataclasses.replace(W.config(2), psf=W.gaussian_weights(6, sigma))
    _, g = W.image_2d(cfg, 7, 1024, 1024)
    search = P.GcvSearch(lo, 1.0, 128)
    rf, rmu, rc = _ref_deblur(cfg, cfg.psf, g, smoother, search)
    kk = int(np.argmin(rc))
    assert 0 < kk < search.count - 1, kk  # the case this test exists for
    _, f, mu, k = _gpu_deblur_single(cfg, cfg.psf, g, smoother, search)
    _check_single(f, mu, k, rf, rmu, rc)
    monkeypatch.setenv("FASTDEBLUR_GCV_SCREEN", "0")
    _, f0, mu0, k0 = _gpu_deblur_single(cfg, cfg.psf, g, smoother, search)
    _check_single(f0, mu0, k0, rf, rmu, rc)


@needs_ref
@pytest.mark.parametrize("screen", ["1", "0"])
def test_batch_2d_interior_minima(screen, monkeypatch):
    """A batch sharing one 2D operator (the batched GCV path: GEMM / screen)
    with interior GCV minima, against the reference image by image."""
    monkeypatch.setenv("FASTDEBLUR_GCV_SCREEN", screen)
    cfg = dataclasses.replace(W.config(2), psf=W.gaussian_weights(6, 1.0))
    n, B = 256, 36
    g = np.stack([W.image_2d(cfg, 100 + i, n, n)[1] for i in range(B)])
    search = P.GcvSearch(1e-14, 1.0, 128)
    op = P.build_operator_2d_separable(cfg.psf, cfg.psf, n, n, cfg.bc)
    L = P.smoothing_eigenvalues("laplacian", op)
    rep = P.deblur(op, L, torch.from_numpy(g).cuda(), P.MuChoice(True), search=search)
    p2 = cfg.psf2d()
    out, mu, curve, _ = R.deblur_2d(p2, cfg.bc, 1, g, True, mu_min=search.mu_min,
                                    mu_max=search.mu_max, count=search.count, eig_mode=1,
                                    threads=CORES, want_curve=True)
    bk = np.argmin(curve, axis=1)
    assert np.all((bk > 0) & (bk < search.count - 1))
    assert np.array_equal(np_(rep.best_k), bk)
    assert np.max(np.abs(np_(rep.mu_used) / mu - 1)) < 1e-10
    assert rel(np_(rep.restored), out) < 1e-10


CONFIG3_ITEMS = [0, 1, 255, 511]


@pytest.fixture(scope="module")
def config3_batch():
    cfg = W.config(3)
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    with ProcessPoolExecutor(max_workers=max(1, min(CORES, 16)),
                             mp_context=mp.get_context("fork")) as ex:
        imgs = list(ex.map(_gen3, range(cfg.batch)))
    return np.stack(imgs)


def _gen3(i):
    return W.image_2d(W.config(3), i)[1]


@pytest.mark.parametrize("smoother", [0, 1])
def test_config3_full_batch(config3_batch, smoother):
    """BASELINE config 3: the whole 512 x 1024^2 batch at d = 3 (separable
    one-sided motion blur), fp64 and fp32 storage; images 0, 1, 255, 511
    against the HoTransform oracle (fp64: 1e-10; fp32: 1e-4 against the fp64
    oracle on the rounded input)."""
    cfg = W.config(3)
    bc = W.HOC_FOURIER_D3
    g = config3_batch
    n1, n2 = cfg.n1, cfg.n2
    search = _search(cfg)
    op = P.build_operator_2d_separable(cfg.psf, cfg.psf, n1, n2, bc)
    L = P.smoothing_eigenvalues(SM_NAME[smoother], op)
    psf = O.make_psf(cfg.psf, True)
    oop = O.build_operator_2d(O.separable_psf2d(psf, psf), n1, n2, bc, separable=True)
    s = O.smoothing_eigenvalues_2d(SM_ORACLE[smoother], bc, n1, n2, oop.eigenvalues)
    sel = np.array(CONFIG3_ITEMS)
    for dt, tol in ((torch.float64, 1e-10), (torch.float32, 1e-4)):
        gd = torch.from_numpy(g).to("cuda", dt)
        rep = P.deblur(op, L, gd, P.MuChoice(True), search=search)
        torch.cuda.synchronize()
        gs = np_(gd[torch.from_numpy(sel).cuda()]).astype(np.float64)
        want = O.deblur_2d(oop, s, gs, True, mu_min=cfg.mu_min, mu_max=cfg.mu_max,
                           count=cfg.count)
        assert np.array_equal(np_(rep.best_k)[sel], want.best_k)
        assert np.max(np.abs(np_(rep.mu_used)[sel] / want.mu_used - 1)) < tol
        got = np_(rep.restored[torch.from_numpy(sel).cuda()]).astype(np.float64)
        for i in range(len(sel)):
            assert rel(got[i], want.restored[i]) < tol, (dt, i, rel(got[i], want.restored[i]))
        del gd, rep


CONFIG1_ITEMS = np.concatenate([np.arange(0, 65536, 2048), 1023 + np.arange(0, 65536, 2048)])


@pytest.fixture(scope="module")
def config1_batch():
    cfg = W.config(1)
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    jobs = [(s0, 1024) for s0 in range(0, cfg.batch, 1024)]
    out = np.empty((cfg.batch, cfg.n1))
    with ProcessPoolExecutor(max_workers=max(1, min(CORES, 32)),
                             mp_context=mp.get_context("fork")) as ex:
        for (s0, c), arr in zip(jobs, ex.map(_gen1, jobs)):
            out[s0:s0 + c] = arr
    return out


def _gen1(job):
    s0, c = job
    return W.signals_1d(W.config(1), s0, c)[1]


@pytest.mark.parametrize("bc", [W.HOC_FOURIER_D1, W.HOC_FOURIER_D3, W.HOC_FOURIER])
def test_config1_full_batch(config1_batch, bc):
    """BASELINE config 1: the whole 65,536 x 4096 batch (first-difference
    smoother, 256 lambda in [1e-8, 1]) at d = 1 and d = 3 (and d = 2, the
    reference's hoc-fourier, checked against the reference itself); 64 items
    spread over the batch against the oracle."""
    cfg = W.config(1)
    g = config1_batch
    n = cfg.n1
    search = _search(cfg)
    op = P.build_operator(cfg.psf, n, bc)
    L = P.smoothing_eigenvalues("first-difference", op)
    rep = P.deblur(op, L, torch.from_numpy(g).cuda(), P.MuChoice(True), search=search)
    torch.cuda.synchronize()
    sel = CONFIG1_ITEMS
    oop = O.build_operator(O.make_psf(cfg.psf, normalize=True), n, bc)
    s = O.smoothing_eigenvalues(O.FIRST_DIFFERENCE, bc, n, oop.eigenvalues)
    assert np.max(np.abs(np_(L.eigenvalues()) - s)) < 1e-14
    want = O.deblur(oop, s, g[sel], True, mu_min=cfg.mu_min, mu_max=cfg.mu_max,
                    count=cfg.count)
    assert np.array_equal(np_(rep.best_k)[sel], want.best_k)
    assert np.max(np.abs(np_(rep.mu_used)[sel] / want.mu_used - 1)) < 1e-10
    got = np_(rep.restored)[sel]
    for i in range(len(sel)):
        assert rel(got[i], want.restored[i]) < 1e-10
    if bc == W.HOC_FOURIER and R.available():
        out, mu, curve, _ = R.deblur_1d(cfg.psf, n, bc, 2, g[sel], True, mu_min=cfg.mu_min,
                                        mu_max=cfg.mu_max, count=cfg.count, threads=CORES,
                                        want_curve=True, s_custom=s)
        assert np.array_equal(np_(rep.best_k)[sel], np.argmin(curve, axis=1))
        assert np.max(np.abs(np_(rep.mu_used)[sel] / mu - 1)) < 1e-10
        assert rel(got, out) < 1e-10
