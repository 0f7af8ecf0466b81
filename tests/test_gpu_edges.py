"""Edge cases of the batched device path (empty and ragged
batches, maximum sizes, degenerate items), checked through the C ABI against
the numpy restatement (oracle/fdoracle.py).

* empty batch: no launch, empty outputs, no error;
* ragged batches around the tensor-core screen's 128-item tiles and the pair
  kernels' two-lines-per-DFT packing (1, 2, 127, 129, 257 items), at d = 1
  (direct mixed-radix DFT, m = n - 1 = 1023 = 3 * 11 * 31 -> falls back to
  Bluestein, and m = 4095 = 13 * 9 * 7 * 5) and d = 3 (Bluestein);
* maximum 1D line length of the split-convolution path (n = 16384, the
  config-4 line, DCT of 16382 = 2 * 8191 points);
* constant and all-zero items inside a batch (the reference's degenerate
  GCV cases: a constant G curve ties at every grid point)."""
import numpy as np
import pytest
import torch

import fdoracle as O
import paper_0906_2704_b200 as P
from paper_0906_2704_b200 import workloads as W
from util import gauss, np_, onesided, rel

pytestmark = pytest.mark.gpu

SM = {0: O.IDENTITY, 1: O.LAPLACIAN, 2: O.FIRST_DIFFERENCE}


def _setup(bc, psf, n, smoother):
    op = P.build_operator(psf, n, bc)
    L = P.smoothing_eigenvalues(smoother, op)
    oop = O.build_operator(O.make_psf(psf, normalize=True), n, bc)
    s = O.smoothing_eigenvalues(SM[smoother], bc, n, oop.eigenvalues)
    return op, L, oop, s


def _scenes(n, psf, B, seed, noise=0.005):
    truth, _ = W.signals_1d(W.config(1), seed, B, n=n + len(psf) - 1, m=0)
    return W.add_noise(W.convolve_valid(truth, np.asarray(psf) / np.sum(psf)), noise,
                       W.item_key(seed, np.arange(B, dtype=np.uint64)))


@pytest.mark.parametrize("bc", [O.HOC_COSINE, O.HOC_FOURIER_D1, O.HOC_FOURIER_D3])
def test_empty_batch(bc):
    n = 256
    op, L, _, _ = _setup(bc, onesided(5, 0.3) if bc != O.HOC_COSINE else gauss(3, 1.0), n, 1)
    g = torch.empty((0, n), dtype=torch.float64)
    rep = P.deblur(op, L, g, P.MuChoice(True), search=P.GcvSearch(1e-6, 1.0, 32))
    assert tuple(rep.restored.shape) == (0, n)
    assert rep.mu_used.numel() == 0
    assert tuple(op.analyze(g).shape)[0] == 0


@pytest.mark.parametrize("bc,n", [(O.HOC_FOURIER_D1, 1024), (O.HOC_FOURIER_D3, 1024),
                                  (O.HOC_FOURIER_D1, 4096), (O.HOC_FOURIER_D3, 4096),
                                  (O.HOC_FOURIER, 1024)])
@pytest.mark.parametrize("B", [1, 2, 127, 129, 257])
def test_ragged_batches(bc, n, B):
    psf = onesided(15, 0.2)
    op, L, oop, s = _setup(bc, psf, n, 2)
    g = _scenes(n, psf, B, 900 + B)
    search = (1e-8, 1.0, 256)
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True),
                   search=P.GcvSearch(*search))
    sel = sorted({0, B // 2, B - 1})
    want = O.deblur(oop, s, g[sel], True, mu_min=search[0], mu_max=search[1], count=search[2])
    assert np.array_equal(np_(rep.best_k)[sel], want.best_k)
    assert np.max(np.abs(np_(rep.mu_used)[sel] / want.mu_used - 1)) < 1e-10
    assert rel(np_(rep.restored)[sel], want.restored) < 1e-10


def test_max_line_length_split_convolution():
    """n = 16384 hoc-cosine 1D (config-4 line length): split-half Bluestein
    convolution with per-CTA scratch (M = 16384 beyond shared memory)."""
    n = 16384
    psf = gauss(16, 4.0)
    op, L, oop, s = _setup(O.HOC_COSINE, psf, n, 1)
    g = _scenes(n, psf, 3, 77, noise=0.01)
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True),
                   search=P.GcvSearch(1e-8, 1.0, 512))
    want = O.deblur(oop, s, g, True, mu_min=1e-8, mu_max=1.0, count=512)
    assert np.array_equal(np_(rep.best_k), want.best_k)
    assert np.max(np.abs(np_(rep.mu_used) / want.mu_used - 1)) < 1e-10
    assert rel(np_(rep.restored), want.restored) < 1e-10
    x = np.random.default_rng(3).standard_normal((2, n))
    back = np_(op.synthesize(op.analyze(torch.from_numpy(x)))[0])
    assert rel(back, x) < 1e-10


@pytest.mark.parametrize("bc", [O.HOC_FOURIER_D1, O.HOC_FOURIER_D3, O.HOC_COSINE])
def test_constant_and_zero_items_in_batch(bc):
    """A constant signal is an eigenvector with eigenvalue 1 of every
    polynomial-preserving BC and lies in the Laplacian smoother's null space:
    it is restored exactly whatever mu.  Its G curve is rounding noise (every
    sigma-weighted coefficient is an FFT round-off residue, ~1e-32), so its grid
    argmin is not a parity quantity -- the compiled reference, numpy and cuFFT
    each pick a different one; only the restoration is compared.  A zero item
    gives an identically zero curve: ties everywhere, the geometric mean of the
    grid (regularize.cpp:172-185), best_k 0 -- the pair analysis kernels flag
    all-zero lines so their partner's DFT round-off does not leak into them --
    and an exactly zero restoration.  Both sit among
    ordinary items of a batch large enough for the tensor-core screen."""
    n, B = 512, 200
    psf = onesided(15, 0.2) if bc != O.HOC_COSINE else gauss(10, 3.0)
    op, L, oop, s = _setup(bc, psf, n, 1)
    g = _scenes(n, psf, B, 31)
    g[5] = 0.75
    g[6] = 0.0
    search = (1e-8, 1.0, 256)
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True), want_curve=True,
                   search=P.GcvSearch(*search))
    sel = [4, 6, 7]
    want = O.deblur(oop, s, g[sel], True, mu_min=search[0], mu_max=search[1], count=search[2])
    assert np.array_equal(np_(rep.best_k)[sel], want.best_k)
    assert np.max(np.abs(np_(rep.mu_used)[sel] / want.mu_used - 1)) < 1e-10
    assert rel(np_(rep.restored)[sel], want.restored) < 1e-10
    curve = np_(rep.gcv_curve)
    assert np.max(curve[5]) < 1e-20 * np.min(curve[4])
    assert np.max(np.abs(np_(rep.restored)[5] - 0.75)) < 1e-12
    # the zero item's restoration is exactly zero, as the reference's (its
    # pair partner's inverse-DFT round-off must not leak into it: the pair
    # synthesis kernels flag all-zero filtered lines)
    f = np_(rep.restored)
    assert np.max(np.abs(f[6])) == 0.0
    assert abs(np_(rep.mu_used)[6] - np.sqrt(search[0] * search[1])) < 1e-12


@pytest.mark.parametrize("bc", [O.HOC_FOURIER_D1, O.HOC_FOURIER_D3])
def test_pair_kernels_unaligned_input(bc):
    """The n = 4096 line-pair kernels stage their input lines with bulk copies
    and bulk-store their outputs when the lines are 16-byte aligned; a batch
    that starts 8 bytes off takes their direct-access loads instead.  Both must
    agree with the oracle, and a zero line among the items stays exactly zero
    (zero-line flags of the staged and the direct path)."""
    n, B = 4096, 5
    psf = onesided(15, 0.2)
    op, L, oop, s = _setup(bc, psf, n, 2)
    g = _scenes(n, psf, B, 77)
    g[3] = 0.0
    big = torch.zeros(B * n + 1, dtype=torch.float64, device="cuda")
    view = big[1:].view(B, n)
    view.copy_(torch.from_numpy(g))
    assert view.data_ptr() % 16 == 8
    search = (1e-8, 1.0, 256)
    want = O.deblur(oop, s, g, True, mu_min=search[0], mu_max=search[1], count=search[2])
    for src in (view, torch.from_numpy(g).cuda()):
        rep = P.deblur(op, L, src, P.MuChoice(True), search=P.GcvSearch(*search))
        keep = [0, 1, 2, 4]
        assert np.array_equal(np_(rep.best_k)[keep], want.best_k[keep])
        assert np.max(np.abs(np_(rep.mu_used)[keep] / want.mu_used[keep] - 1)) < 1e-10
        assert rel(np_(rep.restored)[keep], want.restored[keep]) < 1e-10
        assert np.all(np_(rep.restored)[3] == 0.0)


@pytest.mark.parametrize("bc,n", [(O.HOC_FOURIER_D3, 250), (O.HOC_FOURIER_D3, 3000),
                                  (O.HOC_FOURIER_D1, 3000), (O.HOC_FOURIER_D3, 2052)])
def test_pair_kernels_other_fold_sizes(bc, n):
    """Bluestein line-pair kernels at sizes other than config 1's: M = 512 (the
    folded radix-2 stage without thread groups), and M = 8192 with m = 2997,
    2999 (d = 1: one border column) and 2049 (the smallest m of that size) --
    the staged output lines, weight rows and spectral table are sized by m."""
    B = 7
    psf = onesided(9, 0.25)
    op, L, oop, s = _setup(bc, psf, n, 2)
    g = _scenes(n, psf, B, 55 + n)
    search = (1e-8, 1.0, 64)
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True), search=P.GcvSearch(*search))
    want = O.deblur(oop, s, g, True, mu_min=search[0], mu_max=search[1], count=search[2])
    assert np.array_equal(np_(rep.best_k), want.best_k)
    assert np.max(np.abs(np_(rep.mu_used) / want.mu_used - 1)) < 1e-9
    assert rel(np_(rep.restored), want.restored) < 1e-9


@pytest.mark.parametrize("bc", [O.HOC_FOURIER_D1, O.HOC_FOURIER_D3])
def test_pair_kernels_run_to_run_identical(bc):
    """The line-pair kernels hand data between thread groups, the bulk-copy
    engine and the generic proxy through shared memory (staged input, output
    lines assembled in the FFT buffer, skewed thread groups on named
    barriers).  A missing barrier or fence shows up as run-to-run differences:
    three restorations of the same 2,049-item batch (persistent CTAs with
    several pairs each, odd count) must agree bit for bit."""
    n, B = 4096, 2049
    cfg = W.config(1)
    _, g = W.signals_1d(cfg, 3, B)
    op = P.build_operator(cfg.psf, n, bc)
    L = P.smoothing_eigenvalues(2, op)
    gd = torch.from_numpy(g).cuda()
    outs = []
    for _ in range(3):
        rep = P.deblur(op, L, gd, P.MuChoice(True),
                       search=P.GcvSearch(cfg.mu_min, cfg.mu_max, cfg.count))
        torch.cuda.synchronize()
        outs.append((rep.restored.clone(), rep.mu_used.clone(), rep.best_k.clone()))
    for f, mu, k in outs[1:]:
        assert torch.equal(f, outs[0][0])
        assert torch.equal(mu, outs[0][1])
        assert torch.equal(k, outs[0][2])
    assert torch.isfinite(outs[0][0]).all()
