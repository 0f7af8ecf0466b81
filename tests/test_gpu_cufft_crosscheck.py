"""cuFFT cross-check (north_star: "no cuFFT on the product path; cuFFT is used
only as a cross-check").

The numpy restatement (oracle/fdoracle.py) runs every trigonometric transform
through np.fft.fft / np.fft.ifft (trig.cpp's FFTW calls).  Here the oracle's
FFT engine is swapped for cuFFT (torch.fft on cuda:0, complex128) and the
whole restoration -- border fold, interior DFT / DCT / DST, filter, GCV grid,
golden section, synthesis -- is recomputed on top of it; the hand-written
sm_100a kernels must agree with that cuFFT-backed pipeline to the north_star
bar (best_k identical, mu and restoration within 1e-10).  A third opinion next
to the FFTW stand-in (oracle/_ref) and numpy's pocketfft, on the GPU itself.
Plus the direct check: the periodic basis' analyze is the unitary DFT, i.e.
cuFFT with norm="ortho"."""
import types

import numpy as np
import pytest
import torch

import fdoracle as O
import paper_0906_2704_b200 as P
from paper_0906_2704_b200 import workloads as W
from util import gauss, np_, onesided, rel

pytestmark = pytest.mark.gpu


def _cufft(fn):
    def run(a, axis=-1):
        a = np.moveaxis(np.asarray(a, dtype=np.complex128), axis, -1)
        t = torch.from_numpy(np.ascontiguousarray(a)).to("cuda")
        out = fn(t, dim=-1).cpu().numpy()
        return np.moveaxis(out, -1, axis)
    return run


class _NumpyWithCufft:
    """numpy, except that .fft.fft / .fft.ifft are cuFFT."""
    fft = types.SimpleNamespace(fft=_cufft(torch.fft.fft), ifft=_cufft(torch.fft.ifft))

    def __getattr__(self, k):
        return getattr(np, k)


@pytest.fixture
def cufft_oracle(monkeypatch):
    monkeypatch.setattr(O, "np", _NumpyWithCufft())
    return O


@pytest.mark.parametrize("n", [64, 1022, 4093, 4096])
def test_periodic_analyze_is_cufft(n, rng):
    op = P.build_operator([1.0], n, O.PERIODIC)
    x = rng.standard_normal((3, n)) + 1j * rng.standard_normal((3, n))
    got = np_(op.analyze(torch.from_numpy(x)))
    want = torch.fft.fft(torch.from_numpy(x).cuda(), dim=-1, norm="ortho").cpu().numpy()
    assert rel(got, want) < 1e-13, rel(got, want)
    back = np_(op.synthesize(torch.from_numpy(got)))
    assert rel(back, x) < 1e-13


def _scenes(n, psf, B, seed, noise):
    cfg = W.config(1)
    truth, _ = W.signals_1d(cfg, seed, B, n=n + len(psf) - 1, m=0)
    return W.add_noise(W.convolve_valid(truth, np.asarray(psf) / np.sum(psf)), noise,
                       W.item_key(seed, np.arange(B, dtype=np.uint64)))


SM = {0: O.IDENTITY, 1: O.LAPLACIAN, 2: O.FIRST_DIFFERENCE}
CASES = [  # (bc, psf, n, B, smoother, search)
    (O.HOC_COSINE, gauss(10, 3.0), 1024, 1, 0, (1e-6, 1.0, 64)),         # config 0
    (O.HOC_FOURIER_D1, onesided(15, 0.2), 4096, 4, 2, (1e-8, 1.0, 256)),  # config 1, d = 1
    (O.HOC_FOURIER_D3, onesided(15, 0.2), 4096, 4, 2, (1e-8, 1.0, 256)),  # config 1, d = 3
    (O.HOC_FOURIER, onesided(15, 0.2), 4096, 3, 1, (1e-8, 1.0, 256)),
    (O.PERIODIC, gauss(7, 2.0), 4096, 2, 1, (1e-8, 1.0, 128)),
    (O.REFLECTIVE, gauss(7, 2.0), 2049, 2, 0, (1e-8, 1.0, 128)),
    (O.ANTIREFLECTIVE, gauss(7, 2.0), 4096, 2, 1, (1e-8, 1.0, 128)),
]


@pytest.mark.parametrize("bc,psf,n,B,smoother,search", CASES)
def test_deblur_vs_cufft_oracle(cufft_oracle, bc, psf, n, B, smoother, search):
    Oc = cufft_oracle
    op = P.build_operator(psf, n, bc)
    L = P.smoothing_eigenvalues(smoother, op)
    oop = Oc.build_operator(Oc.make_psf(psf, normalize=True), n, bc)
    s = Oc.smoothing_eigenvalues(SM[smoother], bc, n, oop.eigenvalues)
    g = _scenes(n, psf, B, 7 + n + bc, 0.005)
    mu_min, mu_max, K = search
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True), want_curve=True,
                   search=P.GcvSearch(mu_min, mu_max, K))
    want = Oc.deblur(oop, s, g, True, mu_min=mu_min, mu_max=mu_max, count=K, want_curve=True)
    assert np.array_equal(np_(rep.best_k), np.atleast_1d(want.best_k))
    assert np.max(np.abs(np_(rep.mu_used) / want.mu_used - 1)) < 1e-10
    assert rel(np_(rep.restored), want.restored) < 1e-10


def test_deblur_2d_vs_cufft_oracle(cufft_oracle):
    """Config-2 slice: separable Gaussian, hoc-cosine in both directions,
    Laplacian smoother, 128 lambda, on a config-2 scene at 256^2."""
    Oc = cufft_oracle
    n = 256
    h = gauss(12, 2.5)
    op = P.build_operator_2d_separable(h, h, n, n, O.HOC_COSINE)
    L = P.smoothing_eigenvalues("laplacian", op)
    p = Oc.separable_psf2d(Oc.make_psf(h, True), Oc.make_psf(h, True))
    oop = Oc.build_operator_2d(p, n, n, O.HOC_COSINE, separable=True)
    s = Oc.smoothing_eigenvalues_2d(O.LAPLACIAN, O.HOC_COSINE, n, n, oop.eigenvalues)
    _, g = W.image_2d(W.config(2), 0, n, n)
    rep = P.deblur(op, L, torch.from_numpy(g), P.MuChoice(True),
                   search=P.GcvSearch(1e-6, 1.0, 128))
    want = Oc.deblur_2d(oop, s, g, True, mu_min=1e-6, mu_max=1.0, count=128)
    assert int(np_(rep.best_k)) == int(want.best_k)
    assert abs(float(np_(rep.mu_used)) / float(want.mu_used) - 1) < 1e-10
    assert rel(np_(rep.restored), want.restored) < 1e-10
