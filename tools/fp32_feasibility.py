"""Would an fp32-ARITHMETIC transform path meet north_star's 1e-4 bar on config 3?

CPU experiment with the numpy oracle (oracle/fdoracle.py HoTransform, d = 3,
separable one-sided motion blur, 1 % noise, 128 lambda in [1e-6, 1]): the
restoration with every interior DFT evaluated in complex64 (input rounded to
fp32, fp32 FFT, fp32 output) -- border amplitudes, polynomial fold, filter and
GCV sums kept in fp64, i.e. the most favourable split -- against the all-fp64
restoration of the same fp32-rounded image.

    python tools/fp32_feasibility.py [n]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import fdoracle as O  # noqa: E402
from paper_0906_2704_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cfg = W.config(3)
bc = W.HOC_FOURIER_D3
_, g = W.image_2d(cfg, 0, n, n)
g = g.astype(np.float32).astype(np.float64)
psf = O.make_psf(cfg.psf, True)
oop = O.build_operator_2d(O.separable_psf2d(psf, psf), n, n, bc, separable=True)
for sm, name in ((O.IDENTITY, "identity"), (O.LAPLACIAN, "laplacian")):
    s = O.smoothing_eigenvalues_2d(sm, bc, n, n, oop.eigenvalues)
    ref = O.deblur_2d(oop, s, g[None], True, mu_min=cfg.mu_min, mu_max=cfg.mu_max, count=cfg.count)
    orig = O.fourier_apply

    def fourier32(v, forward=True):
        v = np.asarray(v, dtype=np.complex128).astype(np.complex64)
        m = v.shape[-1]
        y = np.fft.fft(v, axis=-1) if forward else np.fft.ifft(v, axis=-1) * m
        return (y.astype(np.complex64) * np.float32(1.0 / np.sqrt(m))).astype(np.complex128)

    O.fourier_apply = fourier32
    try:
        lo = O.deblur_2d(oop, s, g[None], True, mu_min=cfg.mu_min, mu_max=cfg.mu_max,
                         count=cfg.count)
    finally:
        O.fourier_apply = orig
    err = np.linalg.norm(lo.restored - ref.restored) / np.linalg.norm(ref.restored)
    print(f"n={n} {name}: best_k fp64 {ref.best_k[0]} fp32-FFT {lo.best_k[0]}, mu {ref.mu_used[0]:.3e} / "
          f"{lo.mu_used[0]:.3e}, restoration rel err {err:.2e} (bar 1e-4)")
