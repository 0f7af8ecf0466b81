"""Generate tests/golden/*.npz by running the REFERENCE itself (oracle/_ref,
compiled from /root/reference by oracle/Makefile) on seeded inputs.

TEST INFRASTRUCTURE ONLY.  Run here (where /root/reference exists):
    make -C oracle && python oracle/gen_golden.py
The fixtures are committed; the GPU box only reads them.

Contents (all inputs stored with the outputs, so tests never depend on
re-generating bit-identical inputs):
  golden_1d.npz  config 0 exactly (n=1024 hoc-cosine, Gaussian sigma=3 21 taps,
                 identity smoother, GCV 64 lambda in [1e-6, 1]); a config-1
                 slice (4 signals of n=4096, one-sided exp(-k/5) 15 taps,
                 hoc-fourier = the reference's d=2 for nonsymmetric PSFs,
                 first-difference smoother fed as custom eigenvalues, GCV 256
                 lambda in [1e-8, 1]); per-BC analyze / synthesize / matvec /
                 eigenvalues at n = 6, 33, 64.
  golden_2d.npz  a config-2 slice (256^2 hoc-cosine, Gaussian sigma=2.5 25x25
                 separable, Laplacian, 128 lambda in [1e-6,1]); a config-3
                 slice (2 images 96^2, hoc-fourier, one-sided exp(-k/4) 11x11,
                 identity + Laplacian, 128 lambda); a non-separable disk PSF at
                 16x20 through build_operator_2d (three-step eigenvalues).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

import reflib as R  # noqa: E402
from paper_0906_2704_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def first_difference_s(bc, n):
    i = np.arange(n)
    x = np.zeros(n)
    if bc == W.HOC_FOURIER:
        x[1:n - 1] = 2.0 * np.pi * (i[1:n - 1] - 1) / (n - 2)
    elif bc == W.HOC_COSINE:
        x[1:n - 1] = np.pi * (i[1:n - 1] - 1) / (n - 2)
    return np.sqrt(2.0 - 2.0 * np.cos(x))


def gen_1d():
    out = {}
    # ---- config 0, exactly as BASELINE.json states it ----
    c0 = W.config(0)
    truth, g = W.signals_1d(c0, 0, 1)
    rest, mu, curve, res = R.deblur_1d(c0.psf, c0.n1, c0.bc, 0, g, True, mu_min=c0.mu_min,
                                       mu_max=c0.mu_max, count=c0.count, want_curve=True)
    out.update(c0_psf=c0.psf, c0_truth=truth, c0_g=g, c0_restored=rest, c0_mu=mu,
               c0_curve=curve, c0_ghat=R.basis_apply_1d(c0.bc, c0.n1, g[0], True).real)
    # ---- config 1 slice ----
    c1 = W.config(1)
    truth, g = W.signals_1d(c1, 0, 4)
    s = first_difference_s(c1.bc, c1.n1)
    rest, mu, curve, res = R.deblur_1d(c1.psf, c1.n1, c1.bc, 2, g, True, mu_min=c1.mu_min,
                                       mu_max=c1.mu_max, count=c1.count, want_curve=True,
                                       s_custom=s)
    out.update(c1_psf=c1.psf, c1_g=g, c1_s=s, c1_restored=rest, c1_mu=mu, c1_curve=curve,
               c1_imag_residue=res)
    # ---- per-BC transform / operator pins ----
    rng = np.random.default_rng(777)
    sym = W.gaussian_weights(1, 1.0)
    gen = W.onesided_exp_weights(2, 0.5)
    for bc in range(5):
        for n in (6, 33, 64):
            psf = gen if bc in (0, 4) else sym
            x = rng.uniform(-1, 1, n)
            c = rng.uniform(-1, 1, n) + (1j * rng.uniform(-1, 1, n) if bc in (0, 4) else 0)
            f = rng.uniform(-1, 1, n)
            key = f"bc{bc}_n{n}"
            out[key + "_psf"] = psf
            out[key + "_x"] = x
            out[key + "_analyze"] = R.basis_apply_1d(bc, n, x, True)
            out[key + "_c"] = c
            out[key + "_synth"] = R.basis_apply_1d(bc, n, c, False)
            out[key + "_eig"] = R.eigenvalues_1d(psf, n, bc)
            out[key + "_f"] = f
            out[key + "_matvec"] = R.matvec_1d(psf, n, bc, f)[0]
    np.savez_compressed(os.path.join(OUT, "golden_1d.npz"), **out)


def gen_2d():
    out = {}
    c2 = W.config(2)
    truth, g = W.image_2d(c2, 0, 256, 256)
    psf2 = c2.psf2d()
    rest, mu, curve, res = R.deblur_2d(psf2, c2.bc, 1, g, True, mu_min=c2.mu_min,
                                       mu_max=c2.mu_max, count=c2.count, eig_mode=1,
                                       want_curve=True)
    out.update(c2_psf=c2.psf, c2_truth=truth, c2_g=g, c2_restored=rest, c2_mu=mu,
               c2_curve=curve)
    c3 = W.config(3)
    imgs = np.stack([W.image_2d(c3, i, 96, 96)[1] for i in range(2)])
    psf3 = c3.psf2d()
    out.update(c3_psf=c3.psf, c3_g=imgs)
    for sm, name in ((0, "identity"), (1, "laplacian")):
        rest, mu, curve, res = R.deblur_2d(psf3, c3.bc, sm, imgs, True, mu_min=c3.mu_min,
                                           mu_max=c3.mu_max, count=c3.count, eig_mode=1,
                                           want_curve=True)
        out.update({f"c3_{name}_restored": rest, f"c3_{name}_mu": mu,
                    f"c3_{name}_curve": curve, f"c3_{name}_imag_residue": res})
    j = np.arange(-3, 4)
    disk = (j[:, None] ** 2 + j[None, :] ** 2 <= 9).astype(float)
    rng = np.random.default_rng(31)
    f = rng.uniform(0, 1, (16, 20))
    out.update(disk_psf=disk, disk_f=f,
               disk_eig=R.eigenvalues_2d(disk, 16, 20, W.HOC_COSINE, 0),
               disk_matvec=R.matvec_2d(disk, W.HOC_COSINE, f, 0)[0])
    rest, mu, curve, res = R.deblur_2d(disk, W.HOC_COSINE, 1, f, True, mu_min=1e-6, mu_max=1.0,
                                       count=32, eig_mode=0, want_curve=True)
    out.update(disk_restored=rest, disk_mu=mu, disk_curve=curve)
    np.savez_compressed(os.path.join(OUT, "golden_2d.npz"), **out)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    gen_1d()
    gen_2d()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
