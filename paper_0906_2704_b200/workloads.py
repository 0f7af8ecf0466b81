"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference publishes no data; these generators stand in for the
paper's unpublished test signals with the shapes, sizes and value
distributions BASELINE.json names.  Generation follows the reference's
"true-extended" observation model: the scene is sampled on the extended grid
(n + 2m per axis, t = (i - m)/n as in acceptance_main.cpp:387-398), blurred
with ``convolve_valid`` (g_i = sum_j h_j f_{i+j}, pipeline.cpp:15-51) and
perturbed with the reference's ``add_noise`` (SplitMix64 + Box-Muller,
rescaled so ||eta|| = level ||g||, operators.cpp:332-358).

Random parameters come from a counter-based SplitMix64 keyed by
(config, item, draw), so every item is reproducible independently of batch
size or order.  Builder-defined details (documented in DESIGN.md):
  * 1D: cubic coefficients U[-1,1]; 3 bumps a*exp(-((t-c)/w)^2) with
    a ~ U[0.2,1], w ~ U[0.02,0.08], c ~ U[0,1]; a unit step at U[0,1].
  * 2D: quadratic trend with coefficients U[-0.5,0.5] plus 0.5; blobs
    a*exp(-|x-c|^2/w^2), a ~ +-U[0.1,0.6], w ~ U[0.01,0.08], c ~ U[0,1]^2,
    evaluated on their +-6w bounding box; rectangles with corner U[0,1]^2,
    sides U[0.05,0.3], value U[0,1] replacing the region; clip to [0,1].
This module is host-side data preparation only (not timed, not the product's
compute path).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PERIODIC, REFLECTIVE, ANTIREFLECTIVE, HOC_COSINE, HOC_FOURIER = range(5)
HOC_FOURIER_D1, HOC_FOURIER_D3 = 5, 6  # extension codes (include/fastdeblur_b200.h)
IDENTITY, LAPLACIAN, FIRST_DIFFERENCE = range(3)

_GOLD = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x):
    """operators.cpp:78-85."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def bits_to_u01(bits):
    """(0, 1], operators.cpp:88-90."""
    return ((np.asarray(bits, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) + 1.0) \
        * (2.0 ** -53)


def item_key(cfg, item):
    item = np.asarray(item, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return splitmix64((np.uint64(cfg) << np.uint64(40)) + item)


def draw(key, k):
    """k-th uniform (0,1] draw of the stream ``key`` (vectorised over key)."""
    with np.errstate(over="ignore"):
        return bits_to_u01(splitmix64(np.asarray(key, np.uint64) +
                                      np.uint64(k + 1) * _GOLD))


def add_noise(g, level, seed):
    """Reference add_noise (operators.cpp:332-358) over the last axis; ``seed``
    broadcasts against the leading axes."""
    g = np.asarray(g, dtype=np.float64)
    if level == 0.0:
        return g.copy()
    n = g.shape[-1]
    pairs = (n + 1) // 2
    seed = np.asarray(seed, dtype=np.uint64)[..., None]
    p = np.arange(pairs, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u1 = bits_to_u01(splitmix64(seed + (np.uint64(2) * p + np.uint64(1)) * _GOLD))
        u2 = bits_to_u01(splitmix64(seed + (np.uint64(2) * p + np.uint64(2)) * _GOLD))
    r = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * math.pi * u2
    eta = np.empty(np.broadcast_shapes(seed.shape[:-1], g.shape[:-1]) + (2 * pairs,))
    eta[..., 0::2] = r * np.cos(ang)
    eta[..., 1::2] = r * np.sin(ang)
    eta = eta[..., :n]
    gn = np.sum(g * g, axis=-1, keepdims=True)
    en = np.sum(eta * eta, axis=-1, keepdims=True)
    return g + level * np.sqrt(gn / en) * eta


def convolve_valid(ext, w):
    """g_i = sum_j h_j f_{i+j} over the last axis (pipeline.cpp:15-29)."""
    m = (len(w) - 1) // 2
    n = ext.shape[-1] - 2 * m
    g = np.zeros(ext.shape[:-1] + (n,))
    for j in range(-m, m + 1):
        if w[m + j] != 0.0:
            g += w[m + j] * ext[..., m + j:m + j + n]
    return g


def gaussian_weights(m, sigma):
    """psf.cpp:62-69 (normalised by the serial sum)."""
    j = np.arange(-m, m + 1, dtype=np.float64)
    w = np.exp(-j * j / (2.0 * sigma * sigma))
    s = 0.0
    for x in w:
        s += float(x)
    return w / s


def onesided_exp_weights(taps, rate):
    """Centred mask of half-width taps-1 with h_k ∝ exp(-rate k), k = 0..taps-1,
    zero for k < 0 (BASELINE configs 1 and 3)."""
    m = taps - 1
    w = np.zeros(2 * m + 1)
    w[m:] = np.exp(-rate * np.arange(taps))
    s = 0.0
    for x in w:
        s += float(x)
    return w / s


@dataclass
class Config:
    index: int
    dim: int
    n1: int
    n2: int
    batch: int
    psf: np.ndarray      # 1D weights (dim 1) or the per-axis 1D factor (dim 2, separable)
    bc: int
    smoothers: tuple
    mu_min: float
    mu_max: float
    count: int
    noise: float
    blobs: int = 0
    rects: int = 0
    note: str = ""
    # boundary conditions a bench step restores with (each with every
    # smoother); () = (bc,).  ``bc`` stays the reference-supported BC (the
    # reference arm and the golden fixtures use it).
    bcs: tuple = ()
    # storage precisions a step restores in ("f64", and "f32" = the fp32
    # storage variant, fp64 arithmetic)
    precisions: tuple = ("f64",)

    @property
    def step_bcs(self):
        return self.bcs or (self.bc,)

    @property
    def pixels(self):
        return self.batch * self.n1 * (self.n2 if self.dim == 2 else 1)

    def psf2d(self):
        return np.outer(self.psf, self.psf) / float(np.sum(np.outer(self.psf, self.psf)))


def config(index: int) -> Config:
    """BASELINE.json configs.  Reference-unsupported features are mapped to the
    nearest supported BC; DESIGN.md states each mapping."""
    if index == 0:
        return Config(0, 1, 1024, 1, 1, gaussian_weights(10, 3.0), HOC_COSINE, (IDENTITY,),
                      1e-6, 1.0, 64, 0.01)
    if index == 1:
        return Config(1, 1, 4096, 1, 65536, onesided_exp_weights(15, 1 / 5), HOC_FOURIER,
                      (FIRST_DIFFERENCE,), 1e-8, 1.0, 256, 0.005,
                      bcs=(HOC_FOURIER_D1, HOC_FOURIER_D3),
                      note="d=1 and d=3 with a nonsymmetric PSF are extensions (not in the "
                           "reference): a step restores the batch at both degrees; the "
                           "reference arm runs its nearest BC, hoc-fourier (d=2)")
    if index == 2:
        return Config(2, 2, 4096, 4096, 1, gaussian_weights(12, 2.5), HOC_COSINE, (LAPLACIAN,),
                      1e-6, 1.0, 128, 0.01, blobs=40, rects=10)
    if index == 3:
        return Config(3, 2, 1024, 1024, 512, onesided_exp_weights(11, 1 / 4), HOC_FOURIER,
                      (IDENTITY, LAPLACIAN), 1e-6, 1.0, 128, 0.01, blobs=40, rects=10,
                      bcs=(HOC_FOURIER_D3,), precisions=("f64", "f32"),
                      note="d=3 is an extension (not in the reference): a step restores the "
                           "batch with the identity and the Laplacian smoother, from fp64 and "
                           "from fp32 storage (fp64 arithmetic in both); the reference "
                           "arm runs its nearest BC, hoc-fourier (d=2); lambda range "
                           "unspecified, [1e-6, 1] used")
    if index == 4:
        return Config(4, 2, 16384, 16384, 1, gaussian_weights(16, 4.0), HOC_COSINE,
                      (LAPLACIAN,), 1e-8, 1.0, 512, 0.01, blobs=80, rects=20)
    raise ValueError(index)


def signals_1d(cfg: Config, first: int, count: int, n: int | None = None,
               m: int | None = None):
    """(truth, observed) for items [first, first+count) of a 1D config."""
    n = cfg.n1 if n is None else n
    m = (len(cfg.psf) - 1) // 2 if m is None else m
    items = np.arange(first, first + count, dtype=np.uint64)
    key = item_key(cfg.index, items)[:, None]
    t = (np.arange(n + 2 * m, dtype=np.float64) - m) / n
    u = [draw(key, k) for k in range(4 + 9 + 1)]
    c = [2.0 * u[k] - 1.0 for k in range(4)]
    f = c[0] + t * (c[1] + t * (c[2] + t * c[3]))
    for j in range(3):
        amp = 0.2 + 0.8 * u[4 + 3 * j]
        width = 0.02 + 0.06 * u[5 + 3 * j]
        cen = u[6 + 3 * j]
        f = f + amp * np.exp(-((t - cen) / width) ** 2)
    f = f + (t >= u[13]).astype(np.float64)
    truth = f[:, m:m + n]
    g = convolve_valid(f, cfg.psf)
    return truth, add_noise(g, cfg.noise, key[:, 0])


def _scene_2d(cfg: Config, item: int, n1: int, n2: int, m1: int, m2: int,
              r0: int = 0, r1: int | None = None):
    """Extended scene (n1+2m1) x (n2+2m2); rows [r0, r1) of it when given (every
    value is elementwise, so a row band equals the same rows of the whole)."""
    key = item_key(cfg.index, np.uint64(item))
    k = iter(range(10_000))
    y = (np.arange(n1 + 2 * m1, dtype=np.float64) - m1) / n1
    x = (np.arange(n2 + 2 * m2, dtype=np.float64) - m2) / n2
    r1 = len(y) if r1 is None else r1
    yy = y[r0:r1]
    a = [float(draw(key, next(k))) - 0.5 for _ in range(6)]
    f = 0.5 + a[0] + a[1] * yy[:, None] + a[2] * x[None, :] + a[3] * (yy * yy)[:, None] + \
        a[4] * yy[:, None] * x[None, :] + a[5] * (x * x)[None, :]
    for _ in range(cfg.blobs):
        amp = (0.1 + 0.5 * float(draw(key, next(k)))) * \
            (1.0 if float(draw(key, next(k))) < 0.5 else -1.0)
        w = 0.01 + 0.07 * float(draw(key, next(k)))
        cy, cx = float(draw(key, next(k))), float(draw(key, next(k)))
        i0 = max(r0, int(math.floor((cy - 6 * w) * n1)) + m1)
        i1 = min(r1, int(math.ceil((cy + 6 * w) * n1)) + m1 + 1)
        j0 = max(0, int(math.floor((cx - 6 * w) * n2)) + m2)
        j1 = min(len(x), int(math.ceil((cx + 6 * w) * n2)) + m2 + 1)
        if i0 < i1 and j0 < j1:
            dy = (y[i0:i1] - cy) ** 2
            dx = (x[j0:j1] - cx) ** 2
            f[i0 - r0:i1 - r0, j0:j1] += amp * np.exp(-(dy[:, None] + dx[None, :]) / (w * w))
    for _ in range(cfg.rects):
        rr, c0 = float(draw(key, next(k))), float(draw(key, next(k)))
        hr = 0.05 + 0.25 * float(draw(key, next(k)))
        hc = 0.05 + 0.25 * float(draw(key, next(k)))
        val = float(draw(key, next(k)))
        sel_y = (yy >= rr) & (yy < rr + hr)
        sel_x = (x >= c0) & (x < c0 + hc)
        f[np.ix_(sel_y, sel_x)] = val
    np.clip(f, 0.0, 1.0, out=f)
    return key, f


def image_2d(cfg: Config, item: int, n1: int | None = None, n2: int | None = None,
             psf: np.ndarray | None = None):
    """(truth, observed) for image ``item`` of a 2D config (separable blur)."""
    n1 = cfg.n1 if n1 is None else n1
    n2 = cfg.n2 if n2 is None else n2
    w = cfg.psf if psf is None else psf
    m = (len(w) - 1) // 2
    key, f = _scene_2d(cfg, item, n1, n2, m, m)
    truth = f[m:m + n1, m:m + n2].copy()
    # separable valid convolution: rows then columns (equals the 2D mask sum
    # for the outer-product mask up to rounding)
    g = convolve_valid(f, w)
    g = convolve_valid(np.ascontiguousarray(g.T), w).T
    obs = add_noise(np.ascontiguousarray(g).reshape(-1), cfg.noise, key).reshape(n1, n2)
    return truth, obs


# ---------------------------------------------------------------------------
# Large images (config 4, 16384^2): the same scene / blur / noise, generated in
# fixed bands of SLAB rows by worker processes into shared memory.  Band
# boundaries do not depend on the worker count, so the image is deterministic;
# the noise norm is the band partial sums added in band order.
SLAB = 256


def _noise_band(key, e0, e1):
    """Gaussian field of add_noise for flat positions [e0, e1) of the image."""
    p = np.arange(e0 // 2, (e1 + 1) // 2, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u1 = bits_to_u01(splitmix64(np.uint64(key) + (np.uint64(2) * p + np.uint64(1)) * _GOLD))
        u2 = bits_to_u01(splitmix64(np.uint64(key) + (np.uint64(2) * p + np.uint64(2)) * _GOLD))
    r = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * math.pi * u2
    eta = np.empty(2 * len(p))
    eta[0::2] = r * np.cos(ang)
    eta[1::2] = r * np.sin(ang)
    s = e0 - 2 * (e0 // 2)
    return eta[s:s + (e1 - e0)]


def _band_job(args):
    from multiprocessing import shared_memory
    phase, ci, item, n1, n2, b0, b1, name, scale, r0, rows = args
    cfg = config(ci)
    w = cfg.psf
    m = (len(w) - 1) // 2
    shm = shared_memory.SharedMemory(name=name)
    try:
        # the shared buffer holds image rows [r0, r0 + rows)
        out = np.ndarray((rows, n2), dtype=np.float64, buffer=shm.buf)
        key = item_key(ci, np.uint64(item))
        if phase == 0:
            _, f = _scene_2d(cfg, item, n1, n2, m, m, b0, b1 + 2 * m)
            g = convolve_valid(f, w)                 # rows
            h = np.zeros((b1 - b0, n2))
            for j in range(-m, m + 1):               # columns, same term order
                if w[m + j] != 0.0:
                    h += w[m + j] * g[m + j:m + j + (b1 - b0)]
            out[b0 - r0:b1 - r0] = h
            eta = _noise_band(key, b0 * n2, b1 * n2)
            return float(np.sum(h * h)), float(np.sum(eta * eta))
        eta = _noise_band(key, b0 * n2, b1 * n2).reshape(b1 - b0, n2)
        out[b0 - r0:b1 - r0] += scale * eta
        return 0.0, 0.0
    finally:
        shm.close()


def image_2d_large(ci: int, item: int, workers: int | None = None, n1: int | None = None,
                   n2: int | None = None) -> np.ndarray:
    """Observed image ``item`` of 2D config ``ci`` built band-parallel (the
    scene, separable valid blur and add_noise of image_2d)."""
    cfg = config(ci)
    n1 = cfg.n1 if n1 is None else n1
    return image_2d_rows(ci, item, 0, n1, workers, n1, n2)


def image_2d_rows(ci: int, item: int, r0: int, r1: int, workers: int | None = None,
                  n1: int | None = None, n2: int | None = None, reduce=None) -> np.ndarray:
    """Rows [r0, r1) of image_2d_large (r0 a multiple of SLAB).  ``reduce`` sums
    the noise-norm partials over the other holders of the image (the ranks of a
    row-slab split); the whole-image norm is their sum."""
    import os
    from concurrent.futures import ProcessPoolExecutor
    from multiprocessing import shared_memory
    cfg = config(ci)
    n1 = cfg.n1 if n1 is None else n1
    n2 = cfg.n2 if n2 is None else n2
    if r0 % SLAB:
        raise ValueError("row ranges start on band boundaries")
    rows = r1 - r0
    shm = shared_memory.SharedMemory(create=True, size=max(rows, 1) * n2 * 8)
    try:
        bands = [(b, min(b + SLAB, r1)) for b in range(r0, r1, SLAB)]
        workers = workers or os.cpu_count() or 1
        with ProcessPoolExecutor(workers) as ex:
            parts = list(ex.map(_band_job, [(0, ci, item, n1, n2, b0, b1, shm.name, 0.0, r0, rows)
                                           for b0, b1 in bands]))
            sums = np.array([sum(p[0] for p in parts), sum(p[1] for p in parts)])
            if reduce is not None:
                sums = np.asarray(reduce(sums), dtype=np.float64)
            scale = cfg.noise * math.sqrt(sums[0] / sums[1])
            list(ex.map(_band_job, [(1, ci, item, n1, n2, b0, b1, shm.name, scale, r0, rows)
                                    for b0, b1 in bands]))
        return np.array(np.ndarray((rows, n2), dtype=np.float64, buffer=shm.buf))
    finally:
        shm.close()
        shm.unlink()
