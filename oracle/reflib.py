"""ctypes binding of oracle/_ref/libfdref.so (the reference compiled from its
own sources by oracle/Makefile, fronted by oracle/ref_capi.cpp).

TEST INFRASTRUCTURE ONLY: used by tests/ (to pin the numpy restatement and the
product against the reference itself), by oracle/gen_golden.py, and by
bench.py's reference arm / cpu_baseline leg.  ``available()`` is False when the
library was not built (e.g. a box that never had /root/reference)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libfdref.so")
LIB_V4_PATH = os.path.join(_HERE, "_ref", "libfdref_v4.so")  # x86-64-v4 (AVX-512) build
_lib = None
_variant = "x86-64-v3"

_dp = C.POINTER(C.c_double)


def available():
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


def prefer_native():
    """Timing legs only (bench.py): switch to the x86-64-v4 build when this
    machine's CPU supports that level (the stand-in for -march=native, see
    oracle/Makefile).  Must be called before the first lib() use; returns the
    -march level in use."""
    global _lib, _variant
    need = {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"}
    try:
        with open("/proc/cpuinfo") as f:
            flags = next((ln.split(":", 1)[1].split() for ln in f if ln.startswith("flags")), [])
    except OSError:
        flags = []
    if _lib is None and os.path.exists(LIB_V4_PATH) and need <= set(flags):
        _lib = C.CDLL(LIB_V4_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _variant = "x86-64-v4"
    return _variant


def variant():
    return _variant


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference status {code}: {msg}")
        self.code = code


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _chk(code):
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def eigenvalues_1d(psf, n, bc):
    psf = _f64(psf)
    re, im = np.empty(n), np.empty(n)
    _chk(lib().ref_eigenvalues_1d(_p(psf), len(psf), n, bc, _p(re), _p(im)))
    return re + 1j * im


def smoother_1d(psf, n, bc, kind):
    psf = _f64(psf)
    s = np.empty(n)
    _chk(lib().ref_smoother_1d(_p(psf), len(psf), n, bc, kind, _p(s)))
    return s


def basis_apply_1d(bc, n, x, analyze=True):
    x = np.asarray(x)
    re, im = _f64(x.real), _f64(np.imag(x))
    ore, oim = np.empty(n), np.empty(n)
    _chk(lib().ref_basis_apply_1d(bc, n, 0 if analyze else 1, _p(re), _p(im), _p(ore), _p(oim)))
    return ore + 1j * oim


def transform_fields(basis, n):
    m = n - 2
    q = np.empty(n)
    alpha = C.c_double()
    bufs = [np.empty(2 * m) for _ in range(6)]
    cap = np.empty(8)
    _chk(lib().ref_transform_fields(basis, n, _p(q), C.byref(alpha), *[_p(b) for b in bufs],
                                    _p(cap)))
    cx = [b[0::2] + 1j * b[1::2] for b in bufs]
    return dict(q=q, alpha=alpha.value, v=cx[0], w=cx[1], row_a=cx[2], row_b=cx[3], c_a=cx[4],
                c_b=cx[5], capacitance=cap[0::2] + 1j * cap[1::2])


def matvec_1d(psf, n, bc, f):
    psf, f = _f64(psf), _f64(f)
    out = np.empty(n)
    res = C.c_double()
    _chk(lib().ref_matvec_1d(_p(psf), len(psf), n, bc, _p(f), _p(out), C.byref(res)))
    return out, res.value


def sweep_mu_1d(psf, n, bc, smoother, g, truth=None, mu_min=1e-12, mu_max=10.0, count=200,
                s_custom=None):
    """sweep_mu (pipeline.cpp:55-115) -> (mus, G, rre, [min_rre, mu_opt, mu_gcv, rre_gcv])."""
    psf, g = _f64(psf), _f64(g)
    t = None if truth is None else _f64(truth)
    sc = None if s_custom is None else _f64(s_custom)
    mus, G, rre, summ = np.empty(count), np.empty(count), np.empty(count), np.empty(4)
    _chk(lib().ref_sweep_mu_1d(_p(psf), len(psf), n, bc, smoother, _p(sc), _p(g), _p(t),
                               C.c_double(mu_min), C.c_double(mu_max), count, _p(mus), _p(G),
                               _p(rre), _p(summ)))
    return mus, G, rre, summ


def gcv_value_1d(psf, n, bc, smoother, g, mu, s_custom=None):
    psf, g = _f64(psf), _f64(g)
    G = C.c_double()
    sc = None if s_custom is None else _f64(s_custom)
    _chk(lib().ref_gcv_value_1d(_p(psf), len(psf), n, bc, smoother, _p(sc), _p(g),
                                C.c_double(mu), C.byref(G)))
    return G.value


def deblur_1d(psf, n, bc, smoother, g, use_gcv=True, fixed_mu=0.0, mu_min=1e-12, mu_max=10.0,
              count=200, threads=1, want_curve=False, s_custom=None):
    """deblur for a [batch, n] array; returns (restored, mu_used, curves, imag_residue)."""
    psf = _f64(psf)
    g = _f64(g).reshape(-1, n)
    B = g.shape[0]
    out = np.empty_like(g)
    mu = np.empty(B)
    res = np.empty(B)
    curve = np.empty((B, count)) if want_curve else None
    sc = None if s_custom is None else _f64(s_custom)
    _chk(lib().ref_deblur_1d(_p(psf), len(psf), n, bc, smoother, _p(sc), int(use_gcv),
                             C.c_double(fixed_mu), C.c_double(mu_min), C.c_double(mu_max),
                             count, C.c_long(B), _p(g), _p(out), _p(mu), _p(curve), _p(res),
                             threads))
    return out, mu, curve, res


_GCV_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)


def gcv_minimize(G, mu_min, mu_max, count):
    """Reference gcv_minimize driven by a Python callable -> (mu, grid values)."""
    cb = _GCV_FN(lambda mu, ctx: float(G(mu)))
    mu = C.c_double()
    curve = np.empty(count)
    _chk(lib().ref_gcv_minimize(cb, None, C.c_double(mu_min), C.c_double(mu_max), count,
                                C.byref(mu), _p(curve)))
    return mu.value, curve


def add_noise(g, level, seed):
    g = _f64(g)
    out = np.empty_like(g)
    _chk(lib().ref_add_noise(_p(g), C.c_long(g.size), C.c_double(level), C.c_ulonglong(seed),
                             _p(out)))
    return out


def convolve_valid(ext, psf):
    ext, psf = _f64(ext), _f64(psf)
    out = np.empty(ext.size - (len(psf) - 1))
    _chk(lib().ref_convolve_valid(_p(ext), C.c_long(ext.size), _p(psf), len(psf), _p(out)))
    return out


def convolve_valid_2d(ext, psf2):
    """convolve_valid_2d (pipeline.cpp:31-51); the shim normalises the mask
    (make_psf2d(..., normalize=true)), so pass a mask of sum 1."""
    ext, psf2 = _f64(ext), _f64(psf2)
    n1, n2 = ext.shape[0] - (psf2.shape[0] - 1), ext.shape[1] - (psf2.shape[1] - 1)
    out = np.empty((n1, n2))
    _chk(lib().ref_convolve_valid_2d(_p(ext), ext.shape[0], ext.shape[1], _p(psf2),
                                     psf2.shape[0], psf2.shape[1], _p(out)))
    return out


def eigenvalues_2d(psf2, n1, n2, bc, eig_mode=0):
    psf2 = _f64(psf2)
    re, im = np.empty(n1 * n2), np.empty(n1 * n2)
    _chk(lib().ref_eigenvalues_2d(_p(psf2), psf2.shape[0], psf2.shape[1], n1, n2, bc, eig_mode,
                                  _p(re), _p(im)))
    return (re + 1j * im).reshape(n1, n2)


def tensor_apply(bc, x, analyze=True):
    x = np.asarray(x)
    n1, n2 = x.shape
    re, im = _f64(x.real), _f64(np.imag(x))
    ore, oim = np.empty((n1, n2)), np.empty((n1, n2))
    _chk(lib().ref_tensor_apply(bc, n1, n2, 0 if analyze else 1, _p(re), _p(im), _p(ore),
                                _p(oim)))
    return ore + 1j * oim


def matvec_2d(psf2, bc, f, eig_mode=0):
    psf2, f = _f64(psf2), _f64(f)
    n1, n2 = f.shape
    out = np.empty_like(f)
    res = C.c_double()
    _chk(lib().ref_matvec_2d(_p(psf2), psf2.shape[0], psf2.shape[1], n1, n2, bc, eig_mode,
                             _p(f), _p(out), C.byref(res)))
    return out, res.value


def deblur_2d(psf2, bc, smoother, g, use_gcv=True, fixed_mu=0.0, mu_min=1e-12, mu_max=10.0,
              count=200, eig_mode=0, threads=1, want_curve=False, s_custom=None):
    psf2 = _f64(psf2)
    g = _f64(g)
    n1, n2 = g.shape[-2:]
    g = g.reshape(-1, n1, n2)
    B = g.shape[0]
    out = np.empty_like(g)
    mu = np.empty(B)
    res = np.empty(B)
    curve = np.empty((B, count)) if want_curve else None
    sc = None if s_custom is None else _f64(s_custom)
    _chk(lib().ref_deblur_2d(_p(psf2), psf2.shape[0], psf2.shape[1], n1, n2, bc, eig_mode,
                             smoother, _p(sc), int(use_gcv), C.c_double(fixed_mu),
                             C.c_double(mu_min), C.c_double(mu_max), count, C.c_long(B), _p(g),
                             _p(out), _p(mu), _p(curve), _p(res), threads))
    return out, mu, curve, res
