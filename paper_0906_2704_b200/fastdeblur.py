"""Python mirror of the reference operator API over the sm_100a C ABI.

The names, argument meaning and error behaviour follow the reference C++ API
(namespace ``fastdeblur``; see include/fastdeblur_b200.h for the file:line of
each function).  Arrays are torch CUDA tensors (float64 / complex128), batched
over leading axes: a 1D operator accepts ``[..., n]``, a 2D operator
``[..., n1, n2]``.  Every computation runs in libfdb200.so on the GPU; there
is no CPU path, and a missing library or device raises immediately.

    op = build_operator(psf, n, "hoc-cosine")
    L = smoothing_eigenvalues("laplacian", op)
    rep = deblur(op, L, g, MuChoice(use_gcv=True), search=GcvSearch(1e-6, 1, 64))
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FASTDEBLUR_LIB: an alternative in-tree build (e.g. the phase-timing variant)
LIB_PATH = os.environ.get("FASTDEBLUR_LIB") or os.path.join(_HERE, "libfdb200.so")

BC = {"periodic": 0, "reflective": 1, "antireflective": 2, "hoc-cosine": 3, "hoc-fourier": 4,
      # extensions (not in the reference): higher-order Fourier borders, degree 1 and 3
      "hoc-fourier-d1": 5, "hoc-fourier-d3": 6}
BC_NAMES = {v: k for k, v in BC.items()}
SMOOTHER = {"identity": 0, "laplacian": 1, "first-difference": 2}


class FastDeblurError(RuntimeError):
    """Base class (errors.hpp:10-13); status 1."""


class ValidationError(FastDeblurError, ValueError):
    """errors.hpp:16-19; status 2."""


class DegenerateError(FastDeblurError, ArithmeticError):
    """errors.hpp:38-41; status 3."""


_lib = None


def lib():
    """Load libfdb200.so (fails loudly when the CUDA library was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FastDeblurError(f"{LIB_PATH} missing: run paper_0906_2704_b200.build")
        L = C.CDLL(LIB_PATH)
        L.fd_last_error.restype = C.c_char_p
        L.fd_kernel_launches.restype = C.c_longlong
        vp, dp, ip, ll = C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_longlong
        L.fd_op_create_1d.argtypes = [dp, ip, ip, ip, ip, C.POINTER(vp)]
        L.fd_op_create_2d.argtypes = [dp, ip, ip, ip, ip, ip, ip, C.POINTER(vp)]
        L.fd_op_create_2d_separable.argtypes = [dp, ip, dp, ip, ip, ip, ip, ip, C.POINTER(vp)]
        L.fd_op_destroy.argtypes = [vp]
        cd = C.c_double
        L.fd_sweep_mu.argtypes = [vp, vp, vp, vp, cd, cd, ip, dp, dp, dp, dp, vp]
        L.fd_slab_analyze.argtypes = [vp, ip, vp, ip, vp, ll, vp]
        L.fd_slab_synthesize.argtypes = [vp, vp, ip, vp, vp, ip, ll, ll, cd, vp]
        L.fd_slab_gcv_partials.argtypes = [vp, vp, vp, ll, ll, cd, cd, ip, dp, dp, vp]
        L.fd_slab_gcv_moments.argtypes = [vp, vp, vp, ll, ll, cd, ip, dp, vp]
        L.fd_gcv_moment_terms.argtypes = [cd, cd, ip, C.POINTER(C.c_int)]
        L.fd_gcv_pick_from_sums.argtypes = [dp, cd, cd, ip, dp, C.POINTER(C.c_int),
                                            C.POINTER(C.c_int), dp, dp]
        L.fd_gcv_golden_from_moments.argtypes = [dp, ip, cd, cd, cd, cd, ip, ip, dp]
        L.fd_op_info.argtypes = [vp] + [C.POINTER(C.c_int)] * 5
        L.fd_op_eigenvalues.argtypes = [vp, vp, vp]
        L.fd_smoother_create.argtypes = [vp, ip, C.POINTER(vp)]
        L.fd_smoother_create_custom.argtypes = [vp, dp, C.POINTER(vp)]
        L.fd_smoother_destroy.argtypes = [vp]
        L.fd_smoother_eigenvalues.argtypes = [vp, vp, vp]
        L.fd_analyze.argtypes = [vp, vp, ip, vp, ll, vp]
        L.fd_synthesize.argtypes = [vp, vp, vp, ip, vp, ll, vp]
        L.fd_matvec.argtypes = [vp, vp, vp, vp, ll, vp]
        L.fd_tikhonov.argtypes = [vp, vp, vp, vp, vp, vp, ll, vp]
        L.fd_gcv_value.argtypes = [vp, vp, vp, C.c_double, vp, ll, vp]
        L.fd_gcv_select.argtypes = [vp, vp, vp, C.c_double, C.c_double, ip, vp, vp, vp, ll, vp]
        L.fd_deblur.argtypes = [vp, vp, vp, ip, C.c_double, C.c_double, C.c_double, ip, vp, vp,
                                vp, vp, vp, ll, vp]
        L.fd_deblur_host.argtypes = [vp, vp, vp, ip, C.c_double, C.c_double, C.c_double, ip,
                                     vp, vp, vp, ll, ll, vp]
        L.fd_deblur_f32.argtypes = L.fd_deblur.argtypes
        L.fd_deblur_host_f32.argtypes = L.fd_deblur_host.argtypes
        L.fd_deblur_host_multi.argtypes = [ip, vp, vp, vp, ip, ip, C.c_double, C.c_double,
                                           C.c_double, ip, vp, vp, vp, ll, ll, vp]
        L.fd_matvec_f32.argtypes = L.fd_matvec.argtypes
        L.fd_bc_for_degree.argtypes = [ip, ip, C.POINTER(C.c_int)]
        L.fd_parse_bc.argtypes = [C.c_char_p]
        L.fd_deblur_smoothers.argtypes = [vp, ip, vp, vp, ip, ip, cd, cd, cd, ip, vp, vp, vp, ll, vp]
        L.fd_convolve_valid.argtypes = [vp, ll, ip, dp, ip, vp, vp]
        L.fd_convolve_valid_2d.argtypes = [vp, ll, ip, ip, dp, ip, ip, vp, vp]
        L.fd_add_noise.argtypes = [vp, ll, ll, cd, C.POINTER(C.c_ulonglong), vp]
        _lib = L
    return _lib


def check(code):
    if code == 0:
        return
    msg = lib().fd_last_error().decode()
    if code == 2:
        raise ValidationError(msg)
    if code == 3:
        raise DegenerateError(msg)
    raise FastDeblurError(msg)


def kernel_launches():
    return int(lib().fd_kernel_launches())


def _bc(bc):
    if isinstance(bc, str):
        if bc not in BC:
            raise ValidationError(f"unknown boundary condition {bc!r}")
        return BC[bc]
    return int(bc)


def _host(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _dev(x, dtype=torch.float64):
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(np.asarray(x))
    if x.dtype != dtype:
        x = x.to(dtype)
    return x.to("cuda").contiguous()


def bc_for_degree(degree, psf_symmetric):
    """north_star 'BC degree d' -> the reference BC (d=1 AR, d=2 hoc-*)."""
    out = C.c_int()
    check(lib().fd_bc_for_degree(int(degree), int(bool(psf_symmetric)), C.byref(out)))
    return BC_NAMES[out.value]


# ---------------------------------------------------------------------------
# operators
# ---------------------------------------------------------------------------
class BlurOperator:
    """BlurOperatorT / BlurOperator2DT (operators.hpp:70-83, multidim.hpp:62-73)."""

    def __init__(self, handle, dim, n1, n2, bc, complex_basis):
        self._h = handle
        self.dim, self.n1, self.n2 = dim, n1, n2
        self.bc = bc
        self.complex = bool(complex_basis)

    @property
    def n(self):
        return self.n1

    @property
    def shape(self):
        return (self.n1,) if self.dim == 1 else (self.n1, self.n2)

    @property
    def size(self):
        return self.n1 * (self.n2 if self.dim == 2 else 1)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:
            _lib.fd_op_destroy(h)

    def _count(self, x):
        shp = tuple(x.shape)
        k = len(self.shape)
        if shp[len(shp) - k:] != self.shape:
            raise ValidationError(f"array shape {shp} does not end with {self.shape}")
        return int(np.prod(shp[:len(shp) - k])) if len(shp) > k else 1, shp[:len(shp) - k]

    def eigenvalues(self):
        """operator_eigenvalues / eigenvalues_2d -> complex128 tensor of the op shape."""
        out = torch.empty(self.shape, dtype=torch.complex128, device="cuda")
        check(lib().fd_op_eigenvalues(self._h, _ptr(out), _stream()))
        return out

    def analyze(self, y):
        """SpectralBasis::analyze / tensor_apply(inverse): T_X^{-1} y."""
        cplx_in = torch.is_complex(y) if isinstance(y, torch.Tensor) else np.iscomplexobj(y)
        y = _dev(y, torch.complex128 if cplx_in else torch.float64)
        count, lead = self._count(y)
        out = torch.empty(y.shape, dtype=torch.complex128 if self.complex else torch.float64,
                          device="cuda")
        check(lib().fd_analyze(self._h, _ptr(y), int(cplx_in), _ptr(out), count, _stream()))
        return out

    def synthesize(self, c, complex_out=None):
        """SpectralBasis::synthesize / tensor_apply(forward): T_X c.

        Complex bases return a complex tensor by default; complex_out=False keeps
        the real part and returns (real, imag_residue)."""
        c = _dev(c, torch.complex128 if self.complex else torch.float64)
        count, lead = self._count(c)
        if complex_out is None:
            complex_out = self.complex
        out = torch.empty(c.shape, dtype=torch.complex128 if complex_out else torch.float64,
                          device="cuda")
        res = None if complex_out else torch.zeros(lead, dtype=torch.float64, device="cuda")
        check(lib().fd_synthesize(self._h, _ptr(c), _ptr(out), int(bool(complex_out)),
                                  _ptr(res), count, _stream()))
        return out if complex_out else (out, res)

    def apply(self, f):
        """blur_apply(_2d): (A f, imag_residue).  A float32 f takes the fp32
        storage variant (fd_matvec_f32: fp64 arithmetic, float in / out)."""
        f32 = isinstance(f, torch.Tensor) and f.dtype == torch.float32
        f = _dev(f, torch.float32 if f32 else torch.float64)
        count, lead = self._count(f)
        out = torch.empty_like(f)
        res = torch.zeros(lead, dtype=torch.float64, device="cuda")
        fn = lib().fd_matvec_f32 if f32 else lib().fd_matvec
        check(fn(self._h, _ptr(f), _ptr(out), _ptr(res), count, _stream()))
        return out, res


def _new_op(create, *args):
    h = C.c_void_p()
    check(create(*args, C.byref(h)))
    info = [C.c_int() for _ in range(5)]
    check(lib().fd_op_info(h, *[C.byref(v) for v in info]))
    dim, n1, n2, bc, cx = (v.value for v in info)
    return BlurOperator(h, dim, n1, n2, bc, cx)


def build_operator(psf, n, bc, normalize=True) -> BlurOperator:
    """build_operator(make_psf(psf, normalize), n, bc) (operators.cpp:293-301)."""
    a, p = _host(psf)
    return _new_op(lib().fd_op_create_1d, p, len(a), int(normalize), int(n), _bc(bc))


def build_operator_2d(psf2d, n1, n2, bc, normalize=True) -> BlurOperator:
    """build_operator_2d(make_psf2d(...), n1, n2, bc) (multidim.cpp:309-322)."""
    a, p = _host(psf2d)
    if a.ndim != 2:
        raise ValidationError("2D psf must be a 2D array")
    return _new_op(lib().fd_op_create_2d, p, a.shape[0], a.shape[1], int(normalize), int(n1),
                   int(n2), _bc(bc))


def build_operator_2d_separable(psf_a, psf_b, n1, n2, bc, normalize=True) -> BlurOperator:
    """build_operator_2d(separable_psf2d(a, b), ...) with outer-product eigenvalues."""
    a, pa = _host(psf_a)
    b, pb = _host(psf_b)
    return _new_op(lib().fd_op_create_2d_separable, pa, len(a), pb, len(b), int(normalize),
                   int(n1), int(n2), _bc(bc))


def blur_apply(op: BlurOperator, f):
    return op.apply(f)


class Smoother:
    """SmoothingOperator / SmoothingOperator2D (regularize.hpp:20-23)."""

    def __init__(self, handle, op, kind):
        self._h, self.op, self.kind = handle, op, kind

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:
            _lib.fd_smoother_destroy(h)

    def eigenvalues(self):
        out = torch.empty(self.op.shape, dtype=torch.float64, device="cuda")
        check(lib().fd_smoother_eigenvalues(self._h, _ptr(out), _stream()))
        return out


def smoothing_eigenvalues(kind, op: BlurOperator) -> Smoother:
    """smoothing_eigenvalues(_2d) (regularize.cpp:19-38, multidim.cpp:329-356)."""
    k = SMOOTHER[kind] if isinstance(kind, str) else int(kind)
    h = C.c_void_p()
    check(lib().fd_smoother_create(op._h, k, C.byref(h)))
    return Smoother(h, op, k)


def smoother_from_eigenvalues(op: BlurOperator, s) -> Smoother:
    """SmoothingOperator aggregate with caller-supplied eigenvalues."""
    a, p = _host(s)
    if a.size != op.size:
        raise ValidationError("smoother length != operator order")
    h = C.c_void_p()
    check(lib().fd_smoother_create_custom(op._h, p, C.byref(h)))
    return Smoother(h, op, 3)


# ---------------------------------------------------------------------------
# regularisation
# ---------------------------------------------------------------------------
@dataclass
class GcvSearch:
    """regularize.hpp:99-103."""
    mu_min: float = 1e-12
    mu_max: float = 10.0
    count: int = 200


@dataclass
class GcvResult:
    """regularize.hpp:105-108 (+ the grid argmin, per item)."""
    mu: torch.Tensor
    best_k: torch.Tensor
    curve: torch.Tensor | None


@dataclass
class MuChoice:
    """pipeline.hpp:49-52."""
    use_gcv: bool = False
    fixed_mu: float = 0.0


@dataclass
class RestorationReport:
    """regularize.hpp:126-133 (batched)."""
    restored: torch.Tensor
    mu_used: torch.Tensor
    best_k: torch.Tensor | None
    gcv_curve: torch.Tensor | None
    imag_residue: torch.Tensor


def tikhonov_solve(op: BlurOperator, L: Smoother, g, mu, want_imag_residue=False):
    """tikhonov_solve(_2d) -> (f_reg, imag_residue); mu scalar or per item.

    The imaginary residue of complex bases is a diagnostic (operators.cpp:222-229);
    requesting it runs the exact one-line-per-FFT synthesis, otherwise two real
    lines share each FFT and imag_residue is None."""
    g = _dev(g)
    count, lead = op._count(g)
    mu_t = torch.as_tensor(mu, dtype=torch.float64).to("cuda").expand(lead).contiguous() \
        if np.ndim(mu) == 0 else _dev(mu).reshape(lead).contiguous()
    out = torch.empty_like(g)
    res = torch.zeros(lead, dtype=torch.float64, device="cuda") \
        if (want_imag_residue or not op.complex) else None
    check(lib().fd_tikhonov(op._h, L._h, _ptr(g), _ptr(mu_t), _ptr(out), _ptr(res), count,
                            _stream()))
    return out, res


def gcv_value(op: BlurOperator, L: Smoother, g, mu):
    g = _dev(g)
    count, lead = op._count(g)
    G = torch.empty(lead, dtype=torch.float64, device="cuda")
    check(lib().fd_gcv_value(op._h, L._h, _ptr(g), float(mu), _ptr(G), count, _stream()))
    return G


def gcv_select(op: BlurOperator, L: Smoother, g, search: GcvSearch = GcvSearch(),
               want_curve=True) -> GcvResult:
    g = _dev(g)
    count, lead = op._count(g)
    mu = torch.empty(lead, dtype=torch.float64, device="cuda")
    bk = torch.empty(lead, dtype=torch.int32, device="cuda")
    curve = torch.empty(lead + (search.count,), dtype=torch.float64, device="cuda") \
        if want_curve else None
    check(lib().fd_gcv_select(op._h, L._h, _ptr(g), float(search.mu_min), float(search.mu_max),
                              int(search.count), _ptr(mu), _ptr(bk), _ptr(curve), count,
                              _stream()))
    return GcvResult(mu, bk, curve)


def deblur(op: BlurOperator, L: Smoother, g, mu: MuChoice, want_curve=False,
           search: GcvSearch = GcvSearch(), out=None,
           want_imag_residue=False) -> RestorationReport:
    """deblur(_2d) (pipeline.cpp:120-165).  imag_residue as in tikhonov_solve.
    A float32 g takes the fp32 storage variant (fd_deblur_f32: float in / out,
    fp64 arithmetic)."""
    f32 = isinstance(g, torch.Tensor) and g.dtype == torch.float32
    g = _dev(g, torch.float32 if f32 else torch.float64)
    count, lead = op._count(g)
    restored = torch.empty_like(g) if out is None else out
    mu_used = torch.empty(lead, dtype=torch.float64, device="cuda")
    bk = torch.full(lead, -1, dtype=torch.int32, device="cuda")
    curve = torch.empty(lead + (search.count,), dtype=torch.float64, device="cuda") \
        if want_curve else None
    res = torch.zeros(lead, dtype=torch.float64, device="cuda") \
        if (want_imag_residue or not op.complex) else None
    fn = lib().fd_deblur_f32 if f32 else lib().fd_deblur
    check(fn(op._h, L._h, _ptr(g), int(bool(mu.use_gcv)), float(mu.fixed_mu),
                          float(search.mu_min), float(search.mu_max), int(search.count),
                          _ptr(restored), _ptr(mu_used), _ptr(bk) if mu.use_gcv else None,
                          _ptr(curve), _ptr(res), count, _stream()))
    return RestorationReport(restored, mu_used, bk if mu.use_gcv else None, curve, res)


def deblur_smoothers(op: BlurOperator, Ls, g, mu: MuChoice, search: GcvSearch = GcvSearch(),
                     outs=None):
    """deblur(_2d) of one batch under several smoothing norms of the same
    operator (fd_deblur_smoothers: one analysis, a GCV selection and a filtered
    synthesis per norm).  Returns one RestorationReport per norm, equal to
    separate ``deblur`` calls."""
    f32 = isinstance(g, torch.Tensor) and g.dtype == torch.float32
    g = _dev(g, torch.float32 if f32 else torch.float64)
    count, lead = op._count(g)
    nL = len(Ls)
    outs = [torch.empty_like(g) for _ in range(nL)] if outs is None else list(outs)
    mu_used = torch.empty((nL,) + tuple(lead), dtype=torch.float64, device="cuda")
    bk = torch.full((nL,) + tuple(lead), -1, dtype=torch.int32, device="cuda")
    hs = (C.c_void_p * nL)(*[L._h for L in Ls])
    ps = (C.c_void_p * nL)(*[o.data_ptr() for o in outs])
    check(lib().fd_deblur_smoothers(op._h, nL, hs, _ptr(g), int(f32), int(bool(mu.use_gcv)),
                                    float(mu.fixed_mu), float(search.mu_min),
                                    float(search.mu_max), int(search.count), ps, _ptr(mu_used),
                                    _ptr(bk) if mu.use_gcv else None, count, _stream()))
    zero = torch.zeros(lead, dtype=torch.float64, device="cuda")
    return [RestorationReport(outs[l], mu_used[l], bk[l] if mu.use_gcv else None, None, zero)
            for l in range(nL)]


@dataclass
class SweepPoint:
    """pipeline.hpp:23-28."""
    mu: float
    gcv: float
    rre: float


@dataclass
class BcSweep:
    """pipeline.hpp:30-38."""
    bc: str
    min_rre: float
    mu_opt: float
    mu_gcv: float
    rre_gcv: float
    curve: list


def sweep_mu(op: BlurOperator, L: Smoother, g, truth=None,
             search: GcvSearch = GcvSearch()) -> BcSweep:
    """sweep_mu / sweep_mu_2d (pipeline.cpp:55-115) for one signal or image:
    G and (with truth) the RRE of the Tikhonov solution at every grid mu, the
    RRE-optimal grid mu and the RRE at the GCV choice."""
    g = _dev(g)
    if tuple(g.shape) != op.shape:
        raise ValidationError(f"sweep_mu takes one item of shape {op.shape}")
    t = None if truth is None else _dev(truth)
    if t is not None and tuple(t.shape) != op.shape:
        raise ValidationError("truth shape differs from the signal")
    K = int(search.count)
    mus, G, rr, summ = (np.empty(K), np.empty(K), np.empty(K), np.empty(4))
    dp = C.POINTER(C.c_double)
    check(lib().fd_sweep_mu(op._h, L._h, _ptr(g), _ptr(t), C.c_double(search.mu_min),
                            C.c_double(search.mu_max), K, mus.ctypes.data_as(dp),
                            G.ctypes.data_as(dp), rr.ctypes.data_as(dp), summ.ctypes.data_as(dp),
                            _stream()))
    pts = [SweepPoint(float(m), float(v), float(r)) for m, v, r in zip(mus, G, rr)]
    return BcSweep(BC_NAMES.get(op.bc, op.bc), float(summ[0]), float(summ[1]), float(summ[2]),
                   float(summ[3]), pts)


def deblur_host(op: BlurOperator, L: Smoother, g, mu: MuChoice, search: GcvSearch = GcvSearch(),
                out=None, chunk=0):
    """deblur for HOST arrays (the end-to-end entry point): chunks of the batch
    stream through H2D copy -> deblur -> D2H copy on separate CUDA streams
    (fd_deblur_host).  g: CPU float64 (or float32: fd_deblur_host_f32) tensor
    [..., shape] (pinned for overlap).  Returns (restored, mu_used, best_k) as
    CPU tensors."""
    if not isinstance(g, torch.Tensor):
        g = torch.from_numpy(np.ascontiguousarray(np.asarray(g, dtype=np.float64)))
    if g.is_cuda or g.dtype not in (torch.float64, torch.float32) or not g.is_contiguous():
        raise ValidationError("deblur_host needs a contiguous CPU float64 / float32 tensor")
    count, lead = op._count(g)
    pin = g.is_pinned()
    restored = torch.empty(g.shape, dtype=g.dtype, pin_memory=pin) if out is None else out
    mu_used = torch.empty(lead, dtype=torch.float64, pin_memory=pin)
    bk = torch.full(lead, -1, dtype=torch.int32)
    fn = lib().fd_deblur_host_f32 if g.dtype == torch.float32 else lib().fd_deblur_host
    check(fn(op._h, L._h, _ptr(g), int(bool(mu.use_gcv)), float(mu.fixed_mu),
                               float(search.mu_min), float(search.mu_max), int(search.count),
                               _ptr(restored), _ptr(mu_used), _ptr(bk), count, int(chunk),
                               _stream()))
    return restored, mu_used, bk


def deblur_host_multi(ops, Ls, g, mu: MuChoice, search: GcvSearch = GcvSearch(), outs=None,
                      chunk=0):
    """One host batch restored under several operators of the same shape
    (fd_deblur_host_multi: each chunk is uploaded once).  Returns a list of
    (restored, mu_used, best_k) CPU tensors, one per operator."""
    if not isinstance(g, torch.Tensor):
        g = torch.from_numpy(np.ascontiguousarray(np.asarray(g, dtype=np.float64)))
    if g.is_cuda or g.dtype not in (torch.float64, torch.float32) or not g.is_contiguous():
        raise ValidationError("deblur_host_multi needs a contiguous CPU float64 / float32 tensor")
    k = len(ops)
    if k == 0 or len(Ls) != k:
        raise ValidationError("one smoother per operator")
    count, lead = ops[0]._count(g)
    pin = g.is_pinned()
    outs = outs or [torch.empty(g.shape, dtype=g.dtype, pin_memory=pin) for _ in range(k)]
    mu_used = torch.empty((k,) + tuple(lead), dtype=torch.float64, pin_memory=pin)
    bk = torch.full((k,) + tuple(lead), -1, dtype=torch.int32)
    hops = (C.c_void_p * k)(*[op._h for op in ops])
    hls = (C.c_void_p * k)(*[L._h for L in Ls])
    houts = (C.c_void_p * k)(*[_ptr(o) for o in outs])
    check(lib().fd_deblur_host_multi(k, hops, hls, _ptr(g), int(g.dtype == torch.float32),
                                     int(bool(mu.use_gcv)), float(mu.fixed_mu),
                                     float(search.mu_min), float(search.mu_max),
                                     int(search.count), houts, _ptr(mu_used), _ptr(bk), count,
                                     int(chunk), _stream()))
    return [(outs[i], mu_used[i], bk[i]) for i in range(k)]


# ---------------------------------------------------------------------------
# input generation on the device (pipeline.cpp:14-51, operators.cpp:332-358)
# ---------------------------------------------------------------------------
def convolve_valid(ext, psf):
    """convolve_valid over the last axis of a device array [..., n + 2m] with the
    (2m+1)-tap mask ``psf`` (used as given) -> [..., n]."""
    ext = _dev(ext)
    w = np.ascontiguousarray(psf, dtype=np.float64)
    n = ext.shape[-1] - (len(w) - 1)
    if len(w) % 2 == 0 or n < 1:
        raise ValidationError("psf length must be odd and shorter than the extended signal")
    count = int(np.prod(ext.shape[:-1])) if ext.dim() > 1 else 1
    out = torch.empty(ext.shape[:-1] + (n,), dtype=torch.float64, device="cuda")
    check(lib().fd_convolve_valid(_ptr(ext), count, n, w.ctypes.data_as(C.POINTER(C.c_double)),
                                  len(w), _ptr(out), _stream()))
    return out


def convolve_valid_2d(ext, psf2d):
    """convolve_valid_2d over the last two axes of a device array
    [..., n1 + 2 m1, n2 + 2 m2] with the (2 m1 + 1) x (2 m2 + 1) mask."""
    ext = _dev(ext)
    w = np.ascontiguousarray(psf2d, dtype=np.float64)
    n1, n2 = ext.shape[-2] - (w.shape[0] - 1), ext.shape[-1] - (w.shape[1] - 1)
    if w.shape[0] % 2 == 0 or w.shape[1] % 2 == 0 or n1 < 1 or n2 < 1:
        raise ValidationError("psf sides must be odd and smaller than the extended image")
    count = int(np.prod(ext.shape[:-2])) if ext.dim() > 2 else 1
    out = torch.empty(ext.shape[:-2] + (n1, n2), dtype=torch.float64, device="cuda")
    check(lib().fd_convolve_valid_2d(_ptr(ext), count, n1, n2,
                                     w.ctypes.data_as(C.POINTER(C.c_double)), w.shape[0],
                                     w.shape[1], _ptr(out), _stream()))
    return out


def add_noise(g, level, seeds, item_dims=1):
    """add_noise on a device array, in place: the trailing ``item_dims`` axes
    form one item (flattened row-major, as the reference's 2D callers do);
    ``seeds``: one uint64 per item (scalar for a single item).  Returns g."""
    g = _dev(g)
    n = int(np.prod(g.shape[g.dim() - item_dims:]))
    count = int(np.prod(g.shape[:g.dim() - item_dims])) if g.dim() > item_dims else 1
    s = np.ascontiguousarray(np.broadcast_to(np.asarray(seeds, dtype=np.uint64), (count,)))
    check(lib().fd_add_noise(_ptr(g), count, n, float(level),
                             s.ctypes.data_as(C.POINTER(C.c_ulonglong)), _stream()))
    return g
