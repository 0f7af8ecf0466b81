"""CPU restatement of the reference's transform + filter + GCV path (numpy).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module, and only as the checker.  The product (``paper_0906_2704_b200``) never
imports it and has no CPU fallback.

Every function restates the reference algorithm it names (paths relative to
``/root/reference/proj``).  Transforms use ``numpy.fft`` (pocketfft) in place
of FFTW; the factorisation around the FFT (reorders, quarter-wave twiddles,
odd extensions, scalings) follows trig.cpp line for line, so results agree
with the reference to rounding (pinned in tests/test_oracle_pins.py against
the reference compiled in ``oracle/_ref`` and against the reference tests'
known answers).

Array conventions: 1D routines act on the last axis (leading axes are a
batch), 2D routines on the last two axes (row-major n1 x n2, multidim.hpp:66).

Extensions beyond the reference (flagged where defined):
  * ``first_difference`` smoother, s = sqrt(2 - 2 cos(node)).
  * higher-order borders ``hoc-fourier-d1`` / ``hoc-fourier-d3`` (degree d = 1
    and 3 for nonsymmetric PSFs, BASELINE configs 1 and 3): the paper's
    construction (polynomial columns with eigenvalue
    1 around an interior trigonometric basis, inverse by Sherman-Morrison-
    Woodbury, Theorem sec:sherm) generalised to k = d border columns; see
    ``HoTransform``.  Not in the reference, so pinned by a dense construction
    (T built entry-wise and solved by LU, as oracle.cpp:102-223 does for the
    reference's own transforms), polynomial preservation, and equality with the
    reference's hoc-fourier operator at d = 2 (tests/test_ho_borders.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

PI = math.pi

# BoundaryCondition (operators.hpp:15-21) codes, shared with the C-ABI.
PERIODIC, REFLECTIVE, ANTIREFLECTIVE, HOC_COSINE, HOC_FOURIER = range(5)
# extension codes (not in the reference): higher-order Fourier borders
HOC_FOURIER_D1, HOC_FOURIER_D3 = 5, 6
BC_NAMES = ("periodic", "reflective", "antireflective", "hoc-cosine", "hoc-fourier",
            "hoc-fourier-d1", "hoc-fourier-d3")
# (k_left, k_right, degree) of the generalised borders; the d = 2 member
# ("ho-2", borders (1, 1)) is the same operator as the reference's hoc-fourier
HO_BORDERS = {HOC_FOURIER_D1: (1, 0, 1), HOC_FOURIER_D3: (2, 1, 3)}
# BoundaryBasis (boundary.hpp:18)
B_AR, B_HC, B_HF = range(3)
# SmootherKind (regularize.hpp:15) + extension
IDENTITY, LAPLACIAN, FIRST_DIFFERENCE = range(3)


class ValidationError(ValueError):
    """errors.hpp:16-19 (CLI exit code 2)."""


class DegenerateError(ArithmeticError):
    """errors.hpp:38-41 (CLI exit code 3)."""


def needs_symmetric_psf(bc):  # operators.cpp:94-98
    return bc in (REFLECTIVE, ANTIREFLECTIVE, HOC_COSINE)


def is_complex_basis(bc):  # operators.cpp:100-102 (+ extension codes)
    return bc in (PERIODIC, HOC_FOURIER, HOC_FOURIER_D1, HOC_FOURIER_D3)


def is_boundary_corrected(bc):  # operators.cpp:104-108
    return bc in (ANTIREFLECTIVE, HOC_COSINE, HOC_FOURIER)


def is_higher_order(bc):  # extension
    return bc in HO_BORDERS


# --------------------------------------------------------------------------
# PSF (psf.cpp)
# --------------------------------------------------------------------------
@dataclass
class Psf:
    weights: np.ndarray
    m: int
    symmetric: bool

    def support(self):
        return 2 * self.m + 1

    def at(self, j):
        return self.weights[self.m + j]


def make_psf(weights, normalize=False) -> Psf:
    """psf.cpp:10-37."""
    w = np.asarray(weights, dtype=np.float64).copy()
    if w.size == 0 or w.size % 2 == 0:
        raise ValidationError("psf must have odd length 2m+1")
    if not np.all(np.isfinite(w)):
        raise ValidationError("psf weights must be finite")
    s = 0.0
    for x in w:  # serial sum, as the reference
        s += float(x)
    if normalize:
        if s == 0.0:
            raise ValidationError("psf weights sum to zero; cannot normalize")
        w = w / s
    elif abs(s - 1.0) > 1e-8:
        raise ValidationError("psf weights must sum to 1 (pass normalize to rescale)")
    m = w.size // 2
    sym = bool(np.all(w[m + 1:] == w[:m][::-1]))
    return Psf(w, m, sym)


def gaussian_psf(m, sigma) -> Psf:
    """psf.cpp:62-69."""
    j = np.arange(-m, m + 1, dtype=np.float64)
    return make_psf(np.exp(-j * j / (2.0 * sigma * sigma)), normalize=True)


def symbol_eval(psf: Psf, t):
    """z(t) = sum_j h_j e^{ijt} (psf.cpp:39-52); vectorised over t."""
    t = np.asarray(t, dtype=np.float64)
    if psf.symmetric:
        z = np.full(t.shape, psf.at(0))
        for j in range(1, psf.m + 1):
            z = z + 2.0 * psf.at(j) * np.cos(j * t)
        return z.astype(np.complex128)
    z = np.full(t.shape, psf.at(0), dtype=np.complex128)
    for j in range(1, psf.m + 1):
        c, s = np.cos(j * t), np.sin(j * t)
        z = z + psf.at(j) * (c + 1j * s) + psf.at(-j) * (c - 1j * s)
    return z


# --------------------------------------------------------------------------
# Trig transforms (trig.cpp:116-180)
# --------------------------------------------------------------------------
def fourier_apply(v, forward=True):
    """Unitary DFT F v / F^H v (trig.cpp:116-124)."""
    v = np.asarray(v, dtype=np.complex128)
    m = v.shape[-1]
    y = np.fft.fft(v, axis=-1) if forward else np.fft.ifft(v, axis=-1) * m
    return y * (1.0 / math.sqrt(m))


def _dct_tw(m):
    ang = -0.5 * PI * np.arange(m, dtype=np.float64) / m  # trig.cpp:73-87
    return np.cos(ang) + 1j * np.sin(ang)


def cosine_apply(v, forward=True):
    """Orthogonal DCT-II C v (forward) / C^T v (inverse), trig.cpp:126-160."""
    v = np.asarray(v, dtype=np.float64)
    m = v.shape[-1]
    if m == 1:
        return v.copy()
    tw = _dct_tw(m)
    s0, s = math.sqrt(1.0 / m), math.sqrt(2.0 / m)
    scale = np.full(m, s)
    scale[0] = s0
    half = (m + 1) // 2
    nodd = m // 2
    if forward:
        buf = np.empty(v.shape, dtype=np.complex128)
        buf[..., :half] = v[..., 0::2]
        buf[..., m - 1 - np.arange(nodd)] = v[..., 1::2]
        spec = np.fft.fft(buf, axis=-1)
        return scale * (tw * spec).real
    buf = scale * v * tw
    spec = np.fft.fft(buf, axis=-1)
    out = np.empty(v.shape, dtype=np.float64)
    out[..., 0::2] = spec[..., :half].real
    out[..., 1::2] = spec[..., m - 1 - np.arange(nodd)].real
    return out


def sine_apply(v):
    """DST-I Q v via the odd extension of length 2(m+1), trig.cpp:162-180."""
    v = np.asarray(v, dtype=np.float64)
    m = v.shape[-1]
    ln = 2 * (m + 1)
    buf = np.zeros(v.shape[:-1] + (ln,), dtype=np.complex128)
    buf[..., 1:m + 1] = v
    buf[..., ln - 1 - np.arange(m)] = -v
    spec = np.fft.fft(buf, axis=-1)
    return (-0.5 * math.sqrt(2.0 / (m + 1.0))) * spec[..., 1:m + 1].imag


# --------------------------------------------------------------------------
# Boundary transforms T_X (boundary.cpp)
# --------------------------------------------------------------------------
@dataclass
class StructuredTransform:
    basis: int
    n: int
    q: np.ndarray
    c_a: np.ndarray
    c_b: np.ndarray
    alpha: float
    v: np.ndarray
    w: np.ndarray
    row_a: np.ndarray
    row_b: np.ndarray
    capacitance: np.ndarray  # [m00, m01, m10, m11]
    has_correction: bool
    cav: tuple = (0.0, 0.0, 0.0, 0.0)  # (ca_v, ca_w, cb_v, cb_w)
    a: float = 0.0
    b: float = 0.0
    points: np.ndarray = field(default_factory=lambda: np.zeros(0))


def extended_grid(basis, n):
    """boundary.cpp:132-160 -> (a, b, points)."""
    if n < 5:
        raise ValidationError("boundary transform needs order n >= 5")
    i = np.arange(n)
    if basis == B_AR:
        return 0.0, PI, i * PI / (n - 1)
    if basis == B_HC:
        return (-PI / (2 * n - 4), (2 * n - 3) * PI / (2 * n - 4),
                (2 * i - 1) * PI / (2 * n - 4))
    return -2.0 * PI / (n - 2), 2.0 * PI, (i - 1) * 2.0 * PI / (n - 2)


def _interior_apply(basis, x, forward):
    """boundary.cpp:35-43."""
    if basis == B_HF:
        return fourier_apply(x, forward)
    if basis == B_AR:
        return sine_apply(x)
    return cosine_apply(x, forward)


def _check_capacitance(mm):
    """boundary.cpp:54-64 (2-norm condition <= 1e12)."""
    a2 = np.abs(np.asarray(mm)) ** 2
    t = float(a2.sum())
    det = mm[0] * mm[3] - mm[1] * mm[2]
    d = abs(det) ** 2
    r = math.sqrt(max(t * t - 4.0 * d, 0.0))
    smax = math.sqrt((t + r) / 2.0)
    smin2 = (t - r) / 2.0
    if smin2 <= 0.0 or smax / math.sqrt(smin2) > 1e12:
        raise DegenerateError("degenerate transform: 2x2 capacitance matrix is "
                              "singular or ill-conditioned")


def _assemble(basis, n, q, c_a, c_b, grid):
    """boundary.cpp:132-160."""
    cplx = basis == B_HF
    q = np.asarray(q, dtype=np.float64)
    norm = math.sqrt(sum(float(x) * float(x) for x in q))
    q = q / norm
    q[-1] = 0.0
    alpha = 1.0 / q[0]
    qhat = q[1:n - 1].copy()
    qflip = qhat[::-1].copy()
    dt = np.complex128 if cplx else np.float64
    v = _interior_apply(basis, qhat.astype(dt), True) * (-alpha)
    w = _interior_apply(basis, qflip.astype(dt), True) * (-alpha)
    has_corr = basis != B_AR
    if has_corr:
        # row = X^T c: DCT-II has X^T = X^-1, the DFT matrix is symmetric
        row_a = _interior_apply(basis, c_a, forward=cplx)
        row_b = _interior_apply(basis, c_b, forward=cplx)
        ca_v, ca_w = np.sum(c_a * v), np.sum(c_a * w)
        cb_v, cb_w = np.sum(c_b * v), np.sum(c_b * w)
        cap = np.array([1 + ca_v, ca_w, cb_v, 1 + cb_w], dtype=dt)
        _check_capacitance(cap)
        cav = (ca_v, ca_w, cb_v, cb_w)
    else:
        row_a = np.zeros(n - 2, dtype=dt)
        row_b = np.zeros(n - 2, dtype=dt)
        cap = np.array([1, 0, 0, 1], dtype=dt)
        cav = (0.0, 0.0, 0.0, 0.0)
    a, b, pts = grid
    return StructuredTransform(basis, n, q, np.asarray(c_a, dt), np.asarray(c_b, dt), alpha,
                               v, w, row_a, row_b, cap, has_corr, cav, a, b, pts)


def build_transform(basis, n) -> StructuredTransform:
    """build_real_transform / build_fourier_transform (boundary.cpp:162-217)."""
    grid = extended_grid(basis, n)
    a, b, pts = grid
    m = n - 2
    if basis == B_AR:
        q = 1.0 - np.arange(n) / (n - 1)
        z = np.zeros(m)
        return _assemble(basis, n, q, z, z.copy(), grid)
    q = (b - pts) ** 2
    j = np.arange(m)
    if basis == B_HC:
        scale = np.where(j == 0, math.sqrt(1.0 / m), math.sqrt(2.0 / m))
        c_a = scale * np.cos(j * a)
        c_b = np.where(j % 2 == 0, c_a, -c_a)
        return _assemble(basis, n, q, c_a, c_b, grid)
    q[-1] = 0.0
    scale = 1.0 / math.sqrt(m)
    c_a = scale * (np.cos(j * a) + 1j * np.sin(j * a))
    c_b = np.full(m, scale, dtype=np.complex128)
    return _assemble(basis, n, q, c_a, c_b, grid)


def transform_apply(t: StructuredTransform, u):
    """y = T_X u (boundary.cpp:225-250); batched over leading axes."""
    u = np.asarray(u)
    n = t.n
    if u.shape[-1] != n:
        raise ValidationError("transform_apply: input length != n")
    mid = u[..., 1:n - 1]
    interior = _interior_apply(t.basis, mid, forward=False)
    top = np.sum(t.c_a * mid, axis=-1)
    bottom = np.sum(t.c_b * mid, axis=-1)
    u0, un = u[..., :1], u[..., n - 1:]
    out = np.empty(u.shape, dtype=np.result_type(u, t.v))
    out[..., 0] = t.q[0] * u[..., 0] + top
    out[..., 1:n - 1] = t.q[1:n - 1] * u0 + interior + t.q[n - 2:0:-1] * un
    out[..., n - 1] = bottom + t.q[0] * u[..., n - 1]
    return out


def transform_apply_inverse(t: StructuredTransform, y):
    """v = T_X^-1 y (boundary.cpp:253-289); batched over leading axes."""
    y = np.asarray(y)
    n = t.n
    if y.shape[-1] != n:
        raise ValidationError("transform_apply_inverse: input length != n")
    y1, yn = y[..., :1], y[..., n - 1:]
    mid = y[..., 1:n - 1]
    xi = _interior_apply(t.basis, mid, forward=True)
    out = np.empty(y.shape, dtype=np.result_type(y, t.v))
    out[..., :1] = t.alpha * y1
    out[..., n - 1:] = t.alpha * yn
    out[..., 1:n - 1] = y1 * t.v + xi + yn * t.w
    if t.has_correction:
        ca_v, ca_w, cb_v, cb_w = t.cav
        ra = ca_v * y1 + ca_w * yn + np.sum(t.row_a * mid, axis=-1, keepdims=True)
        rb = cb_v * y1 + cb_w * yn + np.sum(t.row_b * mid, axis=-1, keepdims=True)
        m = t.capacitance
        det = m[0] * m[3] - m[1] * m[2]
        beta0 = (ra * m[3] - rb * m[1]) / det
        beta1 = (rb * m[0] - ra * m[2]) / det
        out[..., :1] -= beta0 * t.alpha
        out[..., n - 1:] -= beta1 * t.alpha
        out[..., 1:n - 1] -= beta0 * t.v + beta1 * t.w
    return out


# --------------------------------------------------------------------------
# Extension: higher-order polynomial borders around a Fourier interior
# --------------------------------------------------------------------------
def legendre_columns(n, degree):
    """Border columns: Legendre polynomials P_1..P_d of t_i = (2i-(n-1))/(n-1),
    each scaled to unit 2-norm on the n grid points.

    The operator A = T diag(d) T^-1 only depends on span(P u {1}) = P_d (the
    eigenvalue-1 eigenspace) and on the interior columns, not on the basis
    chosen for the border columns; this basis is near-orthogonal, which gives
    the smallest cond(T) of the bases tried (the raw monomials
    (b-x)^p of the d = 2 construction give cond(T) 20x larger at d = 3).
    Operation order as build_ho_axis (fd_capi.cu): Bonnet recurrence per
    element, sequential sum of squares, so the table is bit-identical."""
    t = (2.0 * np.arange(n) - (n - 1)) / (n - 1)
    p_prev, p = np.ones(n), t.copy()
    cols = []
    for k in range(1, degree + 1):
        if k > 1:  # Bonnet: k P_k = (2k-1) t P_{k-1} - (k-1) P_{k-2}
            p_prev, p = p, ((2 * k - 1) * t * p - (k - 1) * p_prev) / k
        cols.append(p / math.sqrt(float(np.cumsum(p * p)[-1])))
    return np.stack(cols, axis=1)


def _gauss_jordan_inverse(S):
    """Inverse of the k x k border capacitance by Gauss-Jordan elimination with
    partial pivoting, in the operation order of build_ho_axis (fd_capi.cu):
    cond(S) reaches ~1e6-1e7 at d = 3 (n = 1024-4096), so two different
    inversion orders already differ by ~1e-10; restating one order makes the
    device comparison measure the transforms, not the setup."""
    k = S.shape[0]
    W = [[float(S[r][c]) for c in range(k)] + [1.0 if c == r else 0.0 for c in range(k)]
         for r in range(k)]
    for c in range(k):
        piv = c
        for r in range(c + 1, k):
            if abs(W[r][c]) > abs(W[piv][c]):
                piv = r
        if W[piv][c] == 0.0:
            raise DegenerateError("degenerate transform: border capacitance is singular")
        W[c], W[piv] = W[piv], W[c]
        inv = 1.0 / W[c][c]
        W[c] = [x * inv for x in W[c]]
        for r in range(k):
            if r != c:
                f = W[r][c]
                W[r] = [W[r][j] - f * W[c][j] for j in range(2 * k)]
    return np.array([row[k:] for row in W])


@dataclass
class HoTransform:
    """T = [P_L | Phi | P_R] of order n: k_l + k_r = d polynomial columns (unit
    norm, eigenvalue 1) around the m = n - d interior Fourier columns
    phi_j(x) = e^{ijx}/sqrt(m) sampled on the grid x_i = (i - k_l) 2 pi / m,
    i = 0..n-1 (the paper's T_F of PAPER.md:418-431 at d = 2, with k_l = k_r = 1).

    The interior rows of Phi are F^H; every border row is the row of F^H at the
    2 pi-periodic image of its grid point (wrap), so with E the selection of
    those rows, Phi_B F = E exactly.  With S = P_B - E P_I (k x k):
      analyze   a = S^-1 (y_B - E y_I),  b = F (y_I - P_I a)
      synthesize  y_I = F^H b + P_I a,  y_B = E F^H b + P_B a
    (Schur complement of the unitary block; the rank-k form of the paper's
    Theorem th:inv).  Coefficients are ordered [a_left, b, a_right]."""
    bc: int
    n: int
    kl: int
    kr: int
    m: int
    degree: int
    P: np.ndarray       # (n, k) border columns
    border: np.ndarray  # (k,) grid rows of the border, top then bottom
    wrap: np.ndarray    # (k,) interior index (0..m-1) of each border row's image
    S: np.ndarray
    Sinv: np.ndarray

    @property
    def k(self):
        return self.kl + self.kr


def build_ho_transform(bc, n, borders=None) -> HoTransform:
    """``borders`` = (k_l, k_r, degree) overrides the code's (tests build the
    d = 2 member (1, 1, 2) to pin the family against the reference)."""
    kl, kr, deg = borders if borders is not None else HO_BORDERS[bc]
    k = kl + kr
    m = n - k
    if m < 3:
        raise ValidationError("higher-order borders need n >= degree + 3")
    P = legendre_columns(n, deg)
    border = np.array(list(range(kl)) + [kl + m + j for j in range(kr)])
    wrap = np.array([m - kl + i for i in range(kl)] + list(range(kr)))
    S = P[border, :] - P[kl + wrap, :]
    sv = np.linalg.svd(S, compute_uv=False)
    if sv[-1] <= 0.0 or sv[0] / sv[-1] > 1e12:  # as boundary.cpp:54-64 for k = 2
        raise DegenerateError("degenerate transform: border capacitance is singular or "
                              "ill-conditioned")
    return HoTransform(bc, n, kl, kr, m, deg, P, border, wrap, S, _gauss_jordan_inverse(S))


def ho_analyze(t: HoTransform, y):
    """T^-1 y, batched over leading axes."""
    y = np.asarray(y)
    kl, m = t.kl, t.m
    yI = y[..., kl:kl + m]
    r = y[..., t.border] - yI[..., t.wrap]
    a = r @ t.Sinv.T
    b = fourier_apply(yI - a @ t.P[kl:kl + m, :].T, forward=True)
    out = np.empty(y.shape, dtype=np.complex128)
    out[..., :kl] = a[..., :kl]
    out[..., kl:kl + m] = b
    out[..., kl + m:] = a[..., kl:]
    return out


def ho_synthesize(t: HoTransform, c):
    """T c, batched over leading axes."""
    c = np.asarray(c, dtype=np.complex128)
    kl, m = t.kl, t.m
    a = np.concatenate([c[..., :kl], c[..., kl + m:]], axis=-1)
    u = fourier_apply(c[..., kl:kl + m], forward=False)
    out = np.empty(c.shape, dtype=np.complex128)
    out[..., kl:kl + m] = u + a @ t.P[kl:kl + m, :].T
    out[..., t.border] = u[..., t.wrap] + a @ t.P[t.border, :].T
    return out


def ho_dense(t: HoTransform):
    """T entry-wise: border columns, then e^{i j x_i}/sqrt(m) (test oracle)."""
    x = (np.arange(t.n) - t.kl) * 2.0 * PI / t.m
    phi = np.exp(1j * np.outer(x, np.arange(t.m))) / math.sqrt(t.m)
    return np.hstack([t.P[:, :t.kl], phi, t.P[:, t.kl:]]).astype(np.complex128)


def ho_nodes(bc, n):
    """Symbol nodes: 0 at the border coefficients, 2 pi j / m in the interior."""
    kl, kr, _ = HO_BORDERS[bc]
    m = n - kl - kr
    x = np.zeros(n)
    x[kl:kl + m] = 2.0 * PI * np.arange(m) / m
    return x


# --------------------------------------------------------------------------
# Operators (operators.cpp)
# --------------------------------------------------------------------------
def eigenvalue_grid(bc, n):
    """Symbol nodes (operators.cpp:130-161)."""
    if is_boundary_corrected(bc) and n < 5:
        raise ValidationError("boundary-corrected grids need n >= 5")
    if is_higher_order(bc):
        return ho_nodes(bc, n)
    x = np.zeros(n)
    i = np.arange(n)
    if bc == PERIODIC:
        x = 2.0 * PI * i / n
    elif bc == REFLECTIVE:
        x = PI * i / n
    elif bc == ANTIREFLECTIVE:
        x[:n - 1] = PI * i[:n - 1] / (n - 1)
    elif bc == HOC_COSINE:
        x[1:n - 1] = PI * (i[1:n - 1] - 1) / (n - 2)
    else:
        x[1:n - 1] = 2.0 * PI * (i[1:n - 1] - 1) / (n - 2)
    return x


def validate_build(psf: Psf, n, bc):
    """operators.cpp:62-76."""
    if needs_symmetric_psf(bc) and not psf.symmetric:
        raise ValidationError(f"{BC_NAMES[bc]} boundary conditions require a symmetric psf")
    if is_higher_order(bc):
        kl, kr, _ = HO_BORDERS[bc]
        if n < kl + kr + 3:
            raise ValidationError("higher-order borders need n >= degree + 3")
        if psf.support() > n - kl - kr:
            raise ValidationError("psf support 2m+1 must be <= n-d")
    elif is_boundary_corrected(bc):
        if n < 5:
            raise ValidationError("boundary-corrected operators need n >= 5")
        if psf.support() > n - 2:
            raise ValidationError("psf support 2m+1 must be <= n-2")
    else:
        if n < 1:
            raise ValidationError("operator order must be positive")
        if psf.support() > n:
            raise ValidationError("psf support 2m+1 must be <= n")


def operator_eigenvalues(psf: Psf, n, bc):
    """d = z(node) with pinned boundary eigenvalues 1 (operators.cpp:238-286).

    The reference sums the symbol directly for support <= 64 and uses a wrapped
    FFT otherwise (operators.cpp:23-33); both give z(node) to rounding, and
    this restatement always sums directly.  Real bases return float64.
    """
    validate_build(psf, n, bc)
    if bc == PERIODIC:
        return symbol_eval(psf, 2.0 * PI * np.arange(n) / n)
    if bc == REFLECTIVE:
        return symbol_eval(psf, np.arange(n) * PI / n).real
    if is_higher_order(bc):
        kl, kr, _ = HO_BORDERS[bc]
        d = np.ones(n, dtype=np.complex128)
        d[kl:n - kr] = symbol_eval(psf, 2.0 * PI * np.arange(n - kl - kr) / (n - kl - kr))
        return d
    d = np.ones(n, dtype=np.complex128 if is_complex_basis(bc) else np.float64)
    k = np.arange(n - 2)
    if bc == ANTIREFLECTIVE:
        d[1:n - 1] = symbol_eval(psf, (k + 1) * PI / (n - 1)).real
    elif bc == HOC_COSINE:
        d[1:n - 1] = symbol_eval(psf, k * PI / (n - 2)).real
    else:
        d[1:n - 1] = symbol_eval(psf, 2.0 * PI * k / (n - 2))
    return d


class SpectralBasis:
    """operators.cpp:164-201: synthesize = T_X, analyze = T_X^-1."""

    def __init__(self, bc, n):
        self.bc, self.n = bc, n
        self.t = None
        if bc == ANTIREFLECTIVE:
            self.t = build_transform(B_AR, n)
        elif bc == HOC_COSINE:
            self.t = build_transform(B_HC, n)
        elif bc == HOC_FOURIER:
            self.t = build_transform(B_HF, n)
        self.ho = build_ho_transform(bc, n) if is_higher_order(bc) else None

    @property
    def complex(self):
        return is_complex_basis(self.bc)

    def synthesize(self, c):
        if self.ho is not None:
            return ho_synthesize(self.ho, c)
        if self.t is not None:
            return transform_apply(self.t, c)
        if self.complex:
            return fourier_apply(c, forward=False)
        return cosine_apply(c, forward=False)

    def analyze(self, y):
        if self.ho is not None:
            return ho_analyze(self.ho, y)
        if self.t is not None:
            return transform_apply_inverse(self.t, y)
        if self.complex:
            return fourier_apply(y, forward=True)
        return cosine_apply(y, forward=True)


@dataclass
class BlurOperator:
    bc: int
    n: int
    eigenvalues: np.ndarray
    psf: Psf
    basis: SpectralBasis

    def apply(self, f):
        """Matvec A f (operators.cpp:207-232) -> (out, imag_residue)."""
        f = np.asarray(f, dtype=np.float64)
        if f.shape[-1] != self.n:
            raise ValidationError("blur apply: signal length != operator order")
        if not self.basis.complex:
            return self.basis.synthesize(self.basis.analyze(f) * self.eigenvalues), \
                np.zeros(f.shape[:-1])
        yc = self.basis.synthesize(self.basis.analyze(f.astype(np.complex128)) * self.eigenvalues)
        return yc.real.copy(), np.sqrt(np.sum(yc.imag ** 2, axis=-1))


def build_operator(psf: Psf, n, bc) -> BlurOperator:
    """operators.cpp:293-301."""
    validate_build(psf, n, bc)
    return BlurOperator(bc, n, operator_eigenvalues(psf, n, bc), psf, SpectralBasis(bc, n))


# --------------------------------------------------------------------------
# Regularisation (regularize.hpp / regularize.cpp)
# --------------------------------------------------------------------------
def smoothing_eigenvalues(kind, bc, n, d=None):
    """regularize.cpp:19-38; FIRST_DIFFERENCE is an extension."""
    if kind == IDENTITY:
        return np.ones(n)
    nodes = eigenvalue_grid(bc, n)
    s = 2.0 - 2.0 * np.cos(nodes)
    if kind == FIRST_DIFFERENCE:
        s = np.sqrt(s)
    if d is not None and np.any((s == 0.0) & (np.abs(d) == 0.0)):
        raise ValidationError("incompatible smoother: joint null space with the blur operator")
    return s


def apply_tikhonov_filter(d, s, mu, ghat):
    """ghat * conj(d) / (|d|^2 + mu s^2) (regularize.hpp:42-58)."""
    if np.iscomplexobj(d):
        return ghat * (np.conj(d) / (np.abs(d) ** 2 + mu * s * s))
    return ghat * (d / (d * d + mu * s * s))


def gcv_from_coeffs(d, s, ghat, mu):
    """G(mu) = sum sigma^2 |ghat|^2 / (sum sigma)^2 (regularize.hpp:63-81).

    Sums over the last axis (or the last two axes when ``d`` is 2D)."""
    d2 = np.abs(d) ** 2 if np.iscomplexobj(d) else d * d
    sigma = s * s / (d2 + mu * s * s)
    g2 = np.abs(ghat) ** 2
    axes = tuple(range(-np.ndim(d), 0))
    num = np.sum(sigma * sigma * g2, axis=axes)
    den = np.sum(sigma)
    if den == 0.0:
        raise DegenerateError("degenerate gcv: all smoother eigenvalues are zero")
    return num / (den * den)


@dataclass
class GcvResult:
    mu: float
    mus: np.ndarray
    vals: np.ndarray
    best_k: int
    tied: bool
    evaluations: int


def gcv_grid(mu_min, mu_max, count):
    """Log-spaced grid (regularize.cpp:149-156)."""
    if not (mu_min > 0.0) or not (mu_max > mu_min) or count < 2:
        raise ValidationError("gcv search needs 0 < mu_min < mu_max and count >= 2")
    llo, lhi = math.log(mu_min), math.log(mu_max)
    return np.array([math.exp(llo + (lhi - llo) * k / (count - 1)) for k in range(count)])


def gcv_minimize(G, mu_min, mu_max, count, grid_vals=None) -> GcvResult:
    """gcv_minimize restated verbatim (regularize.cpp:144-214).

    ``G`` maps a scalar mu to G(mu); ``grid_vals`` optionally supplies the grid
    values (vectorised evaluation).  First minimum, 1e-12 relative tie test with
    geometric-midpoint return, golden section in log(mu) on the neighbours to
    exp(b-a)-1 <= 1e-3, final acceptance test G(refined) <= best."""
    mus = gcv_grid(mu_min, mu_max, count)
    vals = np.array([G(m) for m in mus]) if grid_vals is None else np.asarray(grid_vals, float)
    best_k = int(np.argmin(vals))  # first minimum, as std::min_element
    best = float(vals[best_k])
    if best == 0.0:
        tied = np.nonzero(vals == 0.0)[0]
    else:
        tied = np.nonzero(vals <= best + 1e-12 * abs(best))[0]
    evals = 0
    if tied.size > 1:
        mean_log = 0.0
        for k in tied:
            mean_log += math.log(mus[k])
        return GcvResult(math.exp(mean_log / tied.size), mus, vals, best_k, True, 0)
    lo = mus[best_k - 1 if best_k > 0 else 0]
    hi = mus[best_k + 1 if best_k + 1 < count else count - 1]
    a, b = math.log(lo), math.log(hi)
    invphi = 0.6180339887498949
    x1 = b - invphi * (b - a)
    x2 = a + invphi * (b - a)
    f1 = G(math.exp(x1))
    f2 = G(math.exp(x2))
    evals += 2
    while math.exp(b - a) - 1.0 > 1e-3:
        if f1 <= f2:
            b = x2
            x2 = x1
            f2 = f1
            x1 = b - invphi * (b - a)
            f1 = G(math.exp(x1))
        else:
            a = x1
            x1 = x2
            f1 = f2
            x2 = a + invphi * (b - a)
            f2 = G(math.exp(x2))
        evals += 1
    refined = math.exp(0.5 * (a + b))
    evals += 1
    mu = refined if G(refined) <= best else float(mus[best_k])
    return GcvResult(mu, mus, vals, best_k, False, evals)


def _coeffs(op, g):
    """analyze real data in the operator's basis (regularize.cpp:84-89)."""
    g = np.asarray(g, dtype=np.float64)
    return op.basis.analyze(g.astype(np.complex128) if op.basis.complex else g)


def _solve_from_coeffs(op, s, ghat, mu):
    yc = op.basis.synthesize(apply_tikhonov_filter(op.eigenvalues, s, mu, ghat))
    if op.basis.complex:
        return yc.real.copy(), np.sqrt(np.sum(yc.imag ** 2, axis=-1))
    return yc, np.zeros(yc.shape[:-1])


def tikhonov_solve(op: BlurOperator, s, g, mu):
    """regularize.cpp:73-116 -> (f_reg, imag_residue); batched."""
    if mu <= 0.0:
        raise ValidationError("mu must be positive")
    return _solve_from_coeffs(op, s, _coeffs(op, g), mu)


def gcv_value(op: BlurOperator, s, g, mu):
    """regularize.cpp:119-142."""
    if mu <= 0.0:
        raise ValidationError("mu must be positive")
    return gcv_from_coeffs(op.eigenvalues, s, _coeffs(op, g), mu)


def gcv_select(op: BlurOperator, s, g, mu_min, mu_max, count) -> GcvResult:
    """regularize.cpp:217-247 for one signal."""
    ghat = _coeffs(op, g)
    return _select_from_coeffs(op.eigenvalues, s, ghat, mu_min, mu_max, count)


def _select_from_coeffs(d, s, ghat, mu_min, mu_max, count):
    mus = gcv_grid(mu_min, mu_max, count)
    d2 = np.abs(d) ** 2 if np.iscomplexobj(d) else d * d
    g2 = np.abs(ghat) ** 2
    s2 = s * s
    # vectorised grid: sigma[k, i]
    grid = np.empty(count)
    for k0 in range(0, count, 16):
        mk = mus[k0:k0 + 16].reshape((-1,) + (1,) * np.ndim(d))
        sig = s2 / (d2 + mk * s2)
        axes = tuple(range(1, 1 + np.ndim(d)))
        num = np.sum(sig * sig * g2, axis=axes)
        den = np.sum(sig, axis=axes)
        if np.any(den == 0.0):
            raise DegenerateError("degenerate gcv: all smoother eigenvalues are zero")
        grid[k0:k0 + 16] = num / (den * den)
    return gcv_minimize(lambda mu: float(gcv_from_coeffs(d, s, ghat, mu)), mu_min, mu_max,
                        count, grid_vals=grid)


@dataclass
class Restoration:
    restored: np.ndarray
    mu_used: np.ndarray
    best_k: np.ndarray
    imag_residue: np.ndarray
    curves: np.ndarray | None


def deblur(op: BlurOperator, s, g, use_gcv=True, fixed_mu=0.0, mu_min=1e-12, mu_max=10.0,
           count=200, want_curve=False) -> Restoration:
    """deblur / deblur_impl (pipeline.cpp:120-155), batched over leading axes.

    Like the reference, the solve re-analyses g (pipeline.cpp:139-140)."""
    g = np.asarray(g, dtype=np.float64)
    flat = g.reshape(-1, op.n)
    B = flat.shape[0]
    mus_used = np.empty(B)
    best = np.full(B, -1)
    curves = np.empty((B, count)) if want_curve else None
    if use_gcv:
        ghat = _coeffs(op, flat)
        for b in range(B):
            r = _select_from_coeffs(op.eigenvalues, s, ghat[b], mu_min, mu_max, count)
            mus_used[b], best[b] = r.mu, r.best_k
            if want_curve:
                curves[b] = r.vals
    else:
        if not fixed_mu > 0.0:
            raise ValidationError("mu must be positive")
        mus_used[:] = fixed_mu
    out = np.empty_like(flat)
    res = np.empty(B)
    ghat = _coeffs(op, flat)
    for b in range(B):
        out[b], res[b] = _solve_from_coeffs(op, s, ghat[b], mus_used[b])
    shp = g.shape[:-1]
    return Restoration(out.reshape(g.shape), mus_used.reshape(shp), best.reshape(shp),
                       res.reshape(shp), curves)


# --------------------------------------------------------------------------
# 2D (multidim.cpp)
# --------------------------------------------------------------------------
@dataclass
class Psf2D:
    weights: np.ndarray  # (2m1+1, 2m2+1)
    m1: int
    m2: int
    symmetric: bool


def make_psf2d(weights, normalize=False) -> Psf2D:
    """multidim.cpp:81-109."""
    w = np.array(weights, dtype=np.float64)
    r, c = w.shape
    if r % 2 == 0 or c % 2 == 0:
        raise ValidationError("2D psf needs odd rows and cols")
    s = 0.0
    for x in w.ravel():
        s += float(x)
    if normalize:
        w = w / s
    elif abs(s - 1.0) > 1e-8:
        raise ValidationError("2D psf weights must sum to 1 (pass normalize)")
    sym = bool(np.all(w == w[::-1, :]) and np.all(w == w[:, ::-1]))
    return Psf2D(w, r // 2, c // 2, sym)


def separable_psf2d(a: Psf, b: Psf) -> Psf2D:
    """multidim.cpp:122-129."""
    return make_psf2d(np.outer(a.weights, b.weights), normalize=True)


def marginal_sum_columns(p: Psf2D) -> Psf:  # multidim.cpp:143-150
    return make_psf(np.array([sum(float(x) for x in row) for row in p.weights]), normalize=True)


def marginal_sum_rows(p: Psf2D) -> Psf:  # multidim.cpp:152-159
    return make_psf(np.array([sum(float(x) for x in col) for col in p.weights.T]),
                    normalize=True)


def eigenvalues_2d(p: Psf2D, n1, n2, bc, separable=False):
    """Three-step eigenvalue scheme (multidim.cpp:208-272).

    Interior: z2(x1_i, x2_j) by direct summation (real part for real bases);
    the separable factorisation e^{i(j t1 + k t2)} = e^{ij t1} e^{ik t2} turns
    it into E1^T H E2.  Edges from the marginal 1D masks; corners exactly 1.
    ``separable=True`` instead returns the outer product of the marginal 1D
    eigenvalues (equal for separable masks, test_multidim.cpp:106-123)."""
    a1, a2 = marginal_sum_columns(p), marginal_sum_rows(p)
    d1 = operator_eigenvalues(a1, n1, bc)
    d2 = operator_eigenvalues(a2, n2, bc)
    if separable:
        return np.outer(d1, d2)
    x1, x2 = eigenvalue_grid(bc, n1), eigenvalue_grid(bc, n2)
    j = np.arange(-p.m1, p.m1 + 1)
    k = np.arange(-p.m2, p.m2 + 1)
    e1 = np.exp(1j * np.outer(x1, j))  # n1 x rows
    e2 = np.exp(1j * np.outer(k, x2))  # cols x n2
    z = e1 @ p.weights @ e2
    d = z if is_complex_basis(bc) else z.real.copy()
    if is_boundary_corrected(bc):
        d[:, 0] = d1
        d[:, n2 - 1] = d1
        d[0, :] = d2
        d[n1 - 1, :] = d2
        d[0, 0] = d[0, n2 - 1] = d[n1 - 1, 0] = d[n1 - 1, n2 - 1] = 1
    if is_higher_order(bc):  # extension: the same scheme with k_l + k_r border lines
        kl, kr, _ = HO_BORDERS[bc]
        b1 = list(range(kl)) + list(range(n1 - kr, n1))
        b2 = list(range(kl)) + list(range(n2 - kr, n2))
        d[:, b2] = d1[:, None]
        d[b1, :] = d2[None, :]
        d[np.ix_(b1, b2)] = 1
    return d


def tensor_apply(rows: SpectralBasis, cols: SpectralBasis, arr, forward):
    """Columns first, then rows (multidim.cpp:172-198).  forward = synthesize."""
    arr = np.asarray(arr)
    t = np.swapaxes(arr, -1, -2)
    t = rows.synthesize(t) if forward else rows.analyze(t)
    t = np.swapaxes(t, -1, -2)
    return cols.synthesize(t) if forward else cols.analyze(t)


@dataclass
class BlurOperator2D:
    bc: int
    n1: int
    n2: int
    eigenvalues: np.ndarray
    rows: SpectralBasis
    cols: SpectralBasis

    @property
    def complex(self):
        return is_complex_basis(self.bc)

    def analyze(self, g):
        g = np.asarray(g, dtype=np.float64)
        return tensor_apply(self.rows, self.cols, g.astype(np.complex128) if self.complex else g,
                            forward=False)

    def synthesize(self, c):
        yc = tensor_apply(self.rows, self.cols, c, forward=True)
        if self.complex:
            return yc.real.copy(), np.sqrt(np.sum(yc.imag ** 2, axis=(-2, -1)))
        return yc, np.zeros(yc.shape[:-2])

    def apply(self, f):
        """multidim.cpp:278-304."""
        return self.synthesize(self.analyze(f) * self.eigenvalues)


def build_operator_2d(p: Psf2D, n1, n2, bc, separable=False) -> BlurOperator2D:
    """multidim.cpp:309-322 (validate_build_2d, multidim.cpp:15-26)."""
    if needs_symmetric_psf(bc) and not p.symmetric:
        raise ValidationError(f"{BC_NAMES[bc]} boundary conditions require a quadrantally "
                              "symmetric 2D psf")
    slack = 2 if is_boundary_corrected(bc) else 0
    if is_higher_order(bc):
        slack = HO_BORDERS[bc][0] + HO_BORDERS[bc][1]
        if min(n1, n2) < slack + 3:
            raise ValidationError("higher-order borders need n >= degree + 3 per axis")
    if is_boundary_corrected(bc) and (n1 < 5 or n2 < 5):
        raise ValidationError("boundary-corrected 2D operators need n >= 5 per axis")
    if 2 * p.m1 + 1 > n1 - slack or 2 * p.m2 + 1 > n2 - slack:
        raise ValidationError("2D psf support exceeds the per-axis limit")
    d = eigenvalues_2d(p, n1, n2, bc, separable)
    return BlurOperator2D(bc, n1, n2, d, SpectralBasis(bc, n1), SpectralBasis(bc, n2))


def smoothing_eigenvalues_2d(kind, bc, n1, n2, d=None):
    """multidim.cpp:329-356: identity -> 1, laplacian -> s(x1_i) + s(x2_j)."""
    if kind == IDENTITY:
        return np.ones((n1, n2))
    x1, x2 = eigenvalue_grid(bc, n1), eigenvalue_grid(bc, n2)
    s = (2.0 - 2.0 * np.cos(x1))[:, None] + (2.0 - 2.0 * np.cos(x2))[None, :]
    if d is not None and np.any((s == 0.0) & (np.abs(d) == 0.0)):
        raise ValidationError("incompatible smoother: joint null space")
    return s


def deblur_2d(op: BlurOperator2D, s, g, use_gcv=True, fixed_mu=0.0, mu_min=1e-12,
              mu_max=10.0, count=200, want_curve=False) -> Restoration:
    """deblur_2d (pipeline.cpp:157-165); batched over a leading axis."""
    g = np.asarray(g, dtype=np.float64)
    flat = g.reshape(-1, op.n1, op.n2)
    B = flat.shape[0]
    mus_used = np.empty(B)
    best = np.full(B, -1)
    curves = np.empty((B, count)) if want_curve else None
    out = np.empty_like(flat)
    res = np.empty(B)
    for b in range(B):
        ghat = op.analyze(flat[b])
        if use_gcv:
            r = _select_from_coeffs(op.eigenvalues, s, ghat, mu_min, mu_max, count)
            mus_used[b], best[b] = r.mu, r.best_k
            if want_curve:
                curves[b] = r.vals
        else:
            mus_used[b] = fixed_mu
        out[b], res[b] = op.synthesize(apply_tikhonov_filter(op.eigenvalues, s, mus_used[b],
                                                             ghat))
    shp = g.shape[:-2]
    return Restoration(out.reshape(g.shape), mus_used.reshape(shp), best.reshape(shp),
                       res.reshape(shp), curves)


# --------------------------------------------------------------------------
# Input generation (operators.cpp:78-90, 443-469; pipeline.cpp:15-51)
# --------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    """operators.cpp:78-85, vectorised over uint64 arrays."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def bits_to_u01(bits):
    """(0, 1] (operators.cpp:88-90)."""
    return ((np.asarray(bits, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) + 1.0) \
        * (2.0 ** -53)


def add_noise(g, level, seed):
    """g + eta, ||eta|| = level ||g|| (operators.cpp:332-358).  Last axis = signal;
    ``seed`` is a scalar or an array broadcast against the leading axes."""
    g = np.asarray(g, dtype=np.float64)
    if level < 0.0:
        raise ValidationError("noise level must be nonnegative")
    if level == 0.0 or g.shape[-1] == 0:
        return g.copy()
    n = g.shape[-1]
    pairs = (n + 1) // 2
    golden = np.uint64(0x9E3779B97F4A7C15)
    seed = np.asarray(seed, dtype=np.uint64)[..., None]
    p = np.arange(pairs, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u1 = bits_to_u01(splitmix64(seed + (np.uint64(2) * p + np.uint64(1)) * golden))
        u2 = bits_to_u01(splitmix64(seed + (np.uint64(2) * p + np.uint64(2)) * golden))
    r = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * PI * u2
    eta = np.empty(np.broadcast_shapes(seed.shape[:-1], g.shape[:-1]) + (2 * pairs,))
    eta[..., 0::2] = r * np.cos(ang)
    eta[..., 1::2] = r * np.sin(ang)
    eta = eta[..., :n]
    gnorm = np.sum(g * g, axis=-1, keepdims=True)
    enorm = np.sum(eta * eta, axis=-1, keepdims=True)
    scale = level * np.sqrt(gnorm / np.where(enorm == 0.0, 1.0, enorm))
    return g + np.where(enorm == 0.0, 0.0, scale) * eta


def convolve_valid(ext, psf: Psf):
    """g_i = sum_j h_j f_{i+j} (pipeline.cpp:15-29); last axis."""
    ext = np.asarray(ext, dtype=np.float64)
    m = psf.m
    n = ext.shape[-1] - 2 * m
    if n < 1:
        raise ValidationError("extended signal shorter than the psf support")
    g = np.zeros(ext.shape[:-1] + (n,))
    for j in range(-m, m + 1):
        g = g + psf.at(j) * ext[..., m + j:m + j + n]
    return g


def convolve_valid_2d(ext, p: Psf2D):
    """pipeline.cpp:31-51; last two axes."""
    ext = np.asarray(ext, dtype=np.float64)
    rows, cols = ext.shape[-2:]
    n1, n2 = rows - 2 * p.m1, cols - 2 * p.m2
    g = np.zeros(ext.shape[:-2] + (n1, n2))
    for j in range(-p.m1, p.m1 + 1):
        for l in range(-p.m2, p.m2 + 1):
            g = g + p.weights[p.m1 + j, p.m2 + l] * \
                ext[..., p.m1 + j:p.m1 + j + n1, p.m2 + l:p.m2 + l + n2]
    return g


def sweep_mu(op: BlurOperator, s, g, truth=None, mu_min=1e-12, mu_max=10.0, count=200):
    """sweep_mu (pipeline.cpp:55-115): GCV selection, then for every grid mu a
    Tikhonov solve and its rre; the first strict RRE minimum gives mu_opt.
    -> (mus, G, rre, [min_rre, mu_opt, mu_gcv, rre_gcv]) (NaN rre without truth)."""
    g = np.asarray(g, dtype=np.float64)
    r = gcv_select(op, s, g, mu_min, mu_max, count)
    mus = np.asarray(r.mus, dtype=np.float64)
    G = np.asarray(r.vals, dtype=np.float64)
    nan = float("nan")
    if truth is None:
        return mus, G, np.full(count, nan), np.array([nan, nan, r.mu, nan])
    t = np.asarray(truth, dtype=np.float64)
    if np.sum(t * t) == 0.0:
        raise ValidationError("rre: zero ground truth")
    rr = np.array([rre(t, tikhonov_solve(op, s, g, m)[0]) for m in mus])
    best, mu_opt = np.inf, mus[0]
    for k in range(count):
        if rr[k] < best:
            best, mu_opt = rr[k], mus[k]
    return mus, G, rr, np.array([best, mu_opt, r.mu, rre(t, tikhonov_solve(op, s, g, r.mu)[0])])


def rre(truth, restored):
    """regularize.cpp:249-260."""
    truth, restored = np.asarray(truth), np.asarray(restored)
    tn = np.sum(truth * truth, axis=-1)
    return np.sqrt(np.sum((truth - restored) ** 2, axis=-1) / tn)
