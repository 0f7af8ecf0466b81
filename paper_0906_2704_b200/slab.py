"""One 2D image split into row slabs across ranks.

A rank holds rows [r0, r0 + R) of an n1 x n2 image (R = n1 / P).  The
restoration is the reference's deblur_2d (pipeline.cpp:157-165: gcv_select_2d +
tikhonov_solve_2d, multidim.cpp:358-442) with the data movement of SURVEY 8e:

    rows analyze (local, axis 2)
      -> all-to-all transpose to column slabs (C = n2 / P columns, as lines)
    columns analyze (axis 1) -> GCV partial sums -> all-reduce (2 K fp64)
      -> selection on the sums (identical on every rank; moments all-reduced)
    filtered columns synthesis -> all-to-all back -> rows synthesis

The only collectives are the two transposes and the fp64 sum reductions; the
selection (first minimum, 1e-12 ties, golden section) runs on the reduced sums
with the same code as the single-GPU path.  Rows-then-columns equals
tensor_apply's columns-then-rows up to rounding.

`Comm` implementations: `TorchComm` (torch.distributed: NCCL over NVLink on the
GPUs, gloo on CPU) and `ThreadComm` (P ranks as threads of one process: the
single-GPU correctness harness -- the exchange is host-side, no kernel waits on
another).  Backends: `GpuSlabBackend` (the CUDA library); tests plug the numpy
oracle in through the same interface.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import fastdeblur as P


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
class TorchComm:
    """torch.distributed group (one process per GPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_to_all(self, send: torch.Tensor) -> torch.Tensor:
        """send[p] goes to rank p; returns recv[q] = what rank q sent here."""
        send = send.contiguous()
        recv = torch.empty_like(send)
        self.dist.all_to_all_single(recv, send, group=self.group)
        return recv

    def all_reduce_sum(self, x: np.ndarray) -> np.ndarray:
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()


class ThreadComm:
    """P ranks as threads of one process; `view(rank)` is each rank's Comm.
    Sums are taken in rank order (deterministic)."""

    def __init__(self, world: int):
        self.world = world
        self._barrier = threading.Barrier(world)
        self._slots = [None] * world

    def view(self, rank: int):
        return _ThreadRank(self, rank)

    def run(self, fn):
        """fn(comm_view) on every rank in parallel; returns the per-rank results."""
        out, errs = [None] * self.world, []

        def body(r):
            try:
                out[r] = fn(self.view(r))
            except BaseException as e:  # noqa: BLE001
                errs.append(e)
                self._barrier.abort()

        th = [threading.Thread(target=body, args=(r,)) for r in range(self.world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        return out


class _ThreadRank:
    def __init__(self, c: ThreadComm, rank: int):
        self.c, self.rank, self.world = c, rank, c.world

    def _exchange(self, x):
        self.c._slots[self.rank] = x
        self.c._barrier.wait()
        got = list(self.c._slots)
        self.c._barrier.wait()
        return got

    def all_to_all(self, send):
        got = self._exchange(send)
        parts = [got[q][self.rank] for q in range(self.world)]
        return torch.stack(parts) if isinstance(send, torch.Tensor) else np.stack(parts)

    def all_reduce_sum(self, x):
        got = self._exchange(np.asarray(x, dtype=np.float64))
        s = got[0].copy()
        for q in range(1, self.world):
            s = s + got[q]
        return s


# ---------------------------------------------------------------------------
# transposes between row slabs [R, n2, *t] and column slabs [C, n1, *t]
# ---------------------------------------------------------------------------
def _perm(x, order):
    return x.permute(*order) if isinstance(x, torch.Tensor) else np.transpose(x, order)


def _contig(x):
    return x.contiguous() if isinstance(x, torch.Tensor) else np.ascontiguousarray(x)


def rows_to_cols(comm, a, n1, n2):
    Pw = comm.world
    R, Cc = n1 // Pw, n2 // Pw
    tail = tuple(a.shape[2:])
    t = tuple(range(3, 3 + len(tail)))
    send = _contig(_perm(a.reshape((R, Pw, Cc) + tail), (1, 0, 2) + t))  # [P, R, C, *t]
    recv = comm.all_to_all(send)                                       # [src, R, C, *t]
    return _contig(_perm(recv, (2, 0, 1) + t)).reshape((Cc, n1) + tail)


def cols_to_rows(comm, f, n1, n2):
    Pw = comm.world
    R, Cc = n1 // Pw, n2 // Pw
    tail = tuple(f.shape[2:])
    t = tuple(range(3, 3 + len(tail)))
    send = _contig(_perm(f.reshape((Cc, Pw, R) + tail), (1, 2, 0) + t))  # [P, R, C, *t]
    recv = comm.all_to_all(send)                                        # [src, R, C, *t]
    return _contig(_perm(recv, (1, 0, 2) + t)).reshape((R, n2) + tail)


# ---------------------------------------------------------------------------
# selection on reduced sums (the library's host code: fd_gcv_core.h)
# ---------------------------------------------------------------------------
def moment_terms(search):
    J = C.c_int()
    P.check(P.lib().fd_gcv_moment_terms(C.c_double(search.mu_min), C.c_double(search.mu_max),
                                        search.count, C.byref(J)))
    return J.value


def pick_from_sums(num_den, search):
    K = search.count
    nd = np.ascontiguousarray(num_den, dtype=np.float64)
    G = np.empty(K)
    bk, need = C.c_int(), C.c_int()
    center, mu = C.c_double(), C.c_double()
    dp = C.POINTER(C.c_double)
    P.check(P.lib().fd_gcv_pick_from_sums(nd.ctypes.data_as(dp), C.c_double(search.mu_min),
                                          C.c_double(search.mu_max), K, G.ctypes.data_as(dp),
                                          C.byref(bk), C.byref(need), C.byref(center),
                                          C.byref(mu)))
    return G, bk.value, bool(need.value), center.value, mu.value


def golden_from_moments(mom, J, center, best_G, best_k, search):
    m = np.ascontiguousarray(mom, dtype=np.float64)
    mu = C.c_double()
    P.check(P.lib().fd_gcv_golden_from_moments(
        m.ctypes.data_as(C.POINTER(C.c_double)), J, C.c_double(center), C.c_double(best_G),
        C.c_double(search.mu_min), C.c_double(search.mu_max), search.count, best_k,
        C.byref(mu)))
    return mu.value


def golden_direct(G_of, best_k, best_G, search):
    """Coarse grids (no moment series): the golden section of gcv_minimize
    (regularize.cpp:187-213, fd_gcv_core.h gcv_golden) with G evaluated on the
    reduced partial sums."""
    mus = np.exp(np.log(search.mu_min) + (np.log(search.mu_max) - np.log(search.mu_min)) *
                 np.arange(search.count) / (search.count - 1))
    K = search.count
    lo, hi = mus[best_k - 1 if best_k > 0 else 0], mus[best_k + 1 if best_k + 1 < K else K - 1]
    a, b = math.log(lo), math.log(hi)
    invphi = 0.6180339887498949
    x1, x2 = b - invphi * (b - a), a + invphi * (b - a)
    f1, f2 = G_of(math.exp(x1)), G_of(math.exp(x2))
    while math.exp(b - a) - 1.0 > 1e-3:
        if f1 <= f2:
            b, x2, f2 = x2, x1, f1
            x1 = b - invphi * (b - a)
            f1 = G_of(math.exp(x1))
        else:
            a, x1, f1 = x1, x2, f2
            x2 = a + invphi * (b - a)
            f2 = G_of(math.exp(x2))
    refined = math.exp(0.5 * (a + b))
    return refined if G_of(refined) <= best_G else float(mus[best_k])


# ---------------------------------------------------------------------------
# the distributed restoration
# ---------------------------------------------------------------------------
@dataclass
class SlabResult:
    restored: object  # this rank's rows [R, n2]
    mu: float
    best_k: int


def deblur_2d_slabs(backend, comm, g_rows, n1, n2, search) -> SlabResult:
    """deblur_2d with GCV (pipeline.cpp:157-165) of one image whose rows are
    spread over `comm`; g_rows = this rank's rows [n1/P, n2]."""
    Pw = comm.world
    if n1 % Pw or n2 % Pw:
        raise P.ValidationError(f"image {n1}x{n2} does not split evenly over {Pw} ranks")
    Cc = n2 // Pw
    col0 = comm.rank * Cc
    a = backend.row_analyze(g_rows)                  # [R, n2, *t]
    ghat = backend.col_analyze(rows_to_cols(comm, a, n1, n2))  # [C, n1, *t]
    nd = comm.all_reduce_sum(backend.gcv_partials(ghat, col0, search))
    G, best_k, need, center, mu = pick_from_sums(nd, search)
    if need:
        J = moment_terms(search)
        if J > 0:
            mom = comm.all_reduce_sum(backend.gcv_moments(ghat, col0, center, J))
            mu = golden_from_moments(mom, J, center, G[best_k], best_k, search)
        else:
            def G_of(m):
                s = comm.all_reduce_sum(backend.gcv_partials(ghat, col0, search, mus=[m]))
                return s[0] / (s[1] * s[1])
            mu = golden_direct(G_of, best_k, G[best_k], search)
    f = backend.col_synth(ghat, col0, mu)             # [C, n1, *t]
    rows = backend.row_synth(cols_to_rows(comm, f, n1, n2))
    return SlabResult(rows, mu, best_k)


class GpuSlabBackend:
    """Per-rank slab passes on the GPU (fd_slab_* of the C ABI)."""

    def __init__(self, op, L):
        self.op, self.L = op, L
        self.n1, self.n2 = op.n1, op.n2
        self.cplx = op.complex

    def _lines(self, shape, device):
        if self.cplx:
            return torch.empty(shape + (2,), dtype=torch.float64, device=device)
        return torch.empty(shape, dtype=torch.float64, device=device)

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def row_analyze(self, rows):
        rows = rows.contiguous()
        out = self._lines(tuple(rows.shape[:2]), rows.device)
        P.check(P.lib().fd_slab_analyze(self.op._h, 2, C.c_void_p(rows.data_ptr()), 0,
                                        C.c_void_p(out.data_ptr()), rows.shape[0],
                                        self._stream()))
        return out

    def col_analyze(self, cols):
        cols = cols.contiguous()
        out = self._lines(tuple(cols.shape[:2]), cols.device)
        P.check(P.lib().fd_slab_analyze(self.op._h, 1, C.c_void_p(cols.data_ptr()),
                                        1 if self.cplx else 0, C.c_void_p(out.data_ptr()),
                                        cols.shape[0], self._stream()))
        return out

    def gcv_partials(self, ghat, col0, search, mus=None):
        K = search.count if mus is None else len(mus)
        out = np.empty(2 * K)
        dp = C.POINTER(C.c_double)
        mu_arr = None if mus is None else np.ascontiguousarray(mus, dtype=np.float64)
        P.check(P.lib().fd_slab_gcv_partials(
            self.op._h, self.L._h, C.c_void_p(ghat.data_ptr()), ghat.shape[0], col0,
            C.c_double(search.mu_min), C.c_double(search.mu_max), K,
            None if mu_arr is None else mu_arr.ctypes.data_as(dp), out.ctypes.data_as(dp),
            self._stream()))
        return out

    def gcv_moments(self, ghat, col0, center, J):
        out = np.empty(2 * J)
        P.check(P.lib().fd_slab_gcv_moments(
            self.op._h, self.L._h, C.c_void_p(ghat.data_ptr()), ghat.shape[0], col0,
            C.c_double(center), J, out.ctypes.data_as(C.POINTER(C.c_double)), self._stream()))
        return out

    def col_synth(self, ghat, col0, mu):
        out = torch.empty_like(ghat)
        P.check(P.lib().fd_slab_synthesize(self.op._h, self.L._h, 1, C.c_void_p(ghat.data_ptr()),
                                           C.c_void_p(out.data_ptr()), 1 if self.cplx else 0,
                                           ghat.shape[0], col0, C.c_double(mu), self._stream()))
        return out

    def row_synth(self, rows):
        rows = rows.contiguous()
        out = torch.empty(tuple(rows.shape[:2]), dtype=torch.float64, device=rows.device)
        P.check(P.lib().fd_slab_synthesize(self.op._h, None, 2, C.c_void_p(rows.data_ptr()),
                                           C.c_void_p(out.data_ptr()), 0, rows.shape[0], 0,
                                           C.c_double(0.0), self._stream()))
        return out
