"""Row-slab restoration of one 2D image over a real torch.distributed group
(gloo, world 2, CPU) with the numpy oracle as the per-rank compute:
the transposes, the summed GCV partials and moments and the selection on the
sums give the oracle's whole-image deblur_2d (pipeline.cpp:157-165)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleSlabBackend:
    """The slab passes restated in numpy (fdoracle), torch CPU tensors out;
    complex coefficients as [..., 2] doubles like the GPU backend."""

    def __init__(self, oop, s):
        self.oop, self.s = oop, s
        self.d = oop.eigenvalues

    @staticmethod
    def _t(a):
        a = np.ascontiguousarray(a)
        if np.iscomplexobj(a):
            a = np.stack([a.real, a.imag], axis=-1)
        return torch.from_numpy(np.ascontiguousarray(a))

    @staticmethod
    def _np(t):
        a = t.numpy()
        return a[..., 0] + 1j * a[..., 1] if a.ndim == 3 else a

    def row_analyze(self, rows):
        x = self._np(rows)
        return self._t(self.oop.cols.analyze(x.astype(complex) if self.oop.complex else x))

    def col_analyze(self, cols):
        return self._t(self.oop.rows.analyze(self._np(cols)))

    def _slab(self, col0, C):
        return self.d[:, col0:col0 + C].T, self.s[:, col0:col0 + C].T

    def gcv_partials(self, ghat, col0, search, mus=None):
        import fdoracle as O
        gh = self._np(ghat)
        d, s = self._slab(col0, gh.shape[0])
        if mus is None:
            mus = O.gcv_grid(search.mu_min, search.mu_max, search.count)
        ok = s != 0
        r = (np.abs(d) ** 2 / np.where(ok, s, 1) ** 2)[ok]
        w = (np.abs(gh) ** 2)[ok]
        num = [np.sum(w / (r + m) ** 2) for m in mus]
        den = [np.sum(1.0 / (r + m)) for m in mus]
        return np.array(num + den)

    def gcv_moments(self, ghat, col0, center, J):
        gh = self._np(ghat)
        d, s = self._slab(col0, gh.shape[0])
        ok = s != 0
        t = center / ((np.abs(d) ** 2 / np.where(ok, s, 1) ** 2)[ok] + center)  # scaled series
        w = (np.abs(gh) ** 2)[ok]
        A = [np.sum(w * t ** (j + 2)) for j in range(J)]
        B = [np.sum(t ** (j + 1)) for j in range(J)]
        return np.array(A + B)

    def col_synth(self, ghat, col0, mu):
        gh = self._np(ghat)
        d, s = self._slab(col0, gh.shape[0])
        f = gh * np.conj(d) / (np.abs(d) ** 2 + mu * s * s)
        return self._t(self.oop.rows.synthesize(f if self.oop.complex else f.real))

    def row_synth(self, rows):
        y = self.oop.cols.synthesize(self._np(rows))
        return torch.from_numpy(np.ascontiguousarray(np.real(y)))


def _worker(rank, world, port, q, bc):
    sys.path[:0] = [os.path.join(HERE, ".."), os.path.join(HERE, "..", "oracle"), HERE]
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import fdoracle as O
    from paper_0906_2704_b200 import dist, slab
    from paper_0906_2704_b200 import fastdeblur as P
    from paper_0906_2704_b200 import workloads as W
    from util import gauss, onesided
    dist.init(backend="gloo")
    n1, n2 = 48, 64
    psf = gauss(4, 1.5) if bc == O.HOC_COSINE else onesided(5, 0.3)
    p1 = O.make_psf(psf, True)
    oop = O.build_operator_2d(O.separable_psf2d(p1, p1), n1, n2, bc, separable=True)
    s = O.smoothing_eigenvalues_2d(O.LAPLACIAN, bc, n1, n2)
    _, g = W.image_2d(W.config(2), 0, n1, n2)
    R = n1 // world
    search = P.GcvSearch(1e-6, 1.0, 64)
    res = slab.deblur_2d_slabs(OracleSlabBackend(oop, s), slab.TorchComm(),
                               torch.from_numpy(g[rank * R:(rank + 1) * R].copy()), n1, n2,
                               search)
    full = [torch.empty(R, n2, dtype=torch.float64) for _ in range(world)]
    torch.distributed.all_gather(full, res.restored)
    if rank == 0:
        want = O.deblur_2d(oop, s, g, True, mu_min=1e-6, mu_max=1.0, count=64)
        q.put((res.best_k, res.mu, torch.cat(full).numpy(), int(want.best_k),
               float(want.mu_used), want.restored))
    dist.finalize()


@pytest.mark.parametrize("bc", [3, 4])  # hoc-cosine, hoc-fourier
def test_slab_gloo_world2(bc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, bc)) for r in range(2)]
    for p in procs:
        p.start()
    bk, mu, rest, wbk, wmu, wrest = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert bk == wbk
    assert abs(mu / wmu - 1) < 1e-10
    assert np.linalg.norm(rest - wrest) / np.linalg.norm(wrest) < 1e-10
