"""Row-slab distribution of one 2D image on the GPU: P ranks
simulated by threads of one process (ThreadComm: the exchange is host-side, no
kernel waits on another), against the single-GPU deblur of the whole image:
identical best_k, mu and restorations to 1e-10."""
import numpy as np
import pytest
import torch

import paper_0906_2704_b200 as P
from paper_0906_2704_b200 import slab
from paper_0906_2704_b200 import workloads as W
from util import gauss, onesided, rel

pytestmark = pytest.mark.gpu


def image(n1, n2, item=0):
    cfg = W.config(2)
    _, g = W.image_2d(cfg, item, n1, n2)
    return g


@pytest.mark.parametrize("bc,psf,smoother,search,world", [
    ("hoc-cosine", gauss(6, 2.0), "laplacian", (1e-6, 1.0, 128), 1),
    ("hoc-cosine", gauss(6, 2.0), "laplacian", (1e-6, 1.0, 128), 2),
    ("hoc-cosine", gauss(6, 2.0), "laplacian", (1e-6, 1.0, 128), 4),
    ("hoc-cosine", gauss(4, 1.5), "identity", (1e-8, 1.0, 64), 4),
    ("hoc-fourier", onesided(7, 0.25), "laplacian", (1e-6, 1.0, 128), 2),
    ("reflective", gauss(4, 1.5), "laplacian", (1e-6, 1.0, 7), 2),
    # config 4's grid (moment count J = 13) and config 1's (J = 17): the slab
    # moment entry point must accept every count the kernels are built for
    ("hoc-cosine", gauss(6, 2.0), "laplacian", (1e-8, 1.0, 512), 2),
    ("hoc-cosine", gauss(6, 2.0), "laplacian", (1e-8, 1.0, 256), 2),
])
def test_slab_deblur_matches_single_gpu(bc, psf, smoother, search, world):
    n1, n2 = 192, 256
    op = P.build_operator_2d_separable(psf, psf, n1, n2, bc)
    L = P.smoothing_eigenvalues(smoother, op)
    g = image(n1, n2)
    sr = P.GcvSearch(*search)
    ref = P.deblur(op, L, torch.from_numpy(g).cuda(), P.MuChoice(True), search=sr)
    gd = torch.from_numpy(g).cuda()
    R = n1 // world
    backend = slab.GpuSlabBackend(op, L)
    comm = slab.ThreadComm(world)
    res = comm.run(lambda c: slab.deblur_2d_slabs(backend, c, gd[c.rank * R:(c.rank + 1) * R],
                                                  n1, n2, sr))
    restored = torch.cat([r.restored for r in res]).cpu().numpy()
    assert all(r.best_k == int(ref.best_k.cpu()) for r in res)
    assert all(r.mu == res[0].mu for r in res)
    assert abs(res[0].mu / float(ref.mu_used.cpu()) - 1) < 1e-10
    assert rel(restored, ref.restored.cpu().numpy()) < 1e-10


def test_slab_uneven_split_rejected():
    op = P.build_operator_2d_separable(gauss(2, 1.0), gauss(2, 1.0), 30, 32, "hoc-cosine")
    L = P.smoothing_eigenvalues("laplacian", op)
    comm = slab.ThreadComm(4)
    with pytest.raises(P.ValidationError):
        comm.run(lambda c: slab.deblur_2d_slabs(slab.GpuSlabBackend(op, L), c,
                                                torch.zeros(7, 32, dtype=torch.float64,
                                                            device="cuda"),
                                                30, 32, P.GcvSearch(1e-6, 1.0, 16)))
