"""Small line-pair restorations (n = 4096, d = 1 and d = 3, odd batch): a driver
for compute-sanitizer where it is available
    compute-sanitizer --tool racecheck python tools/sanitize_pairs.py
(closed on the measurement pool; tests/test_gpu_edges.py checks run-to-run
bit-identity of the same kernels instead)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_0906_2704_b200 import fastdeblur as P  # noqa: E402
from paper_0906_2704_b200 import workloads as W  # noqa: E402

cfg = W.config(1)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 37
_, g = W.signals_1d(cfg, 0, B)
gd = torch.from_numpy(g).cuda()
for bc in ("hoc-fourier-d1", "hoc-fourier-d3"):
    op = P.build_operator(cfg.psf, cfg.n1, bc)
    L = P.smoothing_eigenvalues("first-difference", op)
    rep = P.deblur(op, L, gd, P.MuChoice(True), search=P.GcvSearch(cfg.mu_min, cfg.mu_max, cfg.count))
    torch.cuda.synchronize()
    print(bc, float(rep.restored.abs().sum()), int(rep.best_k.min()), int(rep.best_k.max()))
