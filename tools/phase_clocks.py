"""Phase split of the real-line kernels on config 1 (timing build of the library):
    python -c "from paper_0906_2704_b200.build import build_library as b; \
               b(out='paper_0906_2704_b200/libfdb200_clk.so', defines=['FD_PHASE_CLOCKS'])"
    FASTDEBLUR_LIB=paper_0906_2704_b200/libfdb200_clk.so python tools/phase_clocks.py
Clocks are summed over CTAs (thread 0 of each), so the split, not the total, is
the result."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_0906_2704_b200 import fastdeblur as P  # noqa: E402
from paper_0906_2704_b200 import workloads as W  # noqa: E402

cfg = W.config(1)
B = 16384
_, g = W.signals_1d(cfg, 0, B)
op = P.build_operator(cfg.psf, cfg.n1, cfg.bc)
L = P.smoothing_eigenvalues("first-difference", op)
gd = torch.from_numpy(g).cuda()
search = P.GcvSearch(cfg.mu_min, cfg.mu_max, cfg.count)
out = (C.c_ulonglong * 8)()
for _ in range(2):
    P.deblur(op, L, gd, P.MuChoice(True), search=search)
torch.cuda.synchronize()
P.lib().fd_phase_clocks(out, 1)
for _ in range(5):
    P.deblur(op, L, gd, P.MuChoice(True), search=search)
torch.cuda.synchronize()
P.lib().fd_phase_clocks(out, 0)
v = np.array(list(out), dtype=np.float64).reshape(2, 4)
for k, name in enumerate(("k_ranalyze", "k_rsynth")):
    t = v[k, :3].sum()
    print(name, "load %.1f%% (staging wait %.1f%%)  convolution %.1f%%  post %.1f%%"
          % (100 * v[k, 0] / t, 100 * v[k, 3] / t, 100 * v[k, 1] / t, 100 * v[k, 2] / t),
          " clocks/line %.0f" % (t / (5 * B)))
