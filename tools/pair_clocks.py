"""Phase split of the line-pair kernels on config 1 at d = 3 (timing build):
    python -c "from paper_0906_2704_b200.build import build_library as b; \
               b(out='paper_0906_2704_b200/libfdb200_clk.so', defines=['FD_PHASE_CLOCKS'])"
    FASTDEBLUR_LIB=paper_0906_2704_b200/libfdb200_clk.so python tools/pair_clocks.py
Run once per FASTDEBLUR_PAIR_EDGE setting.  SM clocks of thread 0 between the
CTA barriers that end each phase, per line pair."""
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
op = P.build_operator(cfg.psf, cfg.n1, "hoc-fourier-d3")
L = P.smoothing_eigenvalues("first-difference", op)
gd = torch.from_numpy(g).cuda()
search = P.GcvSearch(cfg.mu_min, cfg.mu_max, cfg.count)
out = (C.c_ulonglong * 48)()
for _ in range(2):
    P.deblur(op, L, gd, P.MuChoice(True), search=search)
torch.cuda.synchronize()
P.lib().fd_pair_clocks(out, 1)
R = 5
for _ in range(R):
    P.deblur(op, L, gd, P.MuChoice(True), search=search)
torch.cuda.synchronize()
P.lib().fd_pair_clocks(out, 0)
v = np.array(list(out), dtype=np.float64).reshape(4, 12) / (R * B / 2)
names = {0: ["load", "fold", "DIF1", "DIF2", "mid", "DIT2", "DIT1", "combine", "post"],
         1: ["load", "fold", "DIF1", "DIF2", "mid", "DIT2", "DIT1", "combine", "post"],
         2: ["load", "-", "first", "DIF2", "mid", "DIT2", "last", "Zxchg", "post"],
         3: ["load", "xchg", "first", "DIF2", "mid", "DIT2", "last", "-", "post"]}
for k, kn in enumerate(("k_panalyze", "k_psynth", "k_panalyze_e", "k_psynth_e")):
    if v[k].sum() == 0:
        continue
    print(kn, "clocks/pair %.0f:" % v[k].sum(),
          "  ".join("%s %.0f" % (names[k][i], v[k, i]) for i in range(9)))
