"""Dump GPU 1D hoc-cosine restorations at a fixed mu for offline comparison with an extended-precision reference."""
import sys, os, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0906_2704_b200 as P
from paper_0906_2704_b200 import workloads as W
os.makedirs(os.path.join(ROOT, "gpurun_out", "diag"), exist_ok=True)
rng = np.random.default_rng(1)
for n in (1024, 4096):
    x = np.linspace(0, 1, n)
    smooth = 0.3 + 0.5 * x - 0.4 * x * x + 0.3 * np.exp(-((x - 0.4) / 0.05) ** 2)
    y = smooth + 0.005 * rng.standard_normal((4, n))
    op = P.build_operator(W.gaussian_weights(12, 2.5), n, "hoc-cosine")
    L = P.smoothing_eigenvalues("laplacian", op)
    yd = torch.from_numpy(y).cuda()
    c = np.real(op.analyze(yd).cpu().numpy())
    f = P.tikhonov_solve(op, L, yd, 1e-6)
    f = (f[0] if isinstance(f, tuple) else f).cpu().numpy()
    np.savez(os.path.join(ROOT, "gpurun_out", "diag", f"hcf_{n}.npz"), y=y, c=c, f=f)
print("dumped")
