"""Diagnostic: single-image GCV paths on the GPU vs the reference (interior minimum)."""
import sys, os, dataclasses, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'oracle'))
import reflib as R
import paper_0906_2704_b200 as P
from paper_0906_2704_b200 import workloads as W
for sigma, lo, sm in [(2.5, 1e-14, 1), (1.0, 1e-14, 1)]:
    cfg = dataclasses.replace(W.config(2), psf=W.gaussian_weights(6, sigma))
    _, g = W.image_2d(cfg, 7, 1024, 1024)
    p2 = np.outer(cfg.psf, cfg.psf); p2 /= p2.sum()
    out, mu, curve, _ = R.deblur_2d(p2, cfg.bc, sm, g, True, mu_min=lo, mu_max=1.0, count=128,
                                    eig_mode=1, threads=8, want_curve=True)
    k = int(np.argmin(curve[0]))
    print("REF", sigma, lo, sm, "k", k, "mu", mu[0], "G", curve[0][k])
    op = P.build_operator_2d_separable(cfg.psf, cfg.psf, 1024, 1024, cfg.bc)
    L = P.smoothing_eigenvalues(["identity", "laplacian"][sm], op)
    gd = torch.from_numpy(g).cuda()
    search = P.GcvSearch(lo, 1.0, 128)
    for scr in ("1", "0"):
        os.environ["FASTDEBLUR_GCV_SCREEN"] = scr
        for wc in (False, True):
            rep = P.deblur(op, L, gd, P.MuChoice(True), search=search, want_curve=wc)
            torch.cuda.synchronize()
            m = float(rep.mu_used.cpu().reshape(-1)[0]); bk = int(rep.best_k.cpu().reshape(-1)[0])
            print("  screen", scr, "curve", wc, "k", bk, "mu", m, "mu/ref-1", m / mu[0] - 1)
            if wc:
                c = rep.gcv_curve.cpu().numpy().reshape(-1)
                print("     curve rel err max", np.max(np.abs(c / curve[0] - 1)))
    for mm in (mu[0], search.mu_min * np.exp(k * np.log(1.0 / lo) / 127)):
        print("  G_gpu(", mm, ") =", float(P.gcv_value(op, L, gd, mm).cpu().reshape(-1)[0]))
