"""Diagnostic: coefficient-level accuracy of the GPU transforms vs numpy oracle / reference."""
import sys, os, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'oracle'))
import fdoracle as O
import paper_0906_2704_b200 as P
from paper_0906_2704_b200 import workloads as W
rng = np.random.default_rng(1)
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
for n in (1024, 4096):
    for bc, obc in (("hoc-cosine", O.HOC_COSINE),):
        psf = W.gaussian_weights(12, 2.5)
        op = P.build_operator(psf, n, bc)
        oop = O.build_operator(O.make_psf(psf, True), n, obc)
        x = np.linspace(0, 1, n)
        smooth = 0.3 + 0.5 * x - 0.4 * x * x + 0.3 * np.exp(-((x - 0.4) / 0.05) ** 2)
        for name, y in (("white", rng.standard_normal((8, n))), ("smooth+1%", smooth + 0.005 * rng.standard_normal((8, n)))):
            c = op.analyze(torch.from_numpy(y).cuda()).cpu().numpy()
            c = np.real(c)
            co = np.real(O.SpectralBasis(obc, n).analyze(y))
            e = c - co
            print(n, bc, name, "rel coef err", rel(c, co), "border err", np.abs(e[:, [0, -1]]).max(), "interior max", np.abs(e[:, 1:-1]).max(),
                  "coef norm", np.linalg.norm(co) / np.sqrt(8))
            # error spectrum: rms over items in 8 bands
            bands = np.array_split(np.arange(1, n - 1), 8)
            print("    band rms err", ["%.1e" % np.sqrt(np.mean(e[:, b] ** 2)) for b in bands])
            # mpmath-free check: which is closer to a float128 DCT? use longdouble direct transform of the oracle formula
