import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import fdoracle as O, paper_0906_2704_b200 as P
from util import onesided, gauss, np_, rel
a, b = onesided(3, 0.5), onesided(2, 0.3)
psf2 = np.outer(a, b)
rng = np.random.default_rng(1)
for n1, n2 in ((14, 18), (15, 18), (14, 19)):
    f = rng.standard_normal((n1, n2))
    for bc in (O.PERIODIC, O.HOC_FOURIER, O.HOC_FOURIER_D3):
        for sep in (True, False):
            op = P.build_operator_2d_separable(a, b, n1, n2, bc) if sep else P.build_operator_2d(psf2, n1, n2, bc)
            p = O.make_psf2d(psf2, normalize=True)
            oop = O.build_operator_2d(p, n1, n2, bc, separable=sep)
            for smn, sm in (("identity", O.IDENTITY), ("laplacian", O.LAPLACIAN)):
                L = P.smoothing_eigenvalues(smn, op)
                s = O.smoothing_eigenvalues_2d(sm, bc, n1, n2, oop.eigenvalues)
                G = float(np_(P.gcv_value(op, L, torch.from_numpy(f), 1e-3)))
                Go = float(O.gcv_value(oop, s, f, 1e-3)) if hasattr(O, "gcv_value_2d") else None
                # oracle 2d gcv via coefficients
                gh = oop.analyze(f)
                Go = float(O.gcv_from_coeffs(oop.eigenvalues, s, gh, 1e-3))
                fr, _ = P.tikhonov_solve(op, L, torch.from_numpy(f), torch.tensor([1e-3], dtype=torch.float64))
                print((n1, n2), O.BC_NAMES[bc], "sep" if sep else "gen", smn, "G rel %.2e" % abs(G / Go - 1))
