import sys, os, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'oracle'))
import fdoracle as O
import paper_0906_2704_b200 as P
rng = np.random.default_rng(0)
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
for n in (142, 422, 16382):
    op = P.build_operator([1.0], n, "reflective")
    b = O.SpectralBasis(O.REFLECTIVE, n)
    x = rng.standard_normal((3, n))
    got = op.analyze(torch.from_numpy(x).cuda()).cpu().numpy()
    want = b.analyze(x)
    print(n, "analyze rel", rel(got, want), got[0, :4], want[0, :4])
    c = rng.standard_normal((3, n))
    gs = op.synthesize(torch.from_numpy(c).cuda())
    gs = (gs[0] if isinstance(gs, tuple) else gs).cpu().numpy()
    print(n, "synth rel", rel(gs, b.synthesize(c)))
