import sys, numpy as np, torch
sys.path[:0] = ['.', 'oracle', 'tests']
import fdoracle as O
from paper_0906_2704_b200 import fastdeblur as P
from util import rel, np_, gauss
rng = np.random.default_rng(1)
for bc in (O.HOC_COSINE, O.REFLECTIVE, O.PERIODIC, O.HOC_FOURIER):
    for n in (2048, 4096, 8192, 8194, 12000, 16384):
        psf = gauss(16, 4.0)
        op = P.build_operator(psf, n, bc)
        oop = O.build_operator(O.make_psf(psf, True), n, bc)
        b = oop.basis
        x = rng.standard_normal((2, n))
        got = np_(op.analyze(torch.from_numpy(x)))
        want = b.analyze(x.astype(complex) if b.complex else x)
        c = rng.standard_normal((2, n))
        ms = ''
        if not b.complex:
            ms = '%.2e' % rel(np_(op.synthesize(torch.from_numpy(c))[0]), b.synthesize(c))
        ap = rel(np_(op.apply(torch.from_numpy(x))[0]), oop.apply(x)[0])
        print(bc, n, 'analyze %.2e' % rel(got, want), 'synth', ms, 'apply %.2e' % ap, flush=True)
