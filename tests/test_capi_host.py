"""CPU tests of the C ABI: the library loads, exports every symbol the header
declares, validates arguments with the reference's error codes before touching
the device, and its host copy of the gcv_minimize selection logic (the same
__host__ __device__ code the kernels run) matches the reference."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import fdoracle as O
import paper_0906_2704_b200 as P
import reflib as R
from paper_0906_2704_b200 import fastdeblur as FD

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                   "fastdeblur_b200.h")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fd_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    lib = FD.lib()
    names = declared()
    assert len(names) >= 20
    for nm in names:
        assert hasattr(lib, nm), nm


def test_header_cites_reference_interfaces():
    src = open(HDR).read()
    for ref in ("operators.cpp:293-301", "boundary.cpp:253-289", "regularize.cpp:144-214",
                "pipeline.cpp:120-165", "multidim.cpp:309-322"):
        assert ref in src


@pytest.mark.parametrize("call", [
    lambda: P.build_operator([0.5, 0.5], 16, "hoc-cosine"),                # even length
    lambda: P.build_operator([0.6, 0.3, 0.1], 32, "hoc-cosine"),           # nonsymmetric
    lambda: P.build_operator([0.6, 0.3, 0.1], 32, "reflective"),
    lambda: P.build_operator([0.6, 0.3, 0.1], 32, "antireflective"),
    lambda: P.build_operator(np.ones(17), 18, "hoc-cosine"),               # support > n-2
    lambda: P.build_operator(np.ones(17), 16, "periodic"),                 # support > n
    lambda: P.build_operator([1.0], 4, "hoc-cosine"),                      # n < 5
    lambda: P.build_operator([0.3, 0.3, 0.3], 16, "periodic", normalize=False),  # sum != 1
    lambda: P.build_operator([0.5, float("nan"), 0.5], 16, "periodic"),
    lambda: P.build_operator([1.0], 16, "no-such-bc"),
    lambda: P.build_operator_2d(np.ones((2, 3)), 16, 16, "periodic"),      # even rows
    lambda: P.build_operator_2d(np.outer([0.1, 0.9, 0.0], [1, 1, 1]), 16, 16, "hoc-cosine"),
    lambda: P.bc_for_degree(4, True),
    lambda: P.bc_for_degree(0, False),
    lambda: P.build_operator([0.1, 0.2, 0.4, 0.2, 0.1], 7, "hoc-fourier-d3"),  # support > n-3
    lambda: P.build_operator([1.0], 3, "hoc-fourier-d1"),                  # n < d+3
])
def test_validation_errors_match_reference(call):
    """operators.cpp:62-76, psf.cpp:10-37, multidim.cpp:15-26 (status 2)."""
    with pytest.raises(P.ValidationError):
        call()


def test_bc_mapping():
    assert P.bc_for_degree(2, True) == "hoc-cosine"
    assert P.bc_for_degree(2, False) == "hoc-fourier"
    assert P.bc_for_degree(1, True) == "antireflective"
    assert P.bc_for_degree(1, False) == "hoc-fourier-d1"  # extensions
    assert P.bc_for_degree(3, False) == "hoc-fourier-d3"
    assert P.bc_for_degree(3, True) == "hoc-fourier-d3"
    lib = FD.lib()
    for name, code in P.BC.items():
        assert lib.fd_parse_bc(name.encode()) == code
    assert lib.fd_parse_bc(b"bogus") == -1


GCV_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)


def host_minimize(G, mu_min, mu_max, count):
    lib = FD.lib()
    lib.fd_gcv_minimize_host.argtypes = [GCV_FN, C.c_void_p, C.c_double, C.c_double, C.c_int,
                                         C.POINTER(C.c_double), C.POINTER(C.c_int),
                                         C.POINTER(C.c_double)]
    cb = GCV_FN(lambda mu, ctx: float(G(mu)))
    mu, bk = C.c_double(), C.c_int()
    curve = (C.c_double * count)()
    FD.check(lib.fd_gcv_minimize_host(cb, None, mu_min, mu_max, count, C.byref(mu),
                                      C.byref(bk), curve))
    return mu.value, bk.value, np.array(curve[:])


FUNCS = [
    ("interior", lambda m: (math.log(m) + 7.3) ** 2 + 1.0),
    ("left-edge", lambda m: m),
    ("right-edge", lambda m: 1.0 / m),
    ("flat-tie", lambda m: 2.5),
    ("zero", lambda m: 0.0),
    ("two-tied-minima", lambda m: min((math.log(m) + 10) ** 2, (math.log(m) + 4) ** 2)),
    ("rational", lambda m: (1e-3 + m) ** 2 / (1e-6 + m) + 0.25 * math.sin(math.log(m))),
]


@pytest.mark.parametrize("name,G", FUNCS)
@pytest.mark.parametrize("search", [(1e-9, 1.0, 40), (1e-12, 10.0, 200), (1e-6, 1.0, 7),
                                    (1e-8, 1.0, 256)])
def test_gcv_minimize_host_matches_oracle(name, G, search):
    mu, bk, curve = host_minimize(G, *search)
    r = O.gcv_minimize(G, *search)
    assert np.allclose(curve, r.vals, rtol=1e-15, atol=0)
    assert bk == r.best_k
    assert abs(mu / r.mu - 1) < 1e-14


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name,G", FUNCS)
def test_gcv_minimize_host_matches_reference(name, G):
    for search in ((1e-9, 1.0, 40), (1e-12, 10.0, 200)):
        mu, bk, curve = host_minimize(G, *search)
        mu_ref, curve_ref = R.gcv_minimize(G, *search)
        assert np.array_equal(curve, curve_ref)
        assert mu == mu_ref  # same libm, same operation order: bitwise


def test_gcv_minimize_parameter_errors():
    for args in ((0.0, 1.0, 10), (1e-3, 1e-6, 10), (1e-3, 1.0, 1)):
        with pytest.raises(P.ValidationError):
            host_minimize(lambda m: m, *args)


def test_no_cpu_fallback():
    """Without a CUDA device, valid calls fail loudly (status 1) instead of
    computing on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.FastDeblurError) as e:
        P.build_operator([0.25, 0.5, 0.25], 64, "hoc-cosine")
    assert "no CUDA device" in str(e.value)


def test_cli_front_end_parses_without_a_gpu():
    """tools/fastdeblur_b200 (reference tools/fastdeblur.cpp:349-453): --help exits 0,
    parse errors exit 2 before any device work."""
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools",
                       "fastdeblur_b200")
    if not os.path.exists(exe):
        pytest.skip("tools/fastdeblur_b200 not built")
    assert subprocess.run([exe, "--help"], capture_output=True).returncode == 0
    assert subprocess.run([exe], capture_output=True).returncode == 2
    assert subprocess.run([exe, "deblur", "--bogus", "1"], capture_output=True).returncode == 2
