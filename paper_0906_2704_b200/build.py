"""Build the sm_100a shared library in-tree (paper_0906_2704_b200/libfdb200.so).

nvcc cross-compiles without a GPU; the .so travels to the GPU box with the
repository snapshot.  No JIT cache is used."""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfdb200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
         "-Xcompiler", "-O3"]


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    hdr = os.path.join(HERE, "..", "include", "fastdeblur_b200.h")
    return any(os.path.getmtime(s) > t for s in sources() + [hdr])


def build_library(force=False, verbose=False, out=None, defines=()):
    """Compile fd_capi.cu (one translation unit) into `out` (default LIB);
    `defines` adds -D flags (e.g. FD_PHASE_CLOCKS for a timing build)."""
    out = out or LIB
    if out == LIB and not defines and not force and not needs_build():
        return LIB
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    cmd = [nvcc, *ARCH, *FLAGS, *("-D" + d for d in defines), os.path.join(CSRC, "fd_capi.cu"),
           "-o", out + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))
