"""Build libgr.so (the C-ABI library of include/gr.h) for sm_100a, in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, static cudart,
no torch headers or libraries: the boundary is plain C."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libgr.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "gr.h"), __file__]


def build(force: bool = False, verbose: bool = False) -> str:
    stale = not os.path.exists(SO) or any(os.path.getmtime(d) > os.path.getmtime(SO) for d in deps())
    if not (force or stale):
        return SO
    tmp = SO + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-Wall",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-cudart", "static",
           *sources(), "-o", tmp]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv))
