"""Compile oracle/gr_oracle.c into oracle/liborc.so (plain gcc, no SIMD flags).

Test infrastructure only (see oracle/__init__.py)."""
from __future__ import annotations

import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(_HERE, "liborc.so")
SRC = [os.path.join(_HERE, "gr_oracle.c"), os.path.join(_HERE, "gr_oracle.h")]


def build(force: bool = False) -> str:
    stale = not os.path.exists(SO) or any(os.path.getmtime(s) > os.path.getmtime(SO) for s in SRC)
    if force or stale:
        tmp = SO + f".tmp{os.getpid()}"
        cmd = ["gcc", "-std=c11", "-O1", "-fno-fast-math", "-ffp-contract=off", "-Wall",
               "-Werror", "-shared", "-fPIC", SRC[0], "-o", tmp]
        subprocess.run(cmd, check=True)
        os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force=True))
