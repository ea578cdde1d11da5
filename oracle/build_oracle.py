"""Builds the CPU oracle (test infrastructure) into oracle/_build/libppa_oracle.so.

g++ -O3 -fopenmp -ffp-contract=off (no -march=native: the .so travels to
the GPU box, whose host CPU may differ).  LAPACK from scipy's OpenBLAS.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "ppa_oracle.cpp")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libppa_oracle.so")


def _lapack() -> str:
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_1806_08020_b200.build import find_lapack  # noqa: E402  (path helper only)

    return find_lapack()


def build() -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(SRC),
                                                            os.path.getmtime(__file__)):
        return LIB
    lapack = _lapack()
    tmp = LIB + ".tmp"
    cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-Wall", "-o", tmp, SRC, lapack, f"-Wl,-rpath,{os.path.dirname(lapack)}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("oracle build failed")
    shutil.move(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build())
