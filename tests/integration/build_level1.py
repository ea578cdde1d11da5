"""Builds the INTEGRATION.md level-1 binding against the reference's own
headers (proj/include/ppa, read-only, never copied) with a stub <Eigen/Core>
(tests/integration/eigen_stub; Eigen is absent).  The C++ block is extracted
from the document itself, so the document cannot drift from what compiles.

    python tests/integration/build_level1.py   ->  tests/integration/_build/level1

TEST INFRASTRUCTURE ONLY.  Needs /root/reference (present in the build
container, absent on the GPU box: the binary built here travels with the
repository snapshot).
"""
from __future__ import annotations

import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_INC = "/root/reference/proj/include"
OUT = os.path.join(HERE, "_build")
BIN = os.path.join(OUT, "level1")


def extract() -> str:
    txt = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```cpp\n(.*?)```", txt, flags=re.S)
    src = next(b for b in blocks if "class B200PolyOperator" in b)
    path = os.path.join(OUT, "b200_operator.cpp")
    os.makedirs(OUT, exist_ok=True)
    with open(path, "w") as f:
        f.write(src)
    return path


def build() -> str:
    if not os.path.isdir(REF_INC):
        raise FileNotFoundError(REF_INC)
    src = extract()
    lib = os.path.join(ROOT, "paper_1806_08020_b200")
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-Wno-unused-function",
           "-I", os.path.join(HERE, "eigen_stub"), "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
           src, os.path.join(HERE, "level1_main.cpp"), "-o", BIN,
           "-L", lib, "-lppa_b200", f"-Wl,-rpath,{lib}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("level-1 binding failed to compile")
    return BIN


if __name__ == "__main__":
    print(build())
