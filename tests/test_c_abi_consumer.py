"""The C-ABI from plain C (tests/c/abi_consumer.c): it must compile against
include/ppa_b200.h with a C99 compiler and link against libppa_b200.so here;
on the GPU it solves config 1 and must agree with the oracle's eigenvalues."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1806_08020_b200")


def _build(tmp_path):
    exe = str(tmp_path / "abi_consumer")
    cmd = ["cc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "c", "abi_consumer.c"), "-L", PKG, "-lppa_b200",
           f"-Wl,-rpath,{PKG}", "-lm", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_consumer_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_consumer_solves_config1(cuda, tmp_path):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    out = subprocess.run([_build(tmp_path), "1"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    kv = dict(item.split("=", 1) for item in out.stdout.split())
    assert kv["converged"] == "1" and int(kv["n"]) == 5000
    eig = np.sort(np.array([float(v) for v in kv["eig"].split(",")]))
    o = O.solve(O.csr_operator(O.Csr.config(1)), m=30, k=15, nev=10, degree=10, seed=1)
    assert np.allclose(eig, np.sort(o["eigenvalues"].real), rtol=1e-8)
    assert abs(int(kv["mvps"]) - o["cost"]["mvps"]) <= 0.05 * o["cost"]["mvps"]
