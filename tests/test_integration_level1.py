"""INTEGRATION.md level 1: the reference-side binding (B200PolyOperator, a
LinearOperator subclass over host Eigen vectors) compiled from the document
against the reference's own headers (tests/integration/build_level1.py) and
run through LinearOperator::apply."""
import os
import subprocess

import importlib.util

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "integration", "_build", "level1")
REF_INC = "/root/reference/proj/include"
ROOTS = [250.0, 120.0 + 30.0j, 120.0 - 30.0j, 40.0, 3.0]


def _build():
    spec = importlib.util.spec_from_file_location(
        "build_level1", os.path.join(HERE, "integration", "build_level1.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent (GPU box)")
def test_level1_binding_compiles_against_reference_headers():
    assert os.path.exists(_build())


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent (GPU box)")
def test_level1_binding_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: the GPU test runs the binding")
    r = subprocess.run([_build()], capture_output=True, text=True)
    assert r.returncode == 1 and "level1:" in r.stderr  # a CUDA error, no CPU fallback


@pytest.mark.gpu
def test_level1_binding_matches_oracle():
    if not os.path.exists(BIN):
        pytest.skip("level-1 binary not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.split()
    n, mvps, vops, per = (int(v) for v in lines[:4])
    y = np.array([float(v) for v in lines[4:]])
    assert n == 300 and per == 5 and mvps == 5 and y.size == n
    Q = O.Csr.bidiagonal(n)
    x = 1.0 + 0.01 * np.arange(n)
    cost = np.zeros(3)
    ref = O.poly_operator(O.csr_operator(Q), ROOTS).apply(x, cost)
    assert np.array_equal(y, ref)
    assert (mvps, vops) == (int(cost[0]), int(cost[2]))
