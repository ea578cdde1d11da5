"""Generates the committed golden fixtures in tests/golden/ from the CPU oracle.

    python tests/golden/make_golden.py fingerprints c3_poly c1_solve ...

Each fixture records the oracle's output on the seeded BASELINE inputs so the
GPU tests can check full-size parity without running the (slow) oracle on
the GPU box.  The oracle itself is pinned against SPEC.md's known-answer
examples and closed-form spectra (tests/test_oracle_pins.py).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def _c(z):
    z = np.asarray(z, dtype=np.complex128)
    return {"re": z.real.tolist(), "im": z.imag.tolist()}


def fingerprints():
    out = {}
    for k in (1, 2, 3, 4, 5):
        n, nnz, fp = O.Csr.config(k).info()
        out[f"config{k}"] = {"n": n, "nnz": nnz, "fingerprint": str(fp)}
    small = {
        "bidiag777": O.Csr.bidiagonal(777), "convdiff_ref37": O.Csr.convection_diffusion(37),
        "convdiff_ref50": O.Csr.convection_diffusion(50),
        "convdiff_const45": O.Csr.convection_diffusion_const(45, 0.5),
        "laplace3d17": O.Csr.laplacian_3d(17),
        "random_poisson20000_s7": O.Csr.random_poisson(20000, 16.0, 7),
    }
    for name, m in small.items():
        n, nnz, fp = m.info()
        out[name] = {"n": n, "nnz": nnz, "fingerprint": str(fp)}
    return out


def c3_poly():
    O.set_threads(os.cpu_count() or 1)
    A = O.csr_operator(O.Csr.config(3))
    b = O.normal_vector(4096000, 2, 2)
    cost = np.zeros(3)
    t = time.time()
    roots, trunc = O.build_gmres_poly(A, b, 50, cost)
    el = time.time() - t
    pof = O.compute_pof(roots)
    aug = O.add_stability_roots(roots)
    return {"config": 3, "degree": 50, "seed": 2, "stream": 2, "truncated": trunc,
            "base_roots": _c(roots), "roots": _c(aug), "max_log10_pof": pof["max_log10_pof"],
            "total_copies": pof["total_copies"], "cost": cost.tolist(), "oracle_seconds": el}


def _solve_fixture(cfg_id, **kw):
    O.set_threads(os.cpu_count() or 1)
    A = O.csr_operator(O.Csr.config(cfg_id))
    t = time.time()
    r = O.solve(A, **kw)
    return {"config": cfg_id, "params": kw, "eigenvalues": _c(r["eigenvalues"]),
            "residuals": r["residuals"].tolist(), "converged": r["converged"], "cycles": r["cycles"],
            "cost": r["cost"], "rtol": r["rtol"], "norm_estimate": r["norm_estimate"],
            "poly": _c(r["poly"]), "inner_poly": _c(r["inner_poly"]),
            "cycle_max_residual": r["cycle_max_residual"].tolist(),
            "oracle_seconds": time.time() - t}


def _variant_solve(cfg_id, variant, **kw):
    O.set_variant(variant)
    try:
        return _solve_fixture(cfg_id, **kw)
    finally:
        O.set_variant(0)


SOLVE_PARAMS = {
    2: dict(m=50, k=20, nev=20, degree=25, seed=1),
    5: dict(m=30, k=15, nev=20, double=(15, 20), seed=3, allow_nev_above_k=True),
}


def roundoff_floor():
    """The oracle's own roundoff floor on the non-normal configs 2 and 5: the
    same solve under two more summation orders the reference leaves to Eigen
    (oracle variants 1 = classical CGS2 + blocked dots, 2 = MGS2 + blocked
    dots; ppa_oracle.cpp g_variant).  Variant 0 is c{2,5}_solve.json."""
    out = {}
    for cfg_id, kw in SOLVE_PARAMS.items():
        out[f"config{cfg_id}"] = {str(v): _variant_solve(cfg_id, v, **kw) for v in (1, 2)}
    return out


FIXTURES = {
    "roundoff_floor": roundoff_floor,
    "fingerprints": fingerprints,
    "c3_poly": c3_poly,
    "c1_solve": lambda: _solve_fixture(1, m=30, k=15, nev=10, degree=10, seed=1),
    "c2_solve": lambda: _solve_fixture(2, m=50, k=20, nev=20, degree=25, seed=1),
    "c3_solve": lambda: _solve_fixture(3, m=40, k=20, nev=15, degree=50, stability=True, seed=2),
    "c4_solve": lambda: _solve_fixture(4, m=50, k=25, nev=10, degree=30, seed=4),
    "c5_solve": lambda: _solve_fixture(5, m=30, k=15, nev=20, double=(15, 20), seed=3,
                                       allow_nev_above_k=True),
}

if __name__ == "__main__":
    for name in sys.argv[1:]:
        t = time.time()
        data = FIXTURES[name]()
        with open(os.path.join(HERE, f"{name}.json"), "w") as f:
            json.dump(data, f, indent=1)
        print(f"{name}: {time.time() - t:.1f}s", flush=True)
