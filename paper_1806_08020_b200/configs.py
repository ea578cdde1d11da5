"""BASELINE.json workloads (configs 1..5) as solver settings.

Frozen choices: rtol = 1e-8 * ||A||_est (the
reference default, inc/solver.hpp:27-29); config 1 and 2 use seed 1, config
3 seed 2, config 5 seed 3 (as BASELINE states), config 4 seed 4 (unstated in
BASELINE); config 5 keeps BASELINE's k = 15 < nev = 20 through
allow_nev_above_k.
"""
from __future__ import annotations

from ._capi import SolveConfig

CONFIGS = {
    1: dict(name="bidiag-5000", kind="bidiagonal", n=5000, nnz=9999,
            solve=dict(m=30, k=15, nev=10, degree=10, seed=1)),
    2: dict(name="convdiff-1000x1000-Pe0.5", kind="convdiff_const", grid=1000, n=1_000_000,
            nnz=4_996_000, solve=dict(m=50, k=20, nev=20, degree=25, seed=1)),
    3: dict(name="laplace3d-160^3", kind="laplacian_3d", grid=160, n=4_096_000, nnz=28_518_400,
            solve=dict(m=40, k=20, nev=15, degree=50, stability="pof_auto", seed=2)),
    4: dict(name="random-poisson16-2e6", kind="random_poisson", n=2_000_000, nnz=None,
            solve=dict(m=50, k=25, nev=10, degree=30, seed=4)),
    5: dict(name="convdiff-2048x2048-Pe0.5-double15x20", kind="convdiff_const", grid=2048,
            n=4_194_304, nnz=20_963_328,
            solve=dict(m=30, k=15, nev=20, double_d1=15, double_d2=20, seed=3,
                       allow_nev_above_k=True)),
}


def config_solve_config(config: int, **over) -> SolveConfig:
    kw = dict(CONFIGS[config]["solve"])
    kw.update(over)
    return SolveConfig(**kw)
