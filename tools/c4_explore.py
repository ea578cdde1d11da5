"""Config 4 (random Poisson(16) rows, 10 eigenvalues nearest 0): which solver
settings converge?  Prints one JSON line per setting with the per-cycle best
and final max residual.

    python tools/c4_explore.py [setting ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1806_08020_b200 as ppa

SETTINGS = {
    "base": {},
    "harmonic": dict(variant="harmonic"),
    "stab": dict(stability="pof_auto"),
    "harm_stab": dict(variant="harmonic", stability="pof_auto"),
    "d60": dict(degree=60, stability="pof_auto"),
    "d15": dict(degree=15),
    "d0": dict(degree=0, max_cycles=300),
    "m100": dict(m=100, k=50, stability="pof_auto"),
    "harm_m100": dict(m=100, k=50, variant="harmonic", stability="pof_auto"),
}

names = sys.argv[1:] or list(SETTINGS)
csr = ppa.CsrMatrix.config(4)
A = ppa.make_csr_operator(csr)
ppa.solve(ppa.make_csr_operator(ppa.CsrMatrix.config(1)), ppa.config_solve_config(1))
for name in names:
    kw = dict(max_cycles=150)
    kw.update(SETTINGS[name])
    cfg = ppa.config_solve_config(4, **kw)
    t = time.time()
    r = ppa.solve(A, cfg)
    h = r["cycle_max_residual"]
    print(json.dumps({"setting": name, "converged": r["converged"], "cycles": r["cycles"],
                      "seconds": round(time.time() - t, 2), "mvps": r["cost"]["mvps"],
                      "rtol": r["rtol"], "best": float(np.min(h)) if len(h) else None,
                      "last": float(h[-1]) if len(h) else None,
                      "hist": [float(f"{x:.3g}") for x in h[::10]],
                      "eigs": [f"{z.real:.6g}{z.imag:+.3g}j" for z in r["eigenvalues"]]}),
          flush=True)
