"""Solve configs with and without CUDA-graph launch of the polynomial chain
(PPA_CHAIN_GRAPHS), one process per variant: median time to nev over five
solves and a bitwise comparison of the results.

    python tools/graph_ab.py [configs...]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys, numpy as np
sys.path.insert(0, %r)
import paper_1806_08020_b200 as ppa
ppa.solve(ppa.make_csr_operator(ppa.CsrMatrix.config(1)), ppa.config_solve_config(1))
out = {}
for k in map(int, sys.argv[1:]):
    A = ppa.make_csr_operator(ppa.CsrMatrix.config(k))
    cfg = ppa.config_solve_config(k)
    f = ppa.solve_double if cfg.double_d1 else ppa.solve
    f(A, cfg)  # warm (first-solve allocations)
    ts = []
    for _ in range(5):
        r = f(A, cfg)
        ts.append(r["timing"]["total"])
    out[k] = {"s": float(np.median(ts)), "ext": r["timing"]["extend"], "cycles": r["cycles"], "mvps": r["cost"]["mvps"],
              "eig": [float(z.real) for z in r["eigenvalues"]] + [float(z.imag) for z in r["eigenvalues"]],
              "res": [float(x) for x in r["residuals"]]}
print(json.dumps(out))
""" % ROOT

cfgs = sys.argv[1:] or ["1", "2", "3", "5"]
res = {}
for var in ("0", "1"):
    env = dict(os.environ, PPA_CHAIN_GRAPHS="1" if var == "0" else "0")
    r = subprocess.run([sys.executable, "-c", CHILD] + cfgs, env=env, capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[-2000:])
        sys.exit(1)
    res[var] = json.loads(r.stdout.strip().splitlines()[-1])
for k in cfgs:
    a, b = res["0"][k], res["1"][k]
    print(json.dumps({"config": int(k), "graphs_s": round(a["s"], 4), "direct_s": round(b["s"], 4),
                      "graphs_extend": round(a["ext"], 4), "direct_extend": round(b["ext"], 4),
                      "cycles": [a["cycles"], b["cycles"]], "mvps": [a["mvps"], b["mvps"]],
                      "bitwise_equal": a["eig"] == b["eig"] and a["res"] == b["res"]}))
