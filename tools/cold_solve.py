"""Cold vs warm solve of one config in a fresh process (first-use costs:
lazy kernel loading, shared-memory attributes, pools).

    python tools/cold_solve.py [config]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08020_b200 as ppa

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
t0 = time.time()
ppa.lib()
t1 = time.time()
A = ppa.make_csr_operator(ppa.CsrMatrix.config(k))
t2 = time.time()
out = {"config": k, "load_s": round(t1 - t0, 3), "operator_s": round(t2 - t1, 3)}
for name in ("cold", "warm"):
    r = ppa.solve(A, ppa.config_solve_config(k))
    out[name] = {kk: round(v, 4) for kk, v in r["timing"].items()}
print(json.dumps(out))
