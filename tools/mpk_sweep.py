"""Sweep the matrix-powers knobs on config 3 (one process per setting)."""
import json
import os
import subprocess
import sys

CODE = r'''
import os, sys, json, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0); ppa.set_stream(torch.cuda.current_stream())
A = ppa.make_csr_operator(ppa.CsrMatrix.config(3))
roots = ppa.leja_order(np.linspace(30.0, 311000.0, 50))
n = 4096000
v = torch.tensor(ppa.normal_vector(n, 2, 3), device="cuda"); y = torch.empty_like(v)
for _ in range(3): ppa.apply_poly(roots, A, v, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(10): ppa.apply_poly(roots, A, v, y)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"ms": e0.elapsed_time(e1) / 10}))
'''
for env in ([{"PPA_ENABLE_MPK": "0"}] + [{"PPA_ENABLE_MPK": "1", "PPA_MPK_LAG_ROUNDS": str(l), "PPA_MPK_CTAS_PER_SM": str(c), "PPA_MPK_SCHED": s}
            for s in ("ticket", "static") for c in (3, 4) for l in (1.0, 2.0)]):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", CODE], env=e, capture_output=True, text=True, timeout=120)
    out = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
    print(json.dumps(env), out, flush=True)
