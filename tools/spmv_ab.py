"""A/B timing of the SpMV layouts on config 3 pi(A)v (one process per variant).

    python tools/spmv_ab.py [config] VAR=VAL,VAR=VAL ...   (each arg one variant)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0)
ppa.set_stream(torch.cuda.current_stream())
cfg = int(sys.argv[1])
A = ppa.make_csr_operator(ppa.CsrMatrix.config(cfg))
n = A.dim()
roots = ppa.leja_order(np.linspace(30.0, 311000.0, 50))
v = torch.tensor(ppa.normal_vector(n, 2, 3), device="cuda")
out = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    ppa.apply_poly(roots, A, v, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record(); ppa.apply_poly(roots, A, v, out); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 50 * 1e3)
g_us = None
if "--graph" in sys.argv:
    # the same chain captured once as a CUDA graph and replayed
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cs):
        ppa.set_stream(cs)
        ppa.apply_poly(roots, A, v, out)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=cs):
            ppa.apply_poly(roots, A, v, out)
    torch.cuda.synchronize()
    ppa.set_stream(torch.cuda.current_stream())
    gs = []
    for _ in range(10):
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        gs.append(e0.elapsed_time(e1) / 50 * 1e3)
    g_us = float(np.median(gs))
print(json.dumps({"us_per_spmv": float(np.median(ts)), "graph_us_per_spmv": g_us, "layout": A.layout(),
                  "model_gbs": A.model_bytes() / (np.median(ts) * 1e-6) / 1e9,
                  "checksum": float(out.sum().item())}))
""" % ROOT

cfg = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1].isdigit() else "3"
variants = [a for a in sys.argv[1:] if not a.isdigit() and a != "--graph"] or [""]
for var in variants:
    env = dict(os.environ)
    for kv in filter(None, var.split(",")):
        k, v = kv.split("=")
        env[k] = v
    extra = ["--graph"] if "--graph" in sys.argv else []
    r = subprocess.run([sys.executable, "-c", CHILD, cfg] + extra, env=env, capture_output=True,
                       text=True)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
    plans = [ln for ln in r.stderr.splitlines() if "plan" in ln]
    print(json.dumps({"variant": var or "default", "result": line, "plans": plans}))
