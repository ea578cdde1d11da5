"""Setup-phase spread of repeated solves (configs 2 and 3) and the host RNG
time of one start vector, on the GPU box.

    python tools/setup_noise.py
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1806_08020_b200 as ppa  # noqa: E402

torch.cuda.set_device(0)
ppa.set_stream(torch.cuda.current_stream())
print(json.dumps({"cpus": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}))
for n in (1000000, 4096000):
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        ppa.normal_vector(n, 2, 3)
        ts.append(round((time.perf_counter() - t) * 1e3, 2))
    print(json.dumps({"rng_ms": ts, "n": n}))
for k in (2, 3):
    A = ppa.make_csr_operator(ppa.CsrMatrix.config(k))
    c = ppa.config_solve_config(k)
    ppa.solve(A, ppa.config_solve_config(k, max_cycles=1))
    for _ in range(5):
        r = ppa.solve(A, c)
        print(json.dumps({"config": k, "timing": {a: round(b, 4) for a, b in r["timing"].items()}}))
