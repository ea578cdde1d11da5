"""Per-pass cost of the box-grid two-factor pass against the number of planes
(160 x 160 planes, 7-point Laplacian values): separates the per-launch fixed
cost (pipeline fill, drain, launch gap) from the per-step cost.

    python tools/grid2_scaling.py [nz ...]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1806_08020_b200 as ppa  # noqa: E402
from test_gpu_dia2 import _box  # noqa: E402

torch.cuda.set_device(0)
ppa.set_stream(torch.cuda.current_stream())
h2 = 161.0 ** 2
vals = [-h2, -h2, -h2, 6 * h2, -h2, -h2, -h2]
roots = ppa.leja_order(np.linspace(30.0, 311000.0, 50))
for nz in [int(a) for a in sys.argv[1:]] or [9, 18, 36, 72, 160, 320]:
    n, rp, ci, vv = _box(160, 160, nz, vals)
    A = ppa.make_csr_operator(ppa.CsrMatrix.from_arrays(n, rp, ci, vv))
    v = torch.randn(n, dtype=torch.float64, device="cuda")
    out = torch.empty_like(v)
    for _ in range(3):
        ppa.apply_poly(roots, A, v, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        e0.record()
        ppa.apply_poly(roots, A, v, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / 25)
    print(json.dumps({"nz": nz, "n": n, "us_per_pass": round(float(np.median(ts)), 3),
                      "ns_per_row": round(float(np.median(ts)) * 1e3 / n, 4),
                      "grid_pass": A.layout()["grid_pass"]}), flush=True)
