"""ts_combine (V*G, the thick-restart / Ritz-vector recombination) at config-3
shapes against its byte model and cuBLAS dgemm on the same operands.

    python tools/combine_bench.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1806_08020_b200 as ppa

torch.cuda.set_device(0)
ppa.set_stream(torch.cuda.current_stream())
n = 4_096_000
ld = (n + 31) // 32 * 32


def ev(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for d, p, inplace in ((40, 20, True), (40, 15, False), (41, 21, True), (50, 25, True), (30, 20, False)):
    V = torch.randn(d + 1, ld, dtype=torch.float64, device="cuda")
    G = torch.randn(p, d, dtype=torch.float64, device="cuda")  # column-major d x p
    Out = V if inplace else torch.empty(p, ld, dtype=torch.float64, device="cuda")
    ref = (G @ V[:d, :n]).clone()
    ms = ev(lambda: ppa.ts_combine(V.data_ptr(), ld, n, d, G.data_ptr(), p, Out.data_ptr(), ld), 1)
    if inplace:
        V = torch.randn(d + 1, ld, dtype=torch.float64, device="cuda")
        Out = V
        ref = (G @ V[:d, :n]).clone()
        ppa.ts_combine(V.data_ptr(), ld, n, d, G.data_ptr(), p, Out.data_ptr(), ld)
        err = float((Out[:p, :n] - ref).abs().max() / ref.abs().max())
        ms = ev(lambda: ppa.ts_combine(V.data_ptr(), ld, n, d, G.data_ptr(), p, Out.data_ptr(), ld))
    else:
        ppa.ts_combine(V.data_ptr(), ld, n, d, G.data_ptr(), p, Out.data_ptr(), ld)
        err = float((Out[:, :n] - ref).abs().max() / ref.abs().max())
        ms = ev(lambda: ppa.ts_combine(V.data_ptr(), ld, n, d, G.data_ptr(), p, Out.data_ptr(), ld))
    Vs = V[:d, :n]
    cub = ev(lambda: torch.matmul(G, Vs))
    byts = 8.0 * n * (d + p)
    print(json.dumps({"d": d, "p": p, "inplace": inplace, "ms": round(ms, 4),
                      "gbs": round(byts / ms / 1e6, 1), "cublas_ms": round(cub, 4),
                      "max_rel_err": err}))
