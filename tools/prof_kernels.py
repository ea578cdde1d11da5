"""Kernel-profiling driver (run under ncu on one GPU): config 3 pi(A)v, CGS2 and V*Q."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1806_08020_b200 as ppa

what = sys.argv[1] if len(sys.argv) > 1 else "all"
torch.cuda.set_device(0)
ppa.set_stream(torch.cuda.current_stream())
csr = ppa.CsrMatrix.config(3)
n = csr.n
A = ppa.make_csr_operator(csr)
# 8 real roots spread over the config-3 spectrum (the timing does not depend on them)
roots = ppa.leja_order(np.linspace(30.0, 311000.0, 8))
v = torch.tensor(ppa.normal_vector(n, 2, 3), device="cuda")
out = torch.empty(n, dtype=torch.float64, device="cuda")
if what in ("all", "spmv"):
    for _ in range(3):
        ppa.apply_poly(roots, A, v, out)
if what in ("all", "cgs"):
    c = 40
    ld = (n + 31) // 32 * 32
    V = torch.randn((c + 1) * ld, dtype=torch.float64, device="cuda")
    w = torch.randn(n, dtype=torch.float64, device="cuda")
    Hc = torch.empty(c + 2, dtype=torch.float64, device="cuda")
    flag = torch.zeros(2, dtype=torch.int32, device="cuda")
    for _ in range(3):
        ppa.cgs2_step(V, ld, n, c, w, Hc, flag)
    G = torch.randn(c * 20, dtype=torch.float64, device="cuda")
    for _ in range(2):
        ppa.ts_combine(V, ld, n, c, G, 20, V, ld)
torch.cuda.synchronize()
print("done")
