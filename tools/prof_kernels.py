"""Kernel-profiling driver (run under ncu on one GPU): config 3 pi(A)v, CGS2 and V*Q
(PPA_PROF_CONFIG=N picks another BASELINE config).

    python tools/prof_kernels.py [all|spmv|cgs] [auto|sell32|sell32_packed|dia_coded|csr]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1806_08020_b200 as ppa

what = sys.argv[1] if len(sys.argv) > 1 else "all"
layout = sys.argv[2] if len(sys.argv) > 2 else "auto"
torch.cuda.set_device(0)
ppa.set_stream(torch.cuda.current_stream())
csr = ppa.CsrMatrix.config(int(os.environ.get("PPA_PROF_CONFIG", "3")))
n = csr.n
A = ppa.make_csr_operator(csr, layout)
# 8 real roots spread over the config-3 spectrum (the timing does not depend on them)
roots = ppa.leja_order(np.linspace(30.0, 311000.0, 8))
v = torch.tensor(ppa.normal_vector(n, 2, 3), device="cuda")
out = torch.empty(n, dtype=torch.float64, device="cuda")
if what in ("all", "spmv"):
    for _ in range(3):
        ppa.apply_poly(roots, A, v, out)
if what in ("all", "cgs"):
    # real Arnoldi basis so every sweep (incl. the V[:,c] store) runs
    c = 40
    st = ppa.arnoldi_init(v, n, c)
    st.extend(A, c)
    ld = st.ld
    w0 = torch.empty(n, dtype=torch.float64, device="cuda")
    ppa.spmv(A, st.V_ptr + 8 * ld * (c - 1), w0)
    w = torch.empty_like(w0)
    Hc = torch.empty(c + 2, dtype=torch.float64, device="cuda")
    flag = torch.zeros(2, dtype=torch.int32, device="cuda")
    for _ in range(3):
        w.copy_(w0)
        ppa.cgs2_step(st.V_ptr, ld, n, c, w, Hc, flag)
    assert int(flag[0].item()) == 0
    G = torch.randn(c * 20, dtype=torch.float64, device="cuda")
    Y = torch.empty(20 * ld, dtype=torch.float64, device="cuda")
    for _ in range(2):
        ppa.ts_combine(st.V_ptr, ld, n, c, G, 20, Y, ld)
torch.cuda.synchronize()
print("done")
