"""One config-5 pi(A)v (nested double polynomial) for launch-list profiling."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0); ppa.set_stream(torch.cuda.current_stream())
A = ppa.make_csr_operator(ppa.CsrMatrix.config(5))
cfg = ppa.config_solve_config(5)
n = A.dim()
b = torch.tensor(ppa.normal_vector(n, cfg.seed, ppa.STREAM_POLY), device="cuda")
r1, _ = ppa.build_gmres_poly(A, b, cfg.double_d1)
tau = ppa.make_poly_complement_operator(A, r1)
b2 = torch.tensor(ppa.normal_vector(n, cfg.seed, ppa.STREAM_POLY2), device="cuda")
r2, _ = ppa.build_gmres_poly(tau, b2, cfg.double_d2)
op = ppa.make_poly_operator(tau, r2)
print("inner roots", np.round(r1, 1).tolist())
print("outer roots", np.round(r2, 4).tolist())
v = torch.tensor(ppa.normal_vector(n, cfg.seed, ppa.STREAM_ARNOLDI), device="cuda")
y = torch.empty_like(v)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for _ in range(2):
    op.apply(v, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    op.apply(v, y)
e1.record(); torch.cuda.synchronize()
print("ms per apply", e0.elapsed_time(e1) / reps)
