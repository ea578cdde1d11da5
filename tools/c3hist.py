import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0); ppa.set_stream(torch.cuda.current_stream())
A = ppa.make_csr_operator(ppa.CsrMatrix.config(3))
r = ppa.solve(A, ppa.config_solve_config(3))
print(r["rtol"], list(r["cycle_max_residual"]), r["cycles"], r["cost"]["mvps"])
