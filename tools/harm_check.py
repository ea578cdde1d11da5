import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0); ppa.set_stream(torch.cuda.current_stream())
d = np.arange(1.0, 1001.0)
for v in ["ritz", "harmonic"]:
    r = ppa.solve(ppa.make_diagonal(d), ppa.SolveConfig(m=40, k=20, nev=10, degree=0, seed=3, max_cycles=300, variant=v))
    print(v, r["converged"], r["cycles"], r["cost"]["mvps"], np.sort(r["eigenvalues"].real)[:10], r["cycle_max_residual"][-2:])
