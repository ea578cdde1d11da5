import time, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0); ppa.set_stream(torch.cuda.current_stream())
csr = ppa.CsrMatrix.config(3); n = csr.n
A = ppa.make_csr_operator(csr, "sell32"); A2 = ppa.make_csr_operator(csr)
cfg = ppa.config_solve_config(3)
def rep(tag):
    t=time.time(); v=ppa.normal_vector(n, 2, 3); t1=time.time()
    r = ppa.solve(A2, cfg)
    print(tag, f"rng {1e3*(t1-t):.1f} ms", {k: round(v,4) for k,v in r["timing"].items()}, flush=True)
rep("fresh")
xh = torch.empty((20, n), dtype=torch.float64).pin_memory(); yh = torch.empty((20, n), dtype=torch.float64).pin_memory()
rep("after pin")
del xh, yh
rep("after del")
rep("again")
