"""Config-4 residual history on the GPU next to the oracle fixture's."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0); ppa.set_stream(torch.cuda.current_stream())
g = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c4_solve.json")))
A = ppa.make_csr_operator(ppa.CsrMatrix.config(4))
cfg = ppa.config_solve_config(4)
cfg.max_cycles = 6
r = ppa.solve(A, cfg)
print("gpu   ", [float(x) for x in r["cycle_max_residual"]])
print("oracle", g["cycle_max_residual"][:6])
