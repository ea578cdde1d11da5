"""Per-cycle max residual on the GPU next to the oracle fixture (configs 1-5)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0); ppa.set_stream(torch.cuda.current_stream())
for k in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 5]:
    g = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"c{k}_solve.json")))
    A = ppa.make_csr_operator(ppa.CsrMatrix.config(k))
    cfg = ppa.config_solve_config(k)
    r = ppa.solve_double(A, cfg) if k == 5 else ppa.solve(A, cfg)
    h, gh = np.array(r["cycle_max_residual"]), np.array(g["cycle_max_residual"])
    m = min(len(h), len(gh))
    print(k, "gpu", h.tolist(), "oracle", gh.tolist(), "rel", (np.abs(h[:m] - gh[:m]) / gh[:m]).tolist())
