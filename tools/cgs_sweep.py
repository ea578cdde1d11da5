"""CGS2 step time vs basis size c on config 3 (real Arnoldi basis)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0); ppa.set_stream(torch.cuda.current_stream())
A = ppa.make_csr_operator(ppa.CsrMatrix.config(3))
n = A.dim()
v = torch.tensor(ppa.normal_vector(n, 2, 3), device="cuda")
st = ppa.arnoldi_init(v, n, 48)
st.extend(A, 48)
ld = st.ld
out = []
for c in [1, 2, 4, 8, 12, 16, 24, 32, 40, 48]:
    w0 = torch.empty(n, dtype=torch.float64, device="cuda")
    ppa.spmv(A, st.V_ptr + 8 * ld * (c - 1), w0)
    w = torch.empty_like(w0)
    Hc = torch.empty(c + 2, dtype=torch.float64, device="cuda")
    flag = torch.zeros(2, dtype=torch.int32, device="cuda")
    ts = []
    for i in range(8):
        w.copy_(w0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ppa.cgs2_step(st.V_ptr, ld, n, c, w, Hc, flag); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts[2:]))
    out.append({"c": c, "ms": round(ms, 4), "gbs_model": round(8.0 * n * (3 * c + 7) / ms / 1e6, 1)})
print(json.dumps(out))
