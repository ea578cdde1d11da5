import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0)
ppa.set_stream(torch.cuda.current_stream())
A = ppa.make_csr_operator(ppa.CsrMatrix.config(3))
n = A.dim()
b = torch.tensor(ppa.normal_vector(n, 2, ppa.STREAM_POLY), device="cuda")
for ortho in ("dcgs2", "cgs2", "dcgs2", "cgs2"):
    torch.cuda.synchronize(); t = time.perf_counter()
    roots, _ = ppa.build_gmres_poly(A, b, 50, orthogonalization=ortho)
    torch.cuda.synchronize(); print(ortho, "build", round((time.perf_counter() - t) * 1e3, 2), "ms")
# Arnoldi extend alone, c 1..50
for ortho in ("dcgs2", "cgs2"):
    st = ppa.arnoldi_init(b, n, 50); st.set_orthogonalization(ortho)
    torch.cuda.synchronize(); t = time.perf_counter()
    st.extend(A, 50)
    torch.cuda.synchronize(); print(ortho, "extend 50", round((time.perf_counter() - t) * 1e3, 2), "ms")
    del st
r = ppa.solve(A, ppa.config_solve_config(3)); print(r["timing"])
r = ppa.solve(A, ppa.config_solve_config(3)); print(r["timing"])
