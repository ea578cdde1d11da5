import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0); ppa.set_stream(torch.cuda.current_stream())
csr = ppa.CsrMatrix.config(3); n = csr.n
A = ppa.make_csr_operator(csr)
for rep in range(3):
    t0 = time.time(); bh = ppa.normal_vector(n, 2, ppa.STREAM_POLY); t1 = time.time()
    b = torch.tensor(bh, device="cuda"); torch.cuda.synchronize(); t2 = time.time()
    base, _ = ppa.build_gmres_poly(A, b, 50); torch.cuda.synchronize(); t3 = time.time()
    roots = ppa.add_stability_roots(base, len(base)); t4 = time.time()
    print(f"rng {1e3*(t1-t0):.1f} ms  upload {1e3*(t2-t1):.1f}  build {1e3*(t3-t2):.1f}  stab {1e3*(t4-t3):.2f}")
    st = ppa.arnoldi_init(b, n, 50); torch.cuda.synchronize(); t5 = time.time()
    st.extend(A, 50); torch.cuda.synchronize(); t6 = time.time()
    print(f"arnoldi_init {1e3*(t5-t4):.1f}  extend50 {1e3*(t6-t5):.1f}")
r = ppa.solve(A, ppa.config_solve_config(3))
print(r["timing"])
