import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1806_08020_b200 as ppa
torch.cuda.set_device(0)
for cfg, nr in ((1, 10), (3, 50)):
    A = ppa.make_csr_operator(ppa.CsrMatrix.config(cfg)); n = A.dim()
    roots = ppa.leja_order(np.linspace(30.0, 311000.0, nr))
    v = torch.tensor(ppa.normal_vector(n, 2, 3), device="cuda"); out = torch.empty_like(v)
    cs = torch.cuda.Stream(); cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        ppa.set_stream(cs)
        ppa.apply_poly(roots, A, v, out); torch.cuda.synchronize()
        ts = []
        for k in range(5):
            g = torch.cuda.CUDAGraph()
            t = time.perf_counter()
            with torch.cuda.graph(g, stream=cs):
                ppa.apply_poly(roots, A, v, out)
            ts.append(time.perf_counter() - t)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(20): ppa.apply_poly(roots, A, v, out)
        th = (time.perf_counter() - t) / 20
        torch.cuda.synchronize()
    ppa.set_stream(torch.cuda.current_stream())
    print(cfg, "capture+instantiate us", [round(x * 1e6) for x in ts], "host enqueue per apply us", round(th * 1e6))
