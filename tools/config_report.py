"""Per-config measurements on one GPU: pi(A)v throughput with the config's own
polynomial (byte model), CGS2 at the config's m, and time to nev.

    python tools/config_report.py [configs...] > gpurun_out/configs.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1806_08020_b200 as ppa
from paper_1806_08020_b200.configs import CONFIGS


def timed(fn, reps, stream):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def report(k):
    stream = torch.cuda.current_stream()
    t0 = time.time()
    csr = ppa.CsrMatrix.config(k)
    n, nnz, _ = csr.info()
    gen_s = time.time() - t0
    A = ppa.make_csr_operator(csr)
    cfg = ppa.config_solve_config(k)
    bspmv = A.model_bytes()
    out = {"config": k, "name": CONFIGS[k]["name"], "n": n, "nnz": nnz, "B_spmv": bspmv,
           "generate_s": round(gen_s, 3), "layout": A.layout()}
    # pi(A)v with the config's polynomial (built on the device as solve() does)
    b = torch.tensor(ppa.normal_vector(n, cfg.seed, ppa.STREAM_POLY), device="cuda")
    if k == 5:
        r1, _ = ppa.build_gmres_poly(A, b, cfg.double_d1)
        tau = ppa.make_poly_complement_operator(A, r1)
        b2 = torch.tensor(ppa.normal_vector(n, cfg.seed, ppa.STREAM_POLY2), device="cuda")
        r2, _ = ppa.build_gmres_poly(tau, b2, cfg.double_d2)
        op = ppa.make_poly_operator(tau, r2)
        eff = len(r1) * len(r2)
    else:
        roots, _ = ppa.build_gmres_poly(A, b, cfg.degree)
        if cfg.stability == "pof_auto":
            roots = ppa.add_stability_roots(roots, len(roots))
        op = ppa.make_poly_operator(A, roots)
        eff = len(roots)
    v = torch.tensor(ppa.normal_vector(n, cfg.seed, ppa.STREAM_ARNOLDI), device="cuda")
    y = torch.empty_like(v)
    reps = max(3, int(2e10 / (eff * bspmv)))
    ms = timed(lambda: op.apply(v, y), reps, stream)
    out.update(eff_degree=eff, piav_ms=round(ms, 4),
               piav_gbs=round(eff * bspmv / (ms * 1e-3) / 1e9, 1))
    # one SpMV alone
    ms1 = timed(lambda: ppa.spmv(A, v, y), max(10, int(2e9 / bspmv)), stream)
    out.update(spmv_us=round(ms1 * 1e3, 2), spmv_gbs=round(bspmv / (ms1 * 1e-3) / 1e9, 1))
    # time to nev (after a one-cycle warm-up solve: lazy kernel loading)
    warm = ppa.config_solve_config(k)
    warm.max_cycles = 1
    ppa.solve_double(A, warm) if k == 5 else ppa.solve(A, warm)
    r = ppa.solve_double(A, cfg) if k == 5 else ppa.solve(A, cfg)
    lam = r["eigenvalues"]
    status = {2: "residual-certified pseudo-eigenvalues (non-normal: DESIGN.md 4.1)",
              5: "residual-certified pseudo-eigenvalues (non-normal: DESIGN.md 4.1)",
              4: "not converged within max_cycles on the GPU or the oracle (DESIGN.md 4.1)"}
    out.update(eigenvalue_status=status.get(k, "eigenvalues (closed-form checked)"),
               cycles_per_s=round(r["cycles"] / r["timing"]["total"], 3),
               mvps_per_s=round(r["cost"]["mvps"] / r["timing"]["total"], 1))
    gold = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                        "golden", f"c{k}_solve.json")
    if os.path.exists(gold):
        g = json.load(open(gold))
        out.update(oracle_fixture={"seconds": round(g["oracle_seconds"], 1), "cycles": g["cycles"],
                                   "mvps": g["cost"]["mvps"],
                                   "threads": "8 (build container)"})
    out.update(solve_s=round(r["timing"]["total"], 4), converged=r["converged"], cycles=r["cycles"],
               mvps=r["cost"]["mvps"], dots=r["cost"]["dots"], rtol=r["rtol"],
               max_residual=float(np.max(r["residuals"])) if len(r["residuals"]) else None,
               timing={kk: round(vv, 4) for kk, vv in r["timing"].items()},
               eigenvalues_head=[[round(z.real, 6), round(z.imag, 6)] for z in lam[:4]])
    return out


if __name__ == "__main__":
    torch.cuda.set_device(0)
    ppa.set_stream(torch.cuda.current_stream())
    ks = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
    for k in ks:
        print(json.dumps(report(k)), flush=True)
