"""Benchmark: pi(A)v throughput on the 4M-row 3D Laplacian (BASELINE config 3).

One "step" = one application of the preconditioner pi(A) (degree 50 GMRES
polynomial + pof stability copies, Leja order, built on the device from the
seeded start vector) to a device-resident vector: eff_degree fused SpMV-factor
launches over the 424 MB CSR matrix.  `value` is the north-star byte model
(eff_degree x [12 nnz + 4(n+1) + 16 n]) per second, whole job.  `e2e` is the
same metric through the C-ABI with pinned host buffers (H2D of v and D2H of
pi(A)v inside the timed region).  Extra keys report the CGS2 sweep bandwidth
and the solver's time to nev converged eigenpairs.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU: the path does not exchange data on one GPU's workload (north star:
one GPU), so N ranks run N independent replicas ("replicas only", weak
scaling); timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pi(A)v GB/s (north-star byte model), config 3 3D Laplacian 160^3"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class ClockSampler:
    """nvidia-smi sampling (every 50 ms) over the whole run; summary() keeps
    the samples that fall inside the timed regions marked with region()."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []
        self.regions = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.proc = None

    class _Region:
        def __init__(self, owner):
            self.owner = owner

        def __enter__(self):
            self.t0 = time.time()

        def __exit__(self, *a):
            # a sample reports the state of the preceding ~50 ms window
            self.owner.regions.append((self.t0, time.time() + 0.06))

    def region(self):
        return ClockSampler._Region(self)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for t, ln in self.lines:
            if not any(a <= t <= b for a, b in self.regions):
                continue
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "timed_regions": len(self.regions),
                "timed_seconds": round(sum(b - a - 0.06 for a, b in self.regions), 3)}


def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def dist_setup(gpus):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reduce_max(value: float, ws: int, device=None) -> float:
    """Max over ranks (device-timed numbers; nccl on GPU, gloo on CPU)."""
    if ws <= 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_gbs(bytes_per_step: float, ms_per_step: float, ws: int) -> float:
    """Weak-scaling aggregate: every replica moves bytes_per_step per step."""
    return ws * bytes_per_step / (ms_per_step * 1e-3) / 1e9


def load_golden_poly():
    """Config 3's degree-50 GMRES polynomial + pof copies as the oracle built
    it (tests/golden/c3_poly.json): the root set BOTH arms apply."""
    with open(os.path.join(ROOT, "tests", "golden", "c3_poly.json")) as f:
        g = json.load(f)
    roots = np.array(g["roots"]["re"]) + 1j * np.array(g["roots"]["im"])
    base = np.array(g["base_roots"]["re"]) + 1j * np.array(g["base_roots"]["im"])
    return roots, base


def workload_config(n, nnz, roots, base, ws):
    """The `config` dict, identical in both arms."""
    return {"workload": "config3-laplace3d-160^3-pi(A)v", "n": n, "nnz": nnz,
            "eff_degree": len(roots), "base_degree": len(base),
            "roots": "tests/golden/c3_poly.json (oracle-built degree-50 GMRES polynomial, "
                     "Leja order, no pof copies needed)",
            "spmv_launches_per_step": count_launches(roots), "parallelism": f"replicas{ws}",
            "l2": "inputs larger than L2 (424 MB matrix stream per SpMV vs 126 MB L2)"}


def count_launches(roots, two_factor=False):
    """Kernel launches of one pi(A)v (gmres_poly.cpp apply_poly_csr): a real
    root is one launch, a pair two; with the two-factor pass (spmv_dia2.cu)
    two consecutive real roots or one pair share a launch."""
    launches = 0
    i = 0
    r = list(roots)
    while i < len(r):
        pair = abs(r[i].imag) > 1e-13 * abs(r[i])
        if pair:
            launches += 1 if two_factor else 2
            i += 2
        elif two_factor and i + 1 < len(r) and abs(r[i + 1].imag) <= 1e-13 * abs(r[i + 1]):
            launches += 1
            i += 2
        else:
            launches += 1
            i += 1
    return launches


# BASELINE config 3 solve settings (configs.py / tests/golden/c3_solve.json)
SOLVE_C3 = {"m": 40, "k": 20, "nev": 15, "degree": 50, "stability": "pof_auto", "seed": 2}
SOLVE_SMALL = {1: {"m": 30, "k": 15, "nev": 10, "degree": 10, "seed": 1},
               2: {"m": 50, "k": 20, "nev": 20, "degree": 25, "seed": 1},
               5: {"m": 30, "k": 15, "nev": 20, "double": (15, 20), "seed": 3,
                   "allow_nev_above_k": True}}


# --------------------------------------------------------------- reference --
def run_reference(args):
    ws, rank, _ = dist_setup(args.gpus)
    if rank != 0:
        return
    from oracle import oracle as O

    threads = os.cpu_count() or 1
    O.set_threads(threads)
    csr = O.Csr.config(3)
    n, nnz, _ = csr.info()
    A = O.csr_operator(csr)
    roots, base = load_golden_poly()
    bspmv = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n
    # size the per-step sample: ~3 s of CPU work (after one warm call)
    O.time_poly_factors(A, roots, 1, 1)
    t1 = O.time_poly_factors(A, roots, 1, 1)
    nf = int(max(1, min(len(roots), 3.0 / max(t1, 1e-3))))
    for _ in range(args.warmup):
        O.time_poly_factors(A, roots, nf, 1)
    times = [O.time_poly_factors(A, roots, nf, 1) for _ in range(args.steps)]
    t = float(np.mean(times))
    gbs = nf * bspmv / t / 1e9
    # time to nev: the oracle's config-3 solve (solve, inc/solver.hpp:91-94),
    # all host threads, same settings as the GPU arm's time_to_nev
    solve_info = None
    if not args.no_solve:
        p = SOLVE_C3
        r = O.solve(A, p["m"], p["k"], p["nev"], degree=p["degree"], stability=True,
                    seed=p["seed"])
        lam = np.sort(r["eigenvalues"].real)
        solve_info = {"seconds": round(r["wall"], 4), "converged": r["converged"],
                      "cycles": r["cycles"], "mvps": r["cost"]["mvps"], "dots": r["cost"]["dots"],
                      "eff_degree": r["composite_degree"], "smallest": round(float(lam[0]), 6),
                      "timing": {"total": round(r["wall"], 4)}, "threads": threads,
                      "params": p}
    # the other converging configs' solves as well (config 1: the reference's
    # own CPU-runnable case; config 2; config 5, solve_double): same settings
    # as the GPU arm's time_to_nev_configs.  Config 4 does not converge in
    # 100 cycles (6.8e3 s of oracle time) and is left out.
    configs_info = None
    if not args.no_solve:
        configs_info = {}
        for k, p in SOLVE_SMALL.items():
            Ak = O.csr_operator(O.Csr.config(k))
            extra = {kk: p[kk] for kk in ("degree", "double", "allow_nev_above_k") if kk in p}
            r = O.solve(Ak, p["m"], p["k"], p["nev"], seed=p["seed"], **extra)
            configs_info[f"config{k}"] = {"seconds": round(r["wall"], 4), "converged": r["converged"],
                                          "cycles": r["cycles"], "mvps": r["cost"]["mvps"]}
    # one orthogonalisation step of arnoldi_extend at the GPU arm's basis size
    # (MGS + MGS reorthogonalisation, src/arnoldi.cpp:129-150), all host threads
    c_cgs = 40
    t_cgs = O.time_mgs2_step(n, c_cgs, 3)
    cgs_info = {"c": c_cgs, "ms": round(t_cgs * 1e3, 3),
                "gbs_model": round(8.0 * n * (3 * c_cgs + 7) / t_cgs / 1e9, 3),
                "bytes_model": "8n(3c+7)", "reps": 3, "threads": threads,
                "what": "MGS + MGS reorthogonalisation + norm + scaled store of "
                        "arnoldi_extend (src/arnoldi.cpp:129-150), oracle restatement"}
    cpu = {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
           "sample": f"{nf} of {len(roots)} polynomial factors (SpMV+axpy) per step, "
                     "oracle restatement of src/gmres_poly.cpp:117-147, OpenMP rows",
           "sample_factors": nf, **cpu_info()}
    line = {
        "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator; BASELINE config 3)", "impl": "reference",
        "config": workload_config(n, nnz, roots, base, ws),
        "cpu_baseline": cpu,
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "cgs2": cgs_info,
        "time_to_nev": solve_info,
        "time_to_nev_configs": configs_info,
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- b200 --
def cpu_baseline_port(roots):
    """Single-thread oracle (the reference's single-threaded contract)."""
    from oracle import oracle as O

    O.set_threads(1)
    csr = O.Csr.config(3)
    n, nnz, _ = csr.info()
    A = O.csr_operator(csr)
    bspmv = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n
    O.time_poly_factors(A, roots, 1, 1)
    t1 = O.time_poly_factors(A, roots, 1, 1)
    nf = int(max(1, min(len(roots), 10.0 / max(t1, 1e-3))))
    t = O.time_poly_factors(A, roots, nf, 1)
    # one orthogonalisation step at c = 40 (MGS2, src/arnoldi.cpp:129-150)
    t_cgs = O.time_mgs2_step(n, 40, 1)
    return {"value": round(nf * bspmv / t / 1e9, 3), "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"{nf} of {len(roots)} factors of pi(A)v on config 3 "
                      f"({t:.1f} s, single thread, oracle -O3)",
            "cgs2_step_ms": round(t_cgs * 1e3, 2),
            "cgs2_step_gbs_model": round(8.0 * n * (3 * 40 + 7) / t_cgs / 1e9, 3),
            "cgs2_sample": "one MGS2 orthogonalisation step at c = 40 on config 3's n "
                           "(single thread, oracle)", **cpu_info()}


def run_b200(args):
    import torch

    ws, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1806_08020_b200 as ppa

    stream = torch.cuda.current_stream()
    ppa.set_stream(stream)
    clk = ClockSampler(local).start()
    t0 = time.time()
    csr = ppa.CsrMatrix.config(3)
    n, nnz, _ = csr.info()
    # headline: SELL-32 with fp64 values and int32 columns, the layout the
    # north-star byte model describes; the default (automatic) layout is
    # measured the same way below under "default_layout"
    A = ppa.make_csr_operator(csr, "sell32")
    A_auto = ppa.make_csr_operator(csr)
    bspmv = A.model_bytes()
    b = torch.tensor(ppa.normal_vector(n, 2, ppa.STREAM_POLY), device="cuda")
    dev_base, _ = ppa.build_gmres_poly(A, b, 50)
    dev_roots = ppa.add_stability_roots(dev_base, len(dev_base))
    setup_s = time.time() - t0
    # both arms apply the oracle-built root set (the device-built one agrees
    # to roundoff, reported as poly_check)
    roots, base = load_golden_poly()
    poly_check = {"same_count": len(dev_roots) == len(roots),
                  "max_rel_diff": (float(np.max(np.abs(dev_roots - roots) / np.abs(roots)))
                                   if len(dev_roots) == len(roots) else None)}
    launches = count_launches(roots)
    step_bytes = len(roots) * bspmv

    v = torch.tensor(ppa.normal_vector(n, 2, ppa.STREAM_ARNOLDI), device="cuda")
    out = torch.empty(n, dtype=torch.float64, device="cuda")

    def time_pi(op):
        def step():
            ppa.apply_poly(roots, op, v, out)

        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with clk.region():
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
        ms = reduce_max(e0.elapsed_time(e1), ws, "cuda")
        if ws > 1:
            dist.barrier()
        return ms / args.steps

    # e2e: pinned host buffers through the C-ABI batch call: every step does the
    # H2D of its input vector, pi(A)v and the D2H of its result; the copies of
    # neighbouring steps overlap the compute (double-buffered, three streams).
    # pinned host batches shared by both e2e measurements (at most 32 steps:
    # 2 x 32 x 33 MB pinned instead of 2 x steps x 33 MB)
    ke = max(2, min(args.steps, 32))
    xh = torch.empty((ke, n), dtype=torch.float64).pin_memory()
    xh[:] = torch.from_numpy(ppa.normal_vector(n, 2, ppa.STREAM_ARNOLDI))
    yh = torch.empty((ke, n), dtype=torch.float64).pin_memory()

    def time_e2e(op_base):
        op = ppa.make_poly_operator(op_base, roots, len(base))
        op.apply_host_batch(xh[:2], yh[:2])  # warm-up
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        with clk.region():
            f0.record(stream)
            op.apply_host_batch(xh, yh)
            f1.record(stream)
            torch.cuda.synchronize()
        e_ms = reduce_max(f0.elapsed_time(f1) / ke, ws, "cuda")
        match = bool(np.array_equal(yh[ke - 1].numpy(), out.cpu().numpy()))
        return e_ms, match

    ms_step = time_pi(A)
    value = whole_job_gbs(step_bytes, ms_step, ws)
    avg_launch_ms = ms_step / launches
    achieved = bspmv / (avg_launch_ms * 1e-3) / 1e9
    peak, peak_kind = hbm_peak()
    ref_out = out.clone()
    e2e_ms, e2e_match = time_e2e(A)
    e2e_val = whole_job_gbs(step_bytes, e2e_ms, ws)

    # the default layout on the same workload (bit-identical output)
    lay = A_auto.layout()
    ms_auto = time_pi(A_auto)
    auto_match = bool(torch.equal(out, ref_out))
    e2e_auto_ms, e2e_auto_match = time_e2e(A_auto)
    two = bool(lay.get("two_factor_pass"))
    auto_launches = count_launches(roots, two)
    auto_launch_s = ms_auto * 1e-3 / auto_launches
    if two and lay.get("grid_pass"):
        # box-grid two-factor pass: x read once (8n), the second factor's y
        # written once (8n); no matrix bytes at all
        kbytes = 16.0 * n
        kname = ("k_spmv_grid2 (two factors per pass over the box-grid stencil: x planes by "
                 "cp.async.bulk into a shared-memory ring, per-warp mbarrier split barriers)")
        note = ("8n x + 8n y per two-factor launch; bound on the SM side (16 DP ops per row per "
                "factor in the bit-exact mul-then-add order, issue, per-step lockstep of the "
                "warps; DESIGN.md 3.1c), not by HBM")
    elif two:
        # two factors per launch: x read once (8n), the second factor's y
        # written once (8n), one presence byte per row (n)
        kbytes = 17.0 * n
        kname = ("k_spmv_dia2 (two factors per pass: temporally blocked diagonal form, "
                 "x planes by cp.async.bulk into a shared-memory ring)")
        note = ("8n x + 8n y + n presence per two-factor launch; the kernel is issue-bound "
                "(~67% issue slots busy, ncu), not HBM-bound")
    else:
        kbytes = lay["stream_bytes"] + 16.0 * n  # + x gather (8n) + y store (8n)
        kname = ("k_spmv_diam (regular-row diagonal form, marching over the +-plane "
                 "diagonals, fused real-root factor)")
        note = "matrix stream of this layout + 8n x + 8n y"
    default_layout = {
        "layout": lay["layout"], "ms_per_step": round(ms_auto, 4),
        "value": round(whole_job_gbs(step_bytes, ms_auto, ws), 3), "unit": "GB/s (north-star model)",
        "speedup_vs_sell32": round(ms_step / ms_auto, 3),
        "two_factor_pass": two, "launches_per_step": auto_launches,
        "us_per_factor": round(ms_auto * 1e3 / len(roots), 3),
        "e2e": {"value": round(whole_job_gbs(step_bytes, e2e_auto_ms, ws), 3),
                "ms_per_step": round(e2e_auto_ms, 4), "matches_device_result": e2e_auto_match},
        "roofline": {"bound": "hbm", "achieved": round(kbytes / auto_launch_s / 1e9, 2),
                     "peak": peak, "unit": "GB/s",
                     "frac": round(kbytes / auto_launch_s / 1e9 / peak, 4),
                     "kernel": kname,
                     "algorithmic_bytes_per_launch": kbytes,
                     "bytes_note": note},
        "bit_identical_to_sell32": auto_match,
    }
    rows = lay.get("grid_rows_per_pass")
    if two and rows and not any(abs(z.imag) > 1e-13 * abs(z) for z in roots):
        # the box-grid pass's FP64 view: every row evaluation is nd mul + nd
        # add (the sum starts at +0.0) plus the real-root epilogue's mul + add,
        # no FMA (bit-exact mul-then-add order); peak = the measured non-FMA
        # DADD/DMUL rate (tools/micro/fp64_rate.cu: 61.7 lane-ops per clock per
        # SM at 1965 MHz on this pool's B200)
        nd = 7 if lay["grid"][1] > 1 else 5
        flop = float(rows[0] + rows[1]) * (2 * nd + 2)
        fp64_peak = 61.7 * 148 * 1.965e9 / 1e12
        ach = flop / auto_launch_s / 1e12
        default_layout["fp64"] = {
            "bound": "fp64 pipe (no FMA)", "achieved": round(ach, 3), "peak": round(fp64_peak, 2),
            "unit": "TFLOP/s", "frac": round(ach / fp64_peak, 4),
            "flop_per_launch": flop, "row_evaluations_per_launch": list(rows),
            "peak_kind": "measured, tools/micro/fp64_rate.cu"}

    # CGS2 step at basis size c = 40 (config 3's m) on a real Arnoldi basis of
    # A: w = A v_39 orthogonalised against V[:,0:40] (3 sweeps, V[:,40] written).
    c = 40
    st = ppa.arnoldi_init(v, n, c)
    st.extend(A, c)
    ld = st.ld
    Vt = torch.empty(0, dtype=torch.float64, device="cuda")
    w0 = torch.empty(n, dtype=torch.float64, device="cuda")
    ppa.spmv(A, st.V_ptr + 8 * ld * (c - 1), w0)
    w = torch.empty_like(w0)
    Hc = torch.empty(c + 2, dtype=torch.float64, device="cuda")
    flag = torch.zeros(2, dtype=torch.int32, device="cuda")
    reps = 10
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps + 3)]
    for i, (g0, g1) in enumerate(evs):
        w.copy_(w0)
        g0.record(stream)
        ppa.cgs2_step(st.V_ptr, ld, n, c, w, Hc, flag)
        g1.record(stream)
    torch.cuda.synchronize()
    cgs_ms = float(np.mean([g0.elapsed_time(g1) for g0, g1 in evs[3:]]))
    cgs_flag = int(flag[0].item())
    cgs_gbs = 8.0 * n * (3 * c + 7) / (cgs_ms * 1e-3) / 1e9
    cgs_phys = 8.0 * n * (3 * c + 5) / (cgs_ms * 1e-3) / 1e9
    del st, Vt

    # time to nev converged eigenpairs (config 3, matrix already on device):
    # default layout, and the SELL-32 layout for comparison
    solve_info = configs_info = None
    if not args.no_solve:
        cfg = ppa.config_solve_config(3)

        warm = ppa.config_solve_config(3)
        warm.max_cycles = 1

        def solve_on(op):
            # one-cycle warm-up solve first: loads every kernel the solve uses
            # (lazy module loading) so the timed solve measures the solver
            ppa.solve(op, warm)
            with clk.region():
                r = ppa.solve(op, cfg)
            lam = np.sort(r["eigenvalues"].real)
            return {"seconds": round(r["timing"]["total"], 4), "converged": r["converged"],
                    "cycles": r["cycles"], "mvps": r["cost"]["mvps"], "dots": r["cost"]["dots"],
                    "eff_degree": r["composite_degree"], "smallest": round(float(lam[0]), 6),
                    "timing": {k: round(v, 4) for k, v in r["timing"].items()}}

        solve_info = solve_on(A_auto)
        solve_info["layout"] = lay["layout"]
        configs_info = {}
        for k in SOLVE_SMALL:
            Ak = ppa.make_csr_operator(ppa.CsrMatrix.config(k))
            ck, wk = ppa.config_solve_config(k), ppa.config_solve_config(k, max_cycles=1)
            sk = ppa.solve_double if k == 5 else ppa.solve
            sk(Ak, wk)
            with clk.region():
                rk = sk(Ak, ck)
            configs_info[f"config{k}"] = {"seconds": round(rk["timing"]["total"], 4),
                                          "converged": rk["converged"], "cycles": rk["cycles"],
                                          "mvps": rk["cost"]["mvps"],
                                          "timing": {kk: round(vv, 4)
                                                     for kk, vv in rk["timing"].items()}}
        solve_info["orthogonalization"] = cfg.orthogonalization
        solve_info["sell32"] = solve_on(A)
        # classical CGS2 (three sweeps over V per step instead of the default
        # delayed CGS2's two): same eigenpairs and cycle count
        cfg.orthogonalization = "cgs2"
        warm.orthogonalization = "cgs2"
        solve_info["cgs2"] = solve_on(A_auto)

    clk.stop()
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_port(roots)

    traffic = None
    tfile = os.path.join(ROOT, "profiles", "spmv_traffic.json")
    if os.path.exists(tfile):
        with open(tfile) as f:
            traffic = json.load(f).get("traffic_bytes_per_launch")

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator; BASELINE config 3)",
            "config": workload_config(n, nnz, roots, base, ws),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "kernel": "k_spmv_sell32 (fused real-root factor)",
                         "algorithmic_bytes_per_launch": bspmv,
                         # the byte model counts row_ptr (16.4 MB) that SELL-32 never
                         # reads; the ncu DRAM bytes per launch over the same time:
                         "traffic_gbs": (round(traffic / (avg_launch_ms * 1e-3) / 1e9, 2)
                                         if traffic else None),
                         "traffic_frac": (round(traffic / (avg_launch_ms * 1e-3) / 1e9 / peak, 4)
                                          if traffic else None)},
            # e2e: the call a user makes - make_csr_operator(A) (automatic
            # layout), make_poly_operator, apply with host vectors through the
            # C-ABI (ppa_op_apply_host_batch); H2D of v and D2H of pi(A)v in the
            # timed region.  Same metric and unit as `value` (north-star bytes
            # per pi(A)v); the SELL-32 layout's e2e is e2e_sell32.
            "e2e": {"value": round(whole_job_gbs(step_bytes, e2e_auto_ms, ws), 3), "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "ms_per_step": round(e2e_auto_ms, 4), "steps": ke,
                    "layout": lay["layout"] + " (automatic, make_csr_operator default)",
                    "matches_device_result": e2e_auto_match},
            "e2e_sell32": {"value": round(e2e_val, 3), "unit": "GB/s", "ms_per_step": round(e2e_ms, 4),
                           "matches_device_result": e2e_match},
            "default_layout": default_layout,
            "gpu_launches": launches * args.steps,
            "layout": "sell32 (fp64 values, int32 columns)",
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "cgs2": {"c": c, "gbs_model": round(cgs_gbs, 2), "ms": round(cgs_ms, 4),
                     "frac": round(cgs_gbs / peak, 4), "bytes_model": "8n(3c+7)",
                     "gbs_moved": round(cgs_phys, 2), "bytes_moved": "8n(3c+5)",
                     "breakdown_flag": cgs_flag},
            "time_to_nev": solve_info,
            "time_to_nev_configs": configs_info,
            "setup_seconds": round(setup_s, 3),
            "poly_check": poly_check,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def run_sharded(args):
    """Strong scaling of config-3 pi(A)v over row blocks (dist.py): every rank
    owns n/N rows and exchanges halos per SpMV.  Not the driver's contract
    (that is the replica run above); for maintainers with several GPUs."""
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(ws))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1806_08020_b200 as ppa
    from paper_1806_08020_b200.dist import CudaBackend, HaloPlan, ShardedPoly

    stream = torch.cuda.current_stream()
    ppa.set_stream(stream)
    csr = ppa.CsrMatrix.config(3)
    n, nnz, _ = csr.info()
    bspmv = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n
    roots, _ = load_golden_poly()
    if args.grid:
        # z-slabs, halo planes copied by the pass kernel from the neighbours'
        # buffers (dist.ShardedGridPoly)
        from paper_1806_08020_b200.dist import ShardedGridPoly, box_row_ranges

        rp, ci, va = csr.arrays()
        mid = (80 * 160 + 80) * 160 + 80  # an interior row: the 7 diagonal values in order
        sp = ShardedGridPoly(160, 160, 160, [float(t) for t in va[rp[mid]:rp[mid + 1]]], dist)
        r0, r1 = box_row_ranges(160, 160, 160, ws)[rank]
        halo_rows = 4 * 160 * 160
        halo = "fused: the pass kernel copies the neighbours' halo planes (CUDA IPC, epoch flags)"
    else:
        plan = HaloPlan.build(*csr.arrays(), n, dist)
        sp = ShardedPoly(plan, CudaBackend(plan), dist, peer=args.peer)
        r0, r1 = plan.ranges[rank]
        halo_rows = plan.n_left + plan.n_right
        halo = "peer memory (CUDA IPC, epoch flags)" if args.peer else "NCCL point-to-point"
    v = torch.tensor(ppa.normal_vector(n, 2, ppa.STREAM_ARNOLDI)[r0:r1], device="cuda")
    for _ in range(max(args.warmup, 3)):
        sp.apply(roots, v)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        sp.apply(roots, v)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = reduce_max(e0.elapsed_time(e1), ws, "cuda") / args.steps
    if rank == 0:
        print(json.dumps({
            "metric": METRIC + " (row-block sharded)", "value": round(len(roots) * bspmv / (ms * 1e-3) / 1e9, 3),
            "unit": "GB/s", "n_gpus": ws, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "dtype": "f64", "data": "synthetic (seeded generator; BASELINE config 3)",
            "config": {"workload": "config3-laplace3d-160^3-pi(A)v", "parallelism": f"rowblock{ws}",
                       "halo_rows_per_rank": halo_rows, "halo": halo},
        }), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="strong-scaling row-block sharded pi(A)v (dist.py) instead of replicas")
    ap.add_argument("--grid", action="store_true",
                    help="with --sharded: z-slab box-grid passes with the halo fused into the kernel")
    ap.add_argument("--peer", action="store_true",
                    help="with --sharded: halos over peer memory (dist.PeerHalo) instead of NCCL")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.sharded:
        run_sharded(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
