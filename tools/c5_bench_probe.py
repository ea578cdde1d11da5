"""Config 2 / 5 time to nev standalone and after a config-3 solve in the same
process (the bench runs them in that order), with the solve's phase timings.

    python tools/c5_bench_probe.py
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1806_08020_b200 as ppa  # noqa: E402

torch.cuda.set_device(0)
ppa.set_stream(torch.cuda.current_stream())


def run(k, tag):
    A = ppa.make_csr_operator(ppa.CsrMatrix.config(k))
    c, w = ppa.config_solve_config(k), ppa.config_solve_config(k, max_cycles=1)
    s = ppa.solve_double if k == 5 else ppa.solve
    s(A, w)
    for rep in range(2):
        t = time.perf_counter()
        r = s(A, c)
        print(json.dumps({"tag": tag, "config": k, "rep": rep, "wall": round(time.perf_counter() - t, 4),
                          "timing": {a: round(b, 4) for a, b in r["timing"].items()},
                          "cycles": r["cycles"]}), flush=True)


run(5, "first")
run(2, "first")
run(3, "config3")
run(5, "after3")
run(2, "after3")
