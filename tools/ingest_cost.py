"""Operator construction cost per layout (host validation + layout build +
upload), config 3 and config 4, after a warm-up.

    python tools/ingest_cost.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1806_08020_b200 as ppa

torch.cuda.init()
ppa.make_csr_operator(ppa.CsrMatrix.config(1))
for k in (3, 4, 2):
    t = time.perf_counter()
    m = ppa.CsrMatrix.config(k)
    gen = time.perf_counter() - t
    for lay in ("auto", "csr", "sell32", "sell32_packed", "dia_coded"):
        t = time.perf_counter()
        A = ppa.make_csr_operator(m, lay)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(json.dumps({"config": k, "cap": lay, "layout": A.layout()["layout"],
                          "build_s": round(dt, 4), "generate_s": round(gen, 3)}), flush=True)
        del A
