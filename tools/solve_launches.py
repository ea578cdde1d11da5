"""One solve of a BASELINE config after a warm-up solve of the same config,
for an ncu launch list of the time-to-nev path only (the profiler range
covers the timed solve; run ncu with --profile-from-start off):

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \\
        --csv --log-file gpurun_out/solve_launches.csv python tools/solve_launches.py 3
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1806_08020_b200 as ppa

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
A = ppa.make_csr_operator(ppa.CsrMatrix.config(k))
warm = ppa.config_solve_config(k, max_cycles=1)
(ppa.solve_double if k == 5 else ppa.solve)(A, warm)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = (ppa.solve_double if k == 5 else ppa.solve)(A, ppa.config_solve_config(k))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(r["converged"], r["cycles"], r["timing"])
