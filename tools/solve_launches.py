"""One config-3 solve (after a warm-up solve), for an ncu launch list of the
whole time-to-nev path:

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \\
        --log-file gpurun_out/solve_launches.csv python tools/solve_launches.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_08020_b200 as ppa

ppa.solve(ppa.make_csr_operator(ppa.CsrMatrix.config(1)), ppa.config_solve_config(1))
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
r = ppa.solve(ppa.make_csr_operator(ppa.CsrMatrix.config(k)), ppa.config_solve_config(k))
print(r["converged"], r["cycles"], r["timing"])
