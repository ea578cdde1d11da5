set -x
bash tools/prof_round.sh > gpurun_out/pr.log 2>&1; echo pr_rc=$? >> gpurun_out/pr.log
bash tools/prof_dia2.sh > gpurun_out/pd.log 2>&1; echo pd_rc=$? >> gpurun_out/pd.log
python tools/summarize_ncu.py launches gpurun_out/pr_launches.csv gpurun_out/S_bench_launches.md
python tools/summarize_ncu.py launches gpurun_out/pd_solve_launches.csv gpurun_out/S_solve_launches.md
python tools/summarize_ncu.py kernels gpurun_out/pr_sell32.ncu-rep gpurun_out/S_sell32.md "k_spmv_sell32, config 3 (headline layout)"
python tools/summarize_ncu.py kernels gpurun_out/pr_diam.ncu-rep gpurun_out/S_diam.md "k_spmv_diam, config 3, single-factor diagonal kernel"
python tools/summarize_ncu.py kernels gpurun_out/pr_cgs.ncu-rep gpurun_out/S_cgs.md "CGS2 sweeps (k_tspipe), config 3, c = 40"
for c in 3 5 2; do python tools/summarize_ncu.py kernels gpurun_out/pd_dia2_c$c.ncu-rep gpurun_out/S_dia2_c$c.md "k_spmv_dia2, config $c, two factors per launch"; done
mkdir -p /tmp/keep; mv gpurun_out/pd_dia2_c3.ncu-rep /tmp/keep/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
python - <<'P'
import csv,subprocess
P
ls -la gpurun_out; du -sh gpurun_out
