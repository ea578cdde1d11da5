# Two-factor pass captures (one GPU; each command first runs without ncu).
set -e
mkdir -p gpurun_out
python tools/solve_launches.py 3 > gpurun_out/pd_solve_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pd_solve_launches.csv \
    python tools/solve_launches.py 3 > gpurun_out/pd_solve.log 2>&1
for c in 3 5 2; do
  PPA_PROF_CONFIG=$c python tools/prof_kernels.py spmv auto > /dev/null 2>&1
  PPA_PROF_CONFIG=$c ncu --set full --clock-control none --import-source on -k regex:k_spmv_dia2 -s 2 -c 1 \
      -o gpurun_out/pd_dia2_c$c python tools/prof_kernels.py spmv auto > gpurun_out/pd_ncu_c$c.log 2>&1
done
ls -la gpurun_out/pd_*
