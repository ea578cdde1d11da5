# Round-2 profiles (one GPU; every command first runs without ncu).
set -e
mkdir -p gpurun_out /tmp/p2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/p2_bench_plain.log 2>&1
# launch list of the bench command (cold-cache, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p2_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/p2_launch.log 2>&1
# launch list of one config-3 solve (the profiler range covers the timed solve only)
python tools/solve_launches.py 3 > gpurun_out/p2_solve_plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/p2_solve3_launches.csv python tools/solve_launches.py 3 > gpurun_out/p2_solve3.log 2>&1
python tools/solve_launches.py 5 > gpurun_out/p2_solve5_plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/p2_solve5_launches.csv python tools/solve_launches.py 5 > gpurun_out/p2_solve5.log 2>&1
python tools/prof_kernels.py all sell32 > /dev/null 2>&1
# full captures: headline SpMV (SELL-32), the box-grid two-factor pass (configs 3, 5, 2), CGS2 sweeps, V*G
ncu --set full --clock-control none --import-source on -k regex:k_spmv_sell32 -s 2 -c 1 \
    -o /tmp/p2/p2_sell32 python tools/prof_kernels.py spmv sell32 > gpurun_out/p2_ncu1.log 2>&1
for c in 3 5 2; do
  PPA_PROF_CONFIG=$c ncu --set full --clock-control none --import-source on -k regex:k_spmv_grid2 -s 2 -c 1 \
      -o /tmp/p2/p2_grid2_c$c python tools/prof_kernels.py spmv auto > gpurun_out/p2_ncu_g$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_tspipe -s 6 -c 3 \
    -o /tmp/p2/p2_cgs python tools/prof_kernels.py cgs sell32 > gpurun_out/p2_ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ts_combine -s 1 -c 1 \
    -o /tmp/p2/p2_combine python tools/prof_kernels.py cgs sell32 > gpurun_out/p2_ncu4.log 2>&1
# summaries into gpurun_out (the .ncu-rep files stay in /tmp: gpurun_out is capped at 64 MiB)
python tools/summarize_ncu.py launches gpurun_out/p2_bench_launches.csv gpurun_out/p2_bench_launches.md
python tools/summarize_ncu.py launches gpurun_out/p2_solve3_launches.csv gpurun_out/p2_solve3_launches.md
python tools/summarize_ncu.py launches gpurun_out/p2_solve5_launches.csv gpurun_out/p2_solve5_launches.md
for r in /tmp/p2/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_digest.py $r 25 > gpurun_out/${b}_digest.txt 2>&1 || true
  python tools/summarize_ncu.py kernels $r gpurun_out/${b}.md $b || true
done
cp /tmp/p2/p2_grid2_c3.ncu-rep gpurun_out/ || true
ls -la gpurun_out/p2_*
