# Round-2 refresh after the grid2 store-path change and the pinned-pool fix
# (one GPU; every ncu command first runs without ncu).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/p3
(time python -m pytest tests -m gpu -x -q) > gpurun_out/p3_gputest.log 2>&1
tail -3 gpurun_out/p3_gputest.log
python bench.py > gpurun_out/p3_bench.log 2>&1
tail -c 400 gpurun_out/p3_bench.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p3_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/p3_launch.log 2>&1
python tools/solve_launches.py 3 > gpurun_out/p3_solve_plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/p3_solve3_launches.csv python tools/solve_launches.py 3 > gpurun_out/p3_solve3.log 2>&1
python tools/prof_kernels.py spmv auto > /dev/null 2>&1
for c in 3 5; do
  PPA_PROF_CONFIG=$c ncu --set full --clock-control none --import-source on -k regex:k_spmv_grid2 -s 2 -c 1 \
      -o /tmp/p3/p3_grid2_c$c python tools/prof_kernels.py spmv auto > gpurun_out/p3_ncu_g$c.log 2>&1
done
python tools/summarize_ncu.py launches gpurun_out/p3_bench_launches.csv gpurun_out/p3_bench_launches.md
python tools/summarize_ncu.py launches gpurun_out/p3_solve3_launches.csv gpurun_out/p3_solve3_launches.md
for r in /tmp/p3/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_digest.py $r 25 > gpurun_out/${b}_digest.txt 2>&1 || true
  python tools/summarize_ncu.py kernels $r gpurun_out/${b}.md $b || true
done
python tools/config_report.py 1 2 3 5 > gpurun_out/p3_configs.jsonl 2> gpurun_out/p3_configs.err
ls -la gpurun_out/p3_*
