# Round-2 final refresh (one GPU; every ncu command first runs without ncu).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/p4
(time python -m pytest tests -m gpu -x -q) > gpurun_out/p4_gputest.log 2>&1
tail -3 gpurun_out/p4_gputest.log
python bench.py > gpurun_out/p4_bench.log 2>&1
tail -c 300 gpurun_out/p4_bench.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p4_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/p4_launch.log 2>&1
python tools/solve_launches.py 3 > gpurun_out/p4_solve_plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/p4_solve3_launches.csv python tools/solve_launches.py 3 > gpurun_out/p4_solve3.log 2>&1
python tools/prof_kernels.py all auto > /dev/null 2>&1
for c in 3 5; do
  PPA_PROF_CONFIG=$c ncu --set full --clock-control none --import-source on -k regex:k_spmv_grid2 -s 2 -c 1 \
      -o /tmp/p4/p4_grid2_c$c python tools/prof_kernels.py spmv auto > gpurun_out/p4_ncu_g$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_combine_tma -s 1 -c 1 \
    -o /tmp/p4/p4_combine python tools/prof_kernels.py cgs sell32 > gpurun_out/p4_ncu_comb.log 2>&1
python tools/summarize_ncu.py launches gpurun_out/p4_bench_launches.csv gpurun_out/p4_bench_launches.md
python tools/summarize_ncu.py launches gpurun_out/p4_solve3_launches.csv gpurun_out/p4_solve3_launches.md
for r in /tmp/p4/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_digest.py $r 25 > gpurun_out/${b}_digest.txt 2>&1 || true
  python tools/summarize_ncu.py kernels $r gpurun_out/${b}.md $b || true
done
python tools/config_report.py 1 2 3 5 > gpurun_out/p4_configs.jsonl 2> gpurun_out/p4_configs.err
python tools/combine_bench.py > gpurun_out/p4_combine.jsonl 2>&1
python bench.py --sharded --grid --steps 20 > gpurun_out/p4_sharded_grid.log 2>&1
ls -la gpurun_out/p4_*
