# Profiles committed under profiles/ (one GPU; each command first runs without ncu).
set -e
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/pr_bench_plain.log 2>&1
# launch list of the bench command (cold-cache, serialised; shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pr_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/pr_launch.log 2>&1
python tools/prof_kernels.py all sell32 > /dev/null 2>&1
# full captures: headline SpMV (SELL-32), default-layout SpMV, CGS2 sweeps
ncu --set full --clock-control none --import-source on -k regex:k_spmv_sell32 -s 2 -c 1 \
    -o gpurun_out/pr_sell32 python tools/prof_kernels.py spmv sell32 > gpurun_out/pr_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_spmv_dia -s 2 -c 1 \
    -o gpurun_out/pr_diam python tools/prof_kernels.py spmv auto > gpurun_out/pr_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tspipe -s 6 -c 5 \
    -o gpurun_out/pr_cgs python tools/prof_kernels.py cgs sell32 > gpurun_out/pr_ncu3.log 2>&1
ls -la gpurun_out/pr_*
