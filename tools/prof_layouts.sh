set -x
for L in sell32 sell32_packed auto; do
  ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 2 -c 1 -o gpurun_out/r01_spmv_$L python tools/prof_kernels.py spmv $L > gpurun_out/ncu_$L.log 2>&1
done
PPA_DISABLE_DIA_REGULAR=1 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 2 -c 1 -o gpurun_out/r01_spmv_dia_coded python tools/prof_kernels.py spmv auto > gpurun_out/ncu_diacoded.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/bench_nolaunch.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/ncu_launch.log 2>&1
ls gpurun_out
