# V*G: bit-identity of the TMA-fed and register kernels, then timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ts_combine" > gpurun_out/comb_tests.log 2>&1
tail -2 gpurun_out/comb_tests.log
timeout 300 python tools/combine_bench.py > gpurun_out/comb_tma.log 2>&1
PPA_COMBINE_TMA=0 timeout 300 python tools/combine_bench.py > gpurun_out/comb_reg.log 2>&1
echo TMA; cat gpurun_out/comb_tma.log; echo REG; cat gpurun_out/comb_reg.log
