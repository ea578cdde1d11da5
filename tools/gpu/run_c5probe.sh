cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; python tools/c5_bench_probe.py > gpurun_out/c5probe.log 2>&1; cat gpurun_out/c5probe.log
