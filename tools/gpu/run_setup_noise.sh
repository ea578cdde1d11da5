cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; python tools/setup_noise.py > gpurun_out/setup_noise.log 2>&1; cat gpurun_out/setup_noise.log; nproc; cat /proc/loadavg
