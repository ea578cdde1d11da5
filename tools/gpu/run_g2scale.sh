cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; PPA_GRID2_DEBUG=1 python tools/grid2_scaling.py > gpurun_out/g2scale.log 2>&1; cat gpurun_out/g2scale.log
