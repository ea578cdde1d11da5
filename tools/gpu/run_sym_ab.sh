cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_rate tools/micro/fp64_rate.cu && /tmp/fp64_rate > gpurun_out/fp64_rate.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_dia2.py -x -q -k "grid2" > gpurun_out/s1_tests.log 2>&1
tail -3 gpurun_out/s1_tests.log
export PPA_GRID2_DEBUG=1
timeout 600 python tools/spmv_ab.py 3 "" PPA_GRID2_SYM=0 PPA_GRID2_RY=2,PPA_GRID2_TY=6 PPA_GRID2_RY=2,PPA_GRID2_TY=10 PPA_GRID2_RY=3,PPA_GRID2_TY=10 PPA_GRID2_RY=3,PPA_GRID2_TY=4 PPA_GRID2_RY=4,PPA_GRID2_TY=6 PPA_GRID2_RY=2,PPA_GRID2_TY=8 > gpurun_out/s1_ab.log 2>&1
cat gpurun_out/fp64_rate.txt gpurun_out/s1_ab.log
