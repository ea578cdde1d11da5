cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather4_rate tools/micro/gather4_rate.cu -lcuda
timeout 120 /tmp/gather4_rate 1 > gpurun_out/gather4_1.txt 2>&1; echo rc=$? >> gpurun_out/gather4_1.txt

cat gpurun_out/gather4_1.txt
