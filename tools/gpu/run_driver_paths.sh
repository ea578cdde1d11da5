cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4_smoke.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/s4_bench_torchrun.jsonl 2> gpurun_out/s4_bench_torchrun.err; echo "torchrun bench rc=$?"; tail -c 600 gpurun_out/s4_bench_torchrun.jsonl
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/s4_ref_torchrun.jsonl 2> gpurun_out/s4_ref_torchrun.err; echo "torchrun ref rc=$?"; tail -c 900 gpurun_out/s4_ref_torchrun.jsonl
