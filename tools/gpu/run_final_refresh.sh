# last refresh of the round: full GPU suite, smoke, both bench arms (plain runs, no profiler)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(time python -m pytest tests -m gpu -x -q) > gpurun_out/p5_gputest.log 2>&1
tail -4 gpurun_out/p5_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p5_smoke.log 2>&1; tail -1 gpurun_out/p5_smoke.log
python bench.py > gpurun_out/p5_bench.jsonl 2> gpurun_out/p5_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/p5_bench_ref.jsonl 2> gpurun_out/p5_bench_ref.err; echo "ref rc=$?"
tail -c 400 gpurun_out/p5_bench.jsonl; tail -c 400 gpurun_out/p5_bench_ref.jsonl
