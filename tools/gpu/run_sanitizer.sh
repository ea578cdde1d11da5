# compute-sanitizer over every kernel family at small sizes (tools/sanitize_paths.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 600 python tools/sanitize_paths.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -3 gpurun_out/san_plain.log
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 40 --error-exitcode 7 \
      python tools/sanitize_paths.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|all parts done" gpurun_out/san_$tool.log | tail -3
done
