# box-grid pass after a kernel change: bit-exact tests, then per-factor times on configs 3, 5, 2 (twice)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dia2.py tests/test_gpu_fullsize.py tests/test_gpu_guard.py -x -q > gpurun_out/g2chk_tests.log 2>&1
tail -3 gpurun_out/g2chk_tests.log
for rep in 1 2; do
for c in 3 5 2; do
  timeout 300 python tools/spmv_ab.py $c "" $G2_VARIANTS > gpurun_out/g2chk_ab_$c.log 2>&1
  python -c "
import json
for l in open('gpurun_out/g2chk_ab_$c.log'):
    d = json.loads(l); r = d['result']
    try: r = json.loads(r); print('rep $rep config $c', d['variant'], round(r['us_per_spmv'], 3), r['checksum'])
    except Exception: print('config $c', d['variant'], r[-300:])
"
done
done
