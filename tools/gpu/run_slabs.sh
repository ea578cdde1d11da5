# fused-halo slab passes: bit-exact tests, then the box-grid suite (regression) and timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_grid_slabs.py -x -q > gpurun_out/slab_tests.log 2>&1
tail -15 gpurun_out/slab_tests.log
timeout 900 python -m pytest tests/test_gpu_dia2.py -x -q > gpurun_out/g2_tests.log 2>&1
tail -2 gpurun_out/g2_tests.log
for c in 3 5 2; do
  timeout 300 python tools/spmv_ab.py $c "" > gpurun_out/g2_ab_$c.log 2>&1
  python -c "
import json
for l in open('gpurun_out/g2_ab_$c.log'):
    d = json.loads(l); r = d['result']
    try: r = json.loads(r); print('config $c', d['variant'], round(r['us_per_spmv'], 3), r['checksum'])
    except Exception: print('config $c', d['variant'], r[-300:])
"
done
