# A/B of the box-grid pass's cells-per-thread / thread-count plans (config 3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PPA_GRID2_DEBUG=1
timeout 600 python tools/spmv_ab.py 3 "" PPA_GRID2_RY=2,PPA_GRID2_TY=10 PPA_GRID2_RY=4,PPA_GRID2_TY=10 PPA_GRID2_RY=2,PPA_GRID2_TY=8 PPA_GRID2_RY=2,PPA_GRID2_TY=12 PPA_GRID2_RY=3,PPA_GRID2_TY=13 > gpurun_out/ry_ab.log 2>&1
cat gpurun_out/ry_ab.log | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); r = d['result']
    try: us = json.loads(r)['us_per_spmv']
    except Exception: us = r[-120:]
    print(d['variant'], us, d['plans'])
"
