# repeated per-factor timings (noise level of tools/spmv_ab.py)
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  for c in 3 5; do
    timeout 300 python tools/spmv_ab.py $c "" 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); r = json.loads(d['result']); print('rep $rep config $c', round(r['us_per_spmv'], 3))
"
  done
done
