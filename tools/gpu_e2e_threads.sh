B="python bench.py --no-cpu-baseline --no-algo1 --no-sweep"
for t in 16 8 4; do
  FSLD_HOST_THREADS=$t $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('threads $t bench e2e ms', round(d['e2e']['ms_per_step'],3))"
  FSLD_HOST_THREADS=$t PYTHONPATH=. python tools/e2e_iters.py 8192 2>&1 | tail -1 | python -c "import sys; v=[float(x) for x in sys.stdin.read().split(':')[1].split()]; import statistics; print('threads $t iters median(last 30)', statistics.median(v[-30:]))"
done
