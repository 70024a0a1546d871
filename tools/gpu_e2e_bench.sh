B="python bench.py --no-cpu-baseline --no-algo1 --no-sweep"
$B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench e2e ms', d['e2e']['ms_per_step'], 'c_abi', d['e2e']['c_abi']['ms_per_step'])"
OMP_NUM_THREADS=1 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('OMP1 bench e2e ms', d['e2e']['ms_per_step'])"
