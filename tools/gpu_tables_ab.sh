B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep"
for r in 1 2; do
$B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tables', round(d['value']), d['roofline']['kernel_ms'])"
FSLD_NO_TABLES=1 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('compute', round(d['value']), d['roofline']['kernel_ms'])"
done
