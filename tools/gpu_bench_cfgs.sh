# all BASELINE configs through bench.py (short runs), one summary line each
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print('$1', round(d['value']), d['unit'], 'ms/step', round(d['ms_per_step'],4), 'frac', r.get('frac'), 'kernel_ms', r.get('kernel_ms'), '|', json.dumps(d.get('sweep'))[:400] if d.get('sweep') else '')
"; }
for c in cfg1 cfg2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep 2>/dev/null | summ $c; done
timeout 600 python bench.py --config cfg5 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-algo1 2>/dev/null | summ cfg5
timeout 900 python bench.py --config cfg4 --images 20000 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep 2>/dev/null | summ cfg4
