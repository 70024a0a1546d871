# L2 flush variants between timed steps: write (512 MB fill), clean (fill, then a 256 MB read), none
for r in 1 2; do for m in write clean none; do
FSLD_BENCH_FLUSH=$m timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m', round(d['value']), round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4))"
done; done
