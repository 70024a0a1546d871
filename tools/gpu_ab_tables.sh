# A/B of the table-driven brick kernel vs the compute path (bench value, step and kernel ms), then parity
for r in 1 2; do
for mode in tables compute; do
if [ $mode = compute ]; then export FSLD_NO_TABLES=1; else unset FSLD_NO_TABLES; fi
python bench.py --no-cpu-baseline --no-e2e --no-sweep --no-algo1 ${BENCH_ARGS} | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode', round(d['value']), 'step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],4))"
done; done
unset FSLD_NO_TABLES
[ -n "$NO_TESTS" ] || python -m pytest -x -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_capi_c.py 2>&1 | tail -3
