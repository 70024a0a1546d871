# A/B of the table-driven brick kernel vs the compute path, then the parity subset that covers it
set -x
python tools/time_kernels.py 128 512 2>&1 | grep brick | sed 's/^/tables  /'
FSLD_NO_TABLES=1 python tools/time_kernels.py 128 512 2>&1 | grep brick | sed 's/^/compute /'
for r in 1 2; do
python bench.py --no-cpu-baseline --no-e2e --no-sweep --no-algo1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tables', round(d['value']), round(d['ms_per_step'],4))"
FSLD_NO_TABLES=1 python bench.py --no-cpu-baseline --no-e2e --no-sweep --no-algo1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('compute', round(d['value']), round(d['ms_per_step'],4))"
done
python -m pytest -x -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_capi_c.py 2>&1 | tail -15
