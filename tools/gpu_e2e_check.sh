for r in 1 2; do python bench.py --no-cpu-baseline --no-algo1 --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('numpy', round(d['e2e']['ms_per_step'],3), 'c_abi', round(d['e2e']['c_abi']['ms_per_step'],3))"; done
PYTHONPATH=. python tools/e2e_split.py 2>&1 | tail -2
python tools/pcie_probe.py 2>&1 | head -4
