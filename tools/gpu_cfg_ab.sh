# per-config A/B: table-driven brick kernel vs compute path / tile path (bench value, ms, kernel ms)
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), 'step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],4))"; }
B="--no-cpu-baseline --no-e2e --no-sweep --no-algo1"
python bench.py --config cfg1 $B | q cfg1_tables
FSLD_TILE_PATH=1 python bench.py --config cfg1 $B | q cfg1_tile
python bench.py --config cfg2 $B | q cfg2_tables
FSLD_NO_TABLES=1 python bench.py --config cfg2 $B | q cfg2_compute
python bench.py --config cfg4 --images 20000 $B | q cfg4_tables
FSLD_NO_TABLES=1 python bench.py --config cfg4 --images 20000 $B | q cfg4_compute
