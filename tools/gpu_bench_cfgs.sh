# all BASELINE configs through bench.py (short runs)
for c in cfg1 cfg2 cfg3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-420; done
timeout 600 python bench.py --config cfg5 --steps 8 --warmup 2 2>&1 | tail -1
timeout 900 python bench.py --config cfg4 --images 20000 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-420
