# planned bench step (value, ms) for the product build and each ablation / variant build in _lib/exp_*.so
run() { timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-sweep --no-algo1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; }
run base
for f in paper_2311_16100_b200/_lib/exp_*.so; do n=$(basename $f .so); FSLD_LIB_PATH=$f run $n; done
run base
