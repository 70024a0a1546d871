# bench value for the product build and each exp_*.so (tables path), interleaved rounds
run() { FSLD_LIB_PATH=$2 timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-sweep --no-algo1 ${BENCH_ARGS} | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4))"; }
for r in 1 2; do
  run base paper_2311_16100_b200/_lib/libfsld_b200.so
  for f in paper_2311_16100_b200/_lib/exp_*.so; do run $(basename $f .so) $f; done
done
