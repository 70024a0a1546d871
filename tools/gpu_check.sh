# quick GPU check: tests, smoke, short bench (plain, no profiler)
python -m pytest tests -m gpu -q -x 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log
