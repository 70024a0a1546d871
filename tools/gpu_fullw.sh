FSLD_LIB_PATH=paper_2311_16100_b200/_lib/libfsld_b200.so PYTHONPATH=. timeout 900 python tools/prec_probe.py 2>&1 | grep rel
FSLD_NO_TABLES=1 PYTHONPATH=. timeout 900 python tools/prec_probe.py 2>&1 | grep "cfg3\|cfg2" | sed 's/^/compute-path /'
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
export BENCH_ARGS="--steps 20 --warmup 5"
bash tools/exp_value3.sh 2>&1
