timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_det.py tests/test_gpu_step.py -m gpu -x -q 2>&1 | tail -1
PYTHONPATH=. timeout 900 python tools/prec_probe.py 2>&1 | grep "cfg3\|cfg2" | head -4
export BENCH_ARGS="--steps 20 --warmup 5"
bash tools/exp_value3.sh 2>&1
