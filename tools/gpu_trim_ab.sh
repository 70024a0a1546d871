# parity subset with the product build + interleaved A/B against exp builds
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_det.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
export BENCH_ARGS="--steps 20 --warmup 5"
bash tools/exp_value3.sh 2>&1
