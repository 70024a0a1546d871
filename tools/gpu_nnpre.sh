timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -m gpu -x -q -k "nn or cfg1 or golden" 2>&1 | tail -1
export BENCH_ARGS="--steps 20 --warmup 5 --config cfg1"
bash tools/exp_value3.sh 2>&1
