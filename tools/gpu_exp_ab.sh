# correctness of one exp build on the config parity tests + interleaved value A/B of all exp builds
# usage: bash tools/gpu_exp_ab.sh <exp name to test>
FSLD_LIB_PATH=paper_2311_16100_b200/_lib/exp_$1.so timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -x -q 2>&1 | tail -2
export BENCH_ARGS="--steps 20 --warmup 5"
bash tools/exp_value3.sh 2>&1
