# v4 correctness subset + A/B (v4 base, v4 exp builds, v3) on one box
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_step.py -m gpu -x -q > gpurun_out/v4ab_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/v4ab_pytest.log
export BENCH_ARGS="--steps 20 --warmup 5"
bash tools/exp_value3.sh 2>&1
FSLD_KERNEL=v3 FSLD_LIB_PATH=paper_2311_16100_b200/_lib/libfsld_b200.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-sweep --no-algo1 $BENCH_ARGS | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v3', round(d['value']), round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4))"
