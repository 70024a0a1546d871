# NVLS exchange: unit tests, the bench's one-member-team graph, and timing of the NVLS step vs the fused step
timeout 600 python -m pytest tests/test_gpu_nvls.py tests/test_gpu_bench_ranks.py -x -q > gpurun_out/nvls_pytest.log 2>&1; echo pytest=$?; tail -15 gpurun_out/nvls_pytest.log
timeout 600 env FSLD_BENCH_FORCE_DP=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep > gpurun_out/nvls_bench.json 2> gpurun_out/nvls_bench.err; echo bench_nvls=$?
timeout 600 env FSLD_BENCH_FORCE_DP=1 FSLD_COMM=nccl python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep > gpurun_out/nccl_bench.json 2> gpurun_out/nccl_bench.err; echo bench_nccl=$?
for f in nvls nccl; do python -c "
import json; d=json.loads(open('gpurun_out/${f}_bench.json').read().strip().splitlines()[-1])
print('$f', round(d['value']), 'ms', round(d['ms_per_step'],4), 'kern', round(d['roofline']['kernel_ms'],4), d['details']['step'][:60], '|', d['details'].get('exchange'))"; done
tail -3 gpurun_out/nvls_bench.err
