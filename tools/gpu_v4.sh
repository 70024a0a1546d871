# v4 kernel bring-up: GPU tests (v4 default), bench v4 vs v3 (same box)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v4_pytest.log 2>&1; echo pytest=$?; tail -15 gpurun_out/v4_pytest.log
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep"
timeout 300 $B > gpurun_out/v4_bench.json 2> gpurun_out/v4_bench.err; tail -1 gpurun_out/v4_bench.json | cut -c1-300
FSLD_KERNEL=v3 timeout 300 $B > gpurun_out/v3_bench.json 2> gpurun_out/v3_bench.err; tail -1 gpurun_out/v3_bench.json | cut -c1-300
timeout 300 $B > gpurun_out/v4_bench2.json 2>&1; tail -1 gpurun_out/v4_bench2.json | cut -c1-300
