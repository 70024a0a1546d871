# brick DIAG pass: parity tests, the det/parity suites it touches, and the next_rows timings
timeout 900 python -m pytest tests/test_gpu_diag.py tests/test_gpu_det.py tests/test_gpu_parity.py tests/test_gpu_step.py -x -q > gpurun_out/diag_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/diag_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/diag_bench.json 2> gpurun_out/diag_bench.err; echo bench=$?
python -c "
import json; d=json.loads(open('gpurun_out/diag_bench.json').read().strip().splitlines()[-1])
print(json.dumps(d.get('next_rows',{}).get('exact_diag')), d['value'])" 2>&1 | tail -3
