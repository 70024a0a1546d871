timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_parity.py tests/test_gpu_step.py tests/test_capi_host.py -m gpu -x -q 2>&1 | tail -3
PYTHONPATH=. python tools/e2e_iters.py 2>&1 | tail -1
PYTHONPATH=. timeout 300 python tools/e2e_split.py 2>&1 | tail -2
