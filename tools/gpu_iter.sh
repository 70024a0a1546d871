# iteration loop: parity tests, kernel timing, phase profile, bench
python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -20
python tools/time_kernels.py 128 512 2>&1 | tail -2
python tools/phase_prof.py 2>&1 | tail -9
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
