# checkpoint: full GPU suite, smoke, default bench line, ncu launch list + headline capture
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ck_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ck_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ck_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/ck_smoke.log
timeout 900 python bench.py > gpurun_out/ck_bench.json 2> gpurun_out/ck_bench.err; echo bench=$?
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ck_launches.csv $B > gpurun_out/ck_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:brick_loss_grad_kernel -s 3 -c 1 -o gpurun_out/ck_v3 $B > gpurun_out/ck_ncu2.log 2>&1
ncu -i gpurun_out/ck_v3.ncu-rep --page source --csv --print-source sass > gpurun_out/ck_v3_sass.csv 2>/dev/null
tail -1 gpurun_out/ck_ncu2.log
