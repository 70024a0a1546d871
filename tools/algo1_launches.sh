# per-kernel device time of the Algorithm-1 step leg (bench.py algo1_leg on a 4096-image cfg3 dataset)
B="python bench.py --images 4096 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain_algo1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_algo1.csv $B > gpurun_out/ncu_algo1.log 2>&1
tail -1 gpurun_out/plain_algo1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['algorithm1_step']))"
python tools/launches.py gpurun_out/launches_algo1.csv
