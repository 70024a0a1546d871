# launch list of a short bench (cfg3 on 4096 images): per-kernel device time shares
B="python bench.py --images 4096 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1
tail -1 gpurun_out/ncu1.log | cut -c1-200
