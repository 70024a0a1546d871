# ncu --set full of the brick probe batcher (cfg5 sweep, k = 64) and of the tile batcher for comparison
B="python bench.py --config cfg5 --steps 4 --warmup 2"
$B > gpurun_out/plain_hutch.log 2>&1 && \
ncu --set full --clock-control none -k regex:sorted_hutch -s 6 -c 1 -o gpurun_out/prof_hutch $B > gpurun_out/ncu_hutch.log 2>&1
tail -1 gpurun_out/ncu_hutch.log
python tools/ncu_summary.py gpurun_out/prof_hutch.ncu-rep
