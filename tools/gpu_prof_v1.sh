python -m pytest tests -m gpu -q 2>&1 | tail -25
B="python bench.py --images 4096 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v1.csv $B > gpurun_out/ncu1.log 2>&1 ; \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:ILi1ELi2ELb0E -s 3 -c 1 -o gpurun_out/prof_v1 $B > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu2.log
