# ncu --set full of the table-driven brick kernel (one launch of the bench's planned step)
B="python bench.py --images 8192 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep"
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-brick_loss_grad} -s 3 -c 1 -o gpurun_out/prof_v3 $B > gpurun_out/ncu_v3.log 2>&1
tail -1 gpurun_out/ncu_v3.log
ncu -i gpurun_out/prof_v3.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_v3.csv 2>/dev/null
ncu -i gpurun_out/prof_v3.ncu-rep --page raw --csv > gpurun_out/raw_v3.csv 2>/dev/null
