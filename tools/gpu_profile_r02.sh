# round-2 evidence: plain bench line, ncu launch list of the same command, ncu --set full of the
# headline kernel (table-driven brick kernel, fused step) with source, and of the compute-path kernel
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep"
$B > gpurun_out/r02_plain.json 2> gpurun_out/r02_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $B > gpurun_out/r02_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:brick_loss_grad_kernel -s 3 -c 1 -o gpurun_out/r02_v3 $B > gpurun_out/r02_ncu2.log 2>&1
FSLD_NO_TABLES=1 ncu --set full --clock-control none -k regex:sorted_loss_grad_kernel -s 3 -c 1 -o gpurun_out/r02_compute $B > gpurun_out/r02_ncu3.log 2>&1
ncu -i gpurun_out/r02_v3.ncu-rep --page raw --csv > gpurun_out/r02_v3_raw.csv 2>/dev/null
ncu -i gpurun_out/r02_v3.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_v3_sass.csv 2>/dev/null
ncu -i gpurun_out/r02_compute.ncu-rep --page raw --csv > gpurun_out/r02_compute_raw.csv 2>/dev/null
tail -1 gpurun_out/r02_ncu2.log; tail -1 gpurun_out/r02_ncu3.log
