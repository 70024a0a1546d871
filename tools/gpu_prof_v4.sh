# ncu --set full of the v4 kernel (fused step) with source, raw + sass pages
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep"
ncu --set full --clock-control none --import-source on -k regex:brick_loss_grad_v4 -s 3 -c 1 -o gpurun_out/v4p $B > gpurun_out/v4p.log 2>&1
ncu -i gpurun_out/v4p.ncu-rep --page raw --csv > gpurun_out/v4p_raw.csv 2>/dev/null
ncu -i gpurun_out/v4p.ncu-rep --page source --csv --print-source sass > gpurun_out/v4p_sass.csv 2>/dev/null
ncu -i gpurun_out/v4p.ncu-rep --page details > gpurun_out/v4p_details.txt 2>/dev/null
tail -2 gpurun_out/v4p.log
