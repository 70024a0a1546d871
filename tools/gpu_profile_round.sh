# round profile capture: plain bench, launch list, ncu --set full of the fused loss+grad kernel (+ SASS page)
B="python bench.py --images 8192 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:sorted_loss_grad -s 3 -c 1 -o gpurun_out/prof_round $B > gpurun_out/ncu2.log 2>&1
tail -1 gpurun_out/ncu2.log
ncu -i gpurun_out/prof_round.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_round.csv 2>/dev/null
ncu -i gpurun_out/prof_round.ncu-rep --page details --csv > gpurun_out/details_round.csv 2>/dev/null
