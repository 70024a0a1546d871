# ncu --set full of the v3 kernel in an experimental build: bash tools/gpu_prof_exp.sh <exp name>
n=$1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep"
FSLD_KERNEL=v3 FSLD_LIB_PATH=paper_2311_16100_b200/_lib/exp_$n.so ncu --set full --clock-control none --import-source on -k regex:brick_loss_grad_kernel -s 3 -c 1 -o gpurun_out/exp_$n $B > gpurun_out/exp_$n.log 2>&1
ncu -i gpurun_out/exp_$n.ncu-rep --page source --csv --print-source sass > gpurun_out/exp_${n}_sass.csv 2>/dev/null
tail -1 gpurun_out/exp_$n.log
