# ncu --set full of the secondary kernels (one launch each, after warm-up), summarised per kernel
B="python bench.py --images 4096 --steps 3 --warmup 3 --no-cpu-baseline"
for k in sorted_energy precond_step sorted_hutch grad_init apply_step slab_items; do
  ncu --set full --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/aux_$k $B > gpurun_out/ncu_aux_$k.log 2>&1
  python tools/ncu_summary.py gpurun_out/aux_$k.ncu-rep > gpurun_out/aux_$k.txt 2>&1
done
python - <<'PY'
import os
ks = ["sorted_energy", "precond_step", "sorted_hutch", "grad_init", "apply_step", "slab_items"]
for k in ks:
    p = f"gpurun_out/aux_{k}.txt"
    print(open(p).read() if os.path.exists(p) else f"{k}: no capture")
PY
