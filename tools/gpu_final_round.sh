# end-of-round evidence: default bench line, headline-kernel ncu + launch list, secondary kernels,
# host-step timeline and slab A/B (outputs in gpurun_out/, summarised into profiles/ by hand)
python bench.py > gpurun_out/final_bench.log 2>&1; tail -1 gpurun_out/final_bench.log | cut -c1-200
bash tools/gpu_profile_round.sh
bash tools/gpu_prof_aux.sh > gpurun_out/aux_all.txt 2>&1
python tools/host_step_trace.py > gpurun_out/host_trace.txt 2>&1
python tools/host_ab.py 1,8,12,16 > gpurun_out/host_ab.txt 2>&1
python tools/pcie_probe.py > gpurun_out/pcie_probe.txt 2>&1
