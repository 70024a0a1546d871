B="python bench.py --images 8192 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-algo1 --no-sweep"
for f in paper_2311_16100_b200/_lib/libfsld_b200.so paper_2311_16100_b200/_lib/exp_waveonly.so; do
 echo "== $f"
 FSLD_LIB_PATH=$f ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_atom.sum --clock-control none -k regex:sorted_loss_grad -s 3 -c 1 $B 2>&1 | grep -E "duration|wavefronts|inst_executed"
done
