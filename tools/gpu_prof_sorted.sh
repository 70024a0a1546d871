python tools/time_kernels.py 128 512 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sorted_loss_grad -s 2 -c 1 -o gpurun_out/prof_sorted python tools/time_kernels.py 128 512 > gpurun_out/ncu_sorted.log 2>&1
tail -2 gpurun_out/ncu_sorted.log
python -m pytest tests -m gpu -q -x -k "brick_path_matches_tile_path and 256" 2>&1 | grep -E "assert|Error" | head -5
