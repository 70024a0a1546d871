# ncu --set full of the brick kernel + SASS source page (instructions and stalls per opcode)
python tools/time_kernels.py 128 512 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sorted_loss_grad -s 2 -c 1 -o gpurun_out/prof_sorted python tools/time_kernels.py 128 512 > gpurun_out/ncu_sorted.log 2>&1
tail -2 gpurun_out/ncu_sorted.log
ncu -i gpurun_out/prof_sorted.ncu-rep --page source --csv --print-source sass > gpurun_out/sass.csv 2>/dev/null
ncu -i gpurun_out/prof_sorted.ncu-rep --page source --csv --print-source cuda > gpurun_out/src.csv 2>/dev/null
python tools/sass_hot.py gpurun_out/sass.csv | head -40
