# timing of brick vs tile + ncu full capture of the brick kernel
PYTHONPATH=. python tools/debug_brick2.py 2>&1 | tail -3
PYTHONPATH=. python tools/debug_brick2.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:brick_loss_grad -s 4 -c 1 -o gpurun_out/prof_brick python tools/debug_brick2.py > gpurun_out/ncu_brick.log 2>&1
tail -2 gpurun_out/ncu_brick.log
