# all bench lines of the round (default line + the other configs + the reference arm)
python bench.py > gpurun_out/final_cfg3.json 2> gpurun_out/final_cfg3.err
for c in cfg1 cfg2 cfg5; do python bench.py --config $c --no-cpu-baseline > gpurun_out/final_$c.json 2>/dev/null; done
python bench.py --config cfg4 --images 20000 --no-cpu-baseline --no-algo1 > gpurun_out/final_cfg4.json 2>/dev/null
FSLD_NO_TABLES=1 python bench.py --no-cpu-baseline --no-sweep --no-algo1 > gpurun_out/final_cfg3_compute.json 2>/dev/null
python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
nproc > gpurun_out/final_host.txt; lscpu | grep "Model name" >> gpurun_out/final_host.txt
