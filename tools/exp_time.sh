# time the product build and the ablation builds (make them first: bash tools/build_exp.sh NAME -DFSLD_EXP_NAME)
python tools/time_kernels.py 128 512 2>&1 | grep brick | sed 's/^/base       /'
for f in paper_2311_16100_b200/_lib/exp_*.so; do n=$(basename $f .so); FSLD_LIB_PATH=$f python tools/time_kernels.py 128 512 2>&1 | grep brick | sed "s/^/$n /"; done
