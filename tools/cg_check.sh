for f in paper_2311_16100_b200/_lib/libfsld_b200.so paper_2311_16100_b200/_lib/exp_*.so; do
  echo "== $f"; FSLD_LIB_PATH=$f python tools/hvp_err.py 2>&1 | tail -2
  FSLD_LIB_PATH=$f python -m pytest tests/test_gpu_step.py -q -k "reference_solve" 2>&1 | tail -1
done
