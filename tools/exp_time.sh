python tools/time_kernels.py 128 512 2>&1 | grep brick | sed 's/^/base     /'
for v in NO_PASS1 NO_PASS2; do FSLD_LIB_PATH=paper_2311_16100_b200/_lib/exp_$v.so python tools/time_kernels.py 128 512 2>&1 | grep brick | sed "s/^/$v /"; done
