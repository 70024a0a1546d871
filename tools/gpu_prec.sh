for lib in libfsld_b200 exp_lim8 exp_lim64 exp_lim512; do echo "== $lib"; FSLD_LIB_PATH=paper_2311_16100_b200/_lib/$lib.so PYTHONPATH=. timeout 900 python tools/prec_probe.py 2>&1 | grep rel; done
