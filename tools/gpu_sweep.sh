export BENCH_ARGS="--steps 20 --warmup 5"
bash tools/exp_value3.sh 2>&1
