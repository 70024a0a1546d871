# full bench line (loss+grad step, Algorithm-1 step, probe sweep) for the product build and each exp_*.so
run() { timeout 600 python bench.py --no-cpu-baseline --no-e2e | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['value']), round(d['ms_per_step'],4), 'algo1', round(d['algorithm1_step']['ms_per_step'],4), 'sweep', [round(x,3) for x in d['hutchinson_sweep']['ms_per_pass']], 'hvp', round(d['next_rows']['cg_hessian_product']['ms'],2))"; }
run base
for f in paper_2311_16100_b200/_lib/exp_*.so; do n=$(basename $f .so); FSLD_LIB_PATH=$f run $n; done
