P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["e2e"]["ms_per_step"], d["e2e"]["c_abi"]["ms_per_step"])'
echo base; python bench.py --no-cpu-baseline --no-algo1 --no-sweep 2>/dev/null | python -c "$P"
echo nograph; FSLD_NO_GRAPH=1 python bench.py --no-cpu-baseline --no-algo1 --no-sweep 2>/dev/null | python -c "$P"
echo steps3; python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-algo1 --no-sweep 2>/dev/null | python -c "$P"
