# e2e (host-buffer loss+grad) vs the slab count of fsld_loss_grad_host
for n in ${SLABS:-4 6 8 10 12 16 8 10 12}; do
  FSLD_HOST_SLABS=$n timeout 300 python bench.py --no-cpu-baseline --no-algo1 --no-sweep --steps 20 --warmup 5 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('slabs $n', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],4), 'value', round(d['value']))"
done
