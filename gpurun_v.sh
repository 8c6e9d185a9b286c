timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in 0 1; do
LCRW_REV_VARIANT=$v timeout 300 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --chunk 512 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('variant $v', round(d['value']/1e6,1), 'Mpairs/s', round(d['ms_per_step'],1),'ms', {n:(round(v['ms_per_step'],1), round(v.get('tflops',v.get('gbs_algorithmic',0)),1)) for n,v in k.items()}, round(d['clocks']['sm_mhz']), 'e2e', round(d['e2e']['value']/1e6,1))"
done
