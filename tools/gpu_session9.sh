python -m pytest tests/test_gpu_host_api.py -q -x 2>&1 | tail -2
python bench.py --steps 100 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo rc=$?; tail -3 gpurun_out/bench2.err
python -c "
import json;d=json.load(open('gpurun_out/bench2.json'))
print('value',round(d['value']),'frac',round(d['roofline']['frac'],3),'e2e',round(d['e2e']['value'],1),'cpu',d['cpu_baseline']['value'],'clocks',d['clocks'])
for k,v in d['configs'].items(): print(k, {kk:(round(vv,3) if isinstance(vv,float) else vv) for kk,vv in v.items() if kk not in ('note','metric')})
"
