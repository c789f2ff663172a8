mkdir -p gpurun_out
python -m pytest tests/test_gpu_addsub.py -q -x > gpurun_out/pytest_addsub.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_addsub.log
python bench.py --steps 200 --warmup 10 --no-secondary --no-e2e --no-cpu > gpurun_out/bench_grouped.json 2>gpurun_out/bench_grouped.err; echo rc=$?
python bench.py --steps 200 --warmup 10 --no-secondary --no-e2e --no-cpu --ungrouped > gpurun_out/bench_ungrouped.json 2>gpurun_out/bench_ungrouped.err; echo rc=$?
for f in grouped ungrouped; do python -c "
import json;d=json.load(open('gpurun_out/bench_$f.json'));r=d['roofline'];print('$f', round(d['value']), round(d['ms_per_step']*1e3,1),'us', round(r['frac'],3), r['per_size'])"; done
tail -3 gpurun_out/bench_grouped.err
