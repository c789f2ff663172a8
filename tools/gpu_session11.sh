for i in 1 2; do python bench.py --steps 200 --warmup 10 --no-secondary --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))"; done
python -m pytest tests/test_gpu_addsub.py -q -x 2>&1 | tail -1
