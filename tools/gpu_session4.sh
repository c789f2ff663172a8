python -m pytest tests/test_gpu_mul.py -q -x 2>&1 | tail -3
python bench.py --only C3,C4 --steps 20 --warmup 3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        for k,v in d['configs'].items(): print(k, 'frac_imad', round(v['frac_imad'],3), 'kernel_us', round(v['kernel_us'],1), 'pairs/s', '%.3e'%v['kernel_pairs_s'])
    else: print(l.rstrip())
"
