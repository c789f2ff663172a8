for v in 1 2; do echo "V=$v"; DOTG_MUL64=$v python bench.py --only C4 --steps 10 --warmup 3 --no-e2e 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        for k,v in d['configs'].items(): print(k, 'frac_imad', round(v['frac_imad'],3), 'kernel_us', round(v['kernel_us'],1))
"; DOTG_MUL64=$v python -m pytest tests/test_gpu_mul.py -q -x -k "64 or C4 or golden" 2>&1 | tail -1; done
