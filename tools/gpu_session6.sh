for pf in 0 7 1; do echo "PF=$pf"; DOTG_MUL_PF=$pf python bench.py --only C3 --steps 20 --warmup 3 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l)
        for k,v in d['configs'].items(): print(k, 'frac_imad', round(v['frac_imad'],3), 'kernel_us', round(v['kernel_us'],1))
"; done
