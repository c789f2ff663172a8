for ns in 2 3 4; do for mb in 8 24 64; do
  r=$(DOTG_HOST_STREAMS=$ns DOTG_HOST_SLICE_MB=$mb python bench.py --steps 20 --warmup 3 --no-secondary --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['e2e']['value'],1))")
  echo "streams=$ns slice_mb=$mb e2e=$r"
done; done
