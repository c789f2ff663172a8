#!/bin/bash
# End-to-end (host C ABI, pinned buffers) add/sub against the pipeline slice size
# (DOTG_HOST_SLICE_MB): the C2 step and the C1 add + sub batch through bench.py's e2e legs.
for mb in 6 12 24 48; do
  r=$(DOTG_HOST_SLICE_MB=$mb python bench.py --steps 10 --warmup 3 --no-cpu --no-phase --only C1 2>/dev/null | tail -1)
  h=$(DOTG_HOST_SLICE_MB=$mb python bench.py --steps 10 --warmup 3 --no-cpu --no-phase --no-secondary 2>/dev/null | tail -1)
  python - "$mb" "$r" "$h" <<'PY'
import json, sys
mb, r, h = sys.argv[1], json.loads(sys.argv[2]), json.loads(sys.argv[3])
print(json.dumps({"slice_mb": int(mb), "C1_e2e_GBps": r["configs"]["C1"]["e2e"]["value"],
                  "C2_e2e_GBps": h["e2e"]["value"], "C2_transfer_only_GBps": h["e2e"]["transfer_only_GBps"]}))
PY
done
