#!/bin/bash
# k_addsub_ilf variants (DOTG_IL_MODE=5): parity of every forced interleaved route, then the
# graph-timed per-launch sweep over chunk rows / pairs per lane / double buffering / split.
python -m pytest tests/test_gpu_il_routes.py -x -q > gpurun_out/ilf_tests.log 2>&1
for s in "DOTG_ILF_DB=1" "DOTG_ILF_DB=1 DOTG_ILF_PPL=2" "DOTG_ILF_DB=0" "DOTG_ILF_DB=0 DOTG_ILF_PPL=2" \
         "DOTG_ILF_DB=1 DOTG_ILF_WDIV=2" "DOTG_ILF_DB=1 DOTG_ILF_PPL=2 DOTG_ILF_WDIV=2"; do
  r=$(env $s python tools/il_graph.py --only 5 --ms 16,32,64,128,256,512,1024 | tail -1)
  echo "{\"setting\": \"ilf $s\", \"r\": $r}"
done > gpurun_out/ilf_graph.jsonl 2>&1
