#!/bin/bash
# Interleaved add/sub after a routing change: forced-route parity, the interleaved and
# fuzz GPU tests, then the graph-timed auto route against row-major, and knob variants.
python -m pytest tests/test_gpu_il_routes.py tests/test_gpu_addsub.py tests/test_gpu_fuzz.py -x -q > gpurun_out/ilf_tests.log 2>&1
python tools/il_graph.py --only 0,rows > gpurun_out/il_graph_auto.jsonl 2>&1
for s in "DOTG_ILF_G=32" "DOTG_ILF_G=16" "DOTG_ILF_G=8"; do
  r=$(env $s python tools/il_graph.py --only 5 --ms 64,128,256,512,1024 | tail -1)
  echo "{\"setting\": \"$s\", \"r\": $r}" >> gpurun_out/il_graph_auto.jsonl
done
