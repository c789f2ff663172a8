#!/bin/bash
# C3 A/B: DOTG_K16_HYBRID (FP64-pipe middle product) through tools/c3_probe.py, each
# setting in its own process; then the C3-shape parity tests. (r02 also measured a
# two-threads-per-pair last wave this way: profiles/r02_c3_split_tail_ab.txt.)
for cfg in "DOTG_K16_HYBRID=0" "DOTG_K16_HYBRID=1"; do
  echo "{\"cfg\": \"$cfg\", \"r\": $(env $cfg python tools/c3_probe.py 2>&1 | tail -1)}"
done
DOTG_K16_HYBRID=1 python -m pytest tests -m gpu -x -q -k "test_gpu_mul or acceptance" 2>&1 | tail -1
python -m pytest tests -m gpu -x -q -k "test_gpu_mul or acceptance or fuzz or graphs" 2>&1 | tail -1
