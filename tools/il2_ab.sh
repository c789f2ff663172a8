#!/bin/bash
# A/B of the re-read segmented interleaved kernel (k_addsub_il2, DOTG_IL_MODE=3): pairs per
# lane (DOTG_IL2_PPL 1 / 2), through tools/il_modes.py's child; then the interleaved parity
# tests under both settings.
for ppl in 1 2; do
  r=$(DOTG_IL2_PPL=$ppl python tools/il_modes.py --only 3 2>&1 | tail -1)
  echo "{\"ppl\": $ppl, \"r\": $r}"
done
for ppl in 1 2; do
  DOTG_IL2_PPL=$ppl DOTG_IL_MODE=3 python -m pytest tests -m gpu -x -q -k "interleav or addsub or fuzz" 2>&1 | tail -1
done
