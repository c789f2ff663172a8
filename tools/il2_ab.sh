#!/bin/bash
# A/B of the re-read segmented interleaved kernel (DOTG_IL_MODE=3): chunk depth builds
# (tools/build_variants.sh) and DOTG_IL2_WDIV, through tools/il_modes.py's child.
for v in ch4o ch2 ch4o15 ch2o20 ch4o20; do
  for wd in 1; do
    lib=paper_2604_21566_b200/libdotg.so; [ "$v" != base ] && lib=tools/build/libdotg_$v.so
    r=$(DOTG_LIB_PATH=$lib DOTG_IL_MODE=3 DOTG_IL2_WDIV=$wd python tools/il_modes.py --only 3 2>&1 | tail -1)
    echo "{\"variant\": \"$v\", \"wdiv\": $wd, \"r\": $r}"
  done
done
