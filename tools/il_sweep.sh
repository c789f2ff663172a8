#!/bin/bash
# Graph-timed sweep of the interleaved add routes' knobs (tools/il_graph.py):
# k_addsub_il2 chunk depth (compile-time, DOTG_IL2_CH variants) x pairs per lane x segment
# split; thread-per-pair CTA size and unroll. One JSON line per setting.
set -e
cd "$(dirname "$0")/.."
[ -f tools/build/libdotg_un4.so ] || SRC=addsub_batch KERNEL=k_addsub_il2 tools/build_variants.sh ch2 "-DDOTG_IL2_CH=2" ch8 "-DDOTG_IL2_CH=8" \
  un16 "-DDOTG_TPP_UN=16" un4 "-DDOTG_TPP_UN=4" > /dev/null
run() {  # label, env..., -- args
  local label=$1; shift
  r=$(env "$@" python tools/il_graph.py --only $MODE --ms $MS | tail -1)
  echo "{\"setting\": \"$label\", \"r\": $r}"
}
MS=64,128,256,512,1024; MODE=3
for lib in base ch2 ch8; do
  L=""; [ $lib != base ] && L=tools/build/libdotg_$lib.so
  for ppl in 1 2; do for wdiv in 1 2 4; do
    run "il2 $lib ppl$ppl wdiv$wdiv" ${L:+DOTG_LIB_PATH=$L} DOTG_IL2_PPL=$ppl DOTG_IL2_WDIV=$wdiv
  done; done
done
MS=16,32,64,128; MODE=2
for lib in base un16 un4; do
  L=""; [ $lib != base ] && L=tools/build/libdotg_$lib.so
  for bs in 32 64 128 256; do run "tpp $lib block$bs" ${L:+DOTG_LIB_PATH=$L} DOTG_TPP_BLOCK=$bs; done
done
