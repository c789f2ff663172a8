for rep in 1 2; do
for v in "" k32x16 k64x8 k128x4; do
  if [ -z "$v" ]; then echo "== base"; python tools/mul_timing.py 16 | cut -c1-60; else echo "== $v"; DOTG_LIB_PATH=tools/build/libdotg_$v.so python tools/mul_timing.py 16 | cut -c1-60; fi
done
done
