#!/bin/bash
# Experimental builds of libdotg.so with mul_imma.cu compile-time knobs, for A/B timing
# on the GPU box (DOTG_LIB_PATH=tools/build/libdotg_<name>.so python tools/mul_timing.py).
# usage: [SRC=mul_batch] tools/build_variants.sh name "-DKNOB=V ..." [name "-D..."]...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2604_21566_b200/csrc
make -s -C "$CS" -j4
mkdir -p "$ROOT/tools/build"
SRC=${SRC:-mul_imma}
OBJS=$(ls "$CS"/build/*.o | grep -v "/$SRC.o")
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I"$ROOT/include" \
       -Xptxas -v $flags -c "$CS/$SRC.cu" -o "$ROOT/tools/build/${SRC}_$name.o" 2> "$ROOT/tools/build/$name.ptxas.log"
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$ROOT/tools/build/libdotg_$name.so" \
       $OBJS "$ROOT/tools/build/${SRC}_$name.o" -ldl
  echo "$name: $(grep -A3 "${KERNEL:-ILi16}" "$ROOT/tools/build/$name.ptxas.log" | grep -E 'registers|spill' | head -2 | tr '\n' ' ')"
done
