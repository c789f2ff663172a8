#!/bin/bash
# C3 A/B of experimental builds (tools/build_variants.sh): tools/c3_probe.py per library.
for v in "$@"; do
  echo "{\"variant\": \"$v\", \"result\": $(DOTG_LIB_PATH=tools/build/libdotg_$v.so python tools/c3_probe.py 2>&1 | tail -1)}"
done
