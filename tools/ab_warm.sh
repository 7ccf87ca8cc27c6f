#!/bin/bash
# A/B of libtsb builds on the warm and T_max Aztec-4096 states: bash tools/ab_warm.sh lib1.so lib2.so ...
for lib in "$@"; do
  for rep in 1 2; do
    echo "$lib $(TSB_LIB=$PWD/$lib python tools/time_warm.py 2>&1 | tail -1)"
  done
done
