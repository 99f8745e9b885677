#!/bin/bash
# A/B the C3 sweep of library variants: tools/ab_c3.sh lib1.so lib2.so ...
for lib in "$@"; do
  echo "$lib"
  ECO_B200_LIB=$lib timeout 300 python tools/c3_probe.py --horizon 20 --reps 2 --no-count 2>&1 | tail -1
done
