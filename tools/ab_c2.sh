#!/bin/bash
# A/B the C2 bench line of library variants: tools/ab_c2.sh lib1.so lib2.so ... (each run twice, interleaved)
for rep in 1 2; do
  for lib in "$@"; do
    printf "%s " "$lib"
    ECO_B200_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['sweep_ms_per_stage'])"
  done
done
if [ -n "$AB_C4" ]; then
  for lib in "$@"; do
    printf "c4 %s " "$lib"
    ECO_B200_LIB=$lib timeout 300 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['value'])"
  done
fi
