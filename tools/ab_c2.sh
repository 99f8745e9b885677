#!/bin/bash
# A/B the C2 closed-loop bench line of library variants: tools/ab_c2.sh lib1.so lib2.so ... (each run twice, interleaved)
# a lib argument may carry env settings: "ECO_STAGE_ALIAS=1:build/ab/x.so"
for rep in 1 2; do
  for spec in "$@"; do
    lib=${spec##*:}; envs=""; [ "$spec" != "$lib" ] && envs=${spec%:*}
    printf "%s " "$spec"
    env $envs ECO_B200_LIB=$lib timeout 300 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d.get('sweep_ms_per_stage'))"
  done
done
if [ -n "$AB_C4" ]; then
  for spec in "$@"; do
    lib=${spec##*:}; envs=""; [ "$spec" != "$lib" ] && envs=${spec%:*}
    printf "c4 %s " "$spec"
    env $envs ECO_B200_LIB=$lib timeout 300 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['value'])"
  done
fi
