#!/bin/bash
# C4 bench line per batch tile shape (ECO_BATCH_TJ x ECO_BATCH_SLICES) and alias mode
for cfg in "4 8 1" "2 16 1" "4 6 1" "3 10 1" "4 8 0"; do
  set -- $cfg
  printf "tj=%s slices=%s alias=%s " $1 $2 $3
  ECO_BATCH_TJ=$1 ECO_BATCH_SLICES=$2 ECO_BATCH_ALIAS=$3 timeout 300 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['value'])"
done
