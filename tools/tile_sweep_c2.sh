#!/bin/bash
# C2 bench line per stage-tile shape (ECO_TILE_TJ x ECO_TILE_SLICES)
for cfg in "2 16" "4 8" "3 10" "2 12" "4 6"; do
  set -- $cfg
  printf "tj=%s slices=%s " $1 $2
  ECO_TILE_TJ=$1 ECO_TILE_SLICES=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['sweep_ms_per_stage'])"
done
