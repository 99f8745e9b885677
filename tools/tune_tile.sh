#!/bin/bash
# Per-stage sweep time of the C2 workload for several tile shapes / band caps.
CFGS=("2 16 40" "4 8 40" "3 8 40" "2 12 40")
for cfg in "${CFGS[@]}"; do
  set -- $cfg
  ECO_TILE_TJ=$1 ECO_TILE_SLICES=$2 ECO_BAND_KB=$3 python tools/profile_c2.py --steps 20 > /tmp/t.log 2>&1
  python3 - "$1" "$2" "$3" <<'PY'
import sys, ast
l = open("/tmp/t.log").read()
if "{" not in l:
    print("cfg", sys.argv[1:], "FAILED", l[-300:]); sys.exit()
d = ast.literal_eval(l[l.rindex("{"):l.rindex("}") + 1])
print(f"tj={sys.argv[1]} slices={sys.argv[2]} bandKB={sys.argv[3]} us/stage={1e3 * d['dominant_ms'] / d['stages']:.2f} step_ms={d['device_ms'] / 20:.3f}")
PY
done
