#!/bin/bash
# ncu capture of the (v, soc, t) stage kernel on the short C2 workload.
# usage: tools/ncu_stage.sh <out-name> [precision]
set -e
OUT=${1:-stage}
PREC=${2:-fp32}
python tools/profile_c2.py --precision "$PREC" > gpurun_out/${OUT}_plain.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled \
    -k "regex:bellman_stage" -s 5 -c 3 -o gpurun_out/${OUT} \
    python tools/profile_c2.py --precision "$PREC" > gpurun_out/${OUT}_ncu.log 2>&1
tail -2 gpurun_out/${OUT}_ncu.log
