#!/bin/bash
# Per-launch device time of every kernel in the short C2 workload (warm caches).
OUT=${1:-launches}
python tools/profile_c2.py --steps 6 > gpurun_out/${OUT}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 760 -c 120 --csv \
    --log-file gpurun_out/${OUT}.csv python tools/profile_c2.py --steps 6 > gpurun_out/${OUT}_ncu.log 2>&1
tail -1 gpurun_out/${OUT}_ncu.log
