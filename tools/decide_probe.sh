#!/bin/bash
# per-launch decide kernel duration (ncu launch list) for a library build
LIB=${1:-paper_2104_01284_b200/_eco_b200.so}
ECO_B200_LIB=$LIB ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:mpc_decide -s 2 -c 6 \
    --log-file gpurun_out/decide_ll.csv python tools/profile_c2.py --steps 4 > /dev/null 2>&1
python tools/launch_stats.py gpurun_out/decide_ll.csv
