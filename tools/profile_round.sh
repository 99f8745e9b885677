#!/bin/bash
# Round evidence: plain bench run, then the ncu launch list of the same bench
# command (serialised, per-launch times) and one full capture of the stage kernel.
set -x
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err &&
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv \
    --log-file gpurun_out/r_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r_launches.log 2>&1
python tools/profile_c2.py > gpurun_out/r_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:bellman_stage' -s 40 -c 2 -o gpurun_out/r_stage_full python tools/profile_c2.py > gpurun_out/r_full.log 2>&1
ls -la gpurun_out/
