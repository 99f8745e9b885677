#!/bin/bash
# Round evidence for every workload: launch list of the default bench command
# (serialised per-launch times) and one ncu --set full capture of the dominant
# kernel of C2 / C3 / C4.  Each ncu run only after the same command ran clean.
set -x
R=${1:-r01}
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err &&
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv \
    --log-file gpurun_out/${R}_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/profile_c2.py > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:bellman_stage' -s 40 -c 1 \
    -o gpurun_out/${R}_c2_stage python tools/profile_c2.py > /dev/null 2>&1
python tools/c3_probe.py --horizon 2 --reps 1 --no-count > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:bellman_wide' -c 1 \
    -o gpurun_out/${R}_c3_wide python tools/c3_probe.py --horizon 2 --reps 1 --no-count > /dev/null 2>&1
python tools/c4_probe.py 256 > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:bellman_batch' -s 20 -c 1 \
    -o gpurun_out/${R}_c4_batch python tools/c4_probe.py 256 > /dev/null 2>&1
ls -la gpurun_out/
