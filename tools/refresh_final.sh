#!/bin/bash
# round evidence: GPU suite, default C2 bench line, its launch list, one ncu --set full of the stage kernel
R=${1:-r01}
python -m pytest tests -m gpu -q -x > gpurun_out/${R}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${R}_pytest_gpu.log
python bench.py > gpurun_out/${R}_bench_c2.json 2> gpurun_out/${R}_bench_c2.err && tail -1 gpurun_out/${R}_bench_c2.json | cut -c1-400 &&
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv \
    --log-file gpurun_out/${R}_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_stats.py gpurun_out/${R}_launches_c2.csv > gpurun_out/${R}_launches_c2_stats.txt 2>&1; cat gpurun_out/${R}_launches_c2_stats.txt
python tools/profile_c2.py > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:bellman_stage' -s 60 -c 1 \
    -o gpurun_out/${R}_c2_stage python tools/profile_c2.py --steps 8 > /dev/null 2>&1
ls gpurun_out/
