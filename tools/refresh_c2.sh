#!/bin/bash
# GPU suite, the default C2 bench line, and the launch list of the same command
R=${1:-r01}
python -m pytest tests -m gpu -q -x > gpurun_out/${R}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${R}_pytest_gpu.log
python bench.py > gpurun_out/${R}_bench_c2.json 2> gpurun_out/${R}_bench_c2.err && tail -1 gpurun_out/${R}_bench_c2.json &&
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv \
    --log-file gpurun_out/${R}_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_stats.py gpurun_out/${R}_launches_c2.csv > gpurun_out/${R}_launches_c2_stats.txt 2>&1; cat gpurun_out/${R}_launches_c2_stats.txt
