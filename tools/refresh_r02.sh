#!/bin/bash
# Round-2 evidence on the GPU box: GPU suite, bench lines (C3 default, its
# reference arm, C2 / C4 / C5 / N1), launch lists and ncu --set full captures
# of the dominant kernels (each ncu run only after the same command ran clean).
# Summaries here afterwards: tools/ncu_report.py, tools/launch_stats.py.
R=${1:-r02}
O=gpurun_out
python -c "import bench; print(bench.so_digest())" > $O/${R}_so_digest.txt
python -m pytest tests -m gpu -q -x > $O/${R}_pytest_gpu.log 2>&1; tail -2 $O/${R}_pytest_gpu.log
python bench.py > $O/${R}_bench_c3.json 2> $O/${R}_bench_c3.err; tail -c 300 $O/${R}_bench_c3.json
python bench.py --impl reference --steps 20 --warmup 3 > $O/${R}_bench_ref.json 2> $O/${R}_bench_ref.err; tail -c 200 $O/${R}_bench_ref.json
python bench.py --workload c2 > $O/${R}_bench_c2.json 2> $O/${R}_bench_c2.err; tail -c 200 $O/${R}_bench_c2.json
python bench.py --workload c4 > $O/${R}_bench_c4.json 2> $O/${R}_bench_c4.err; tail -c 200 $O/${R}_bench_c4.json
python bench.py --workload c5 --no-cpu-baseline > $O/${R}_bench_c5.json 2> $O/${R}_bench_c5.err; tail -c 200 $O/${R}_bench_c5.json
python bench.py --workload n1 --steps 2 --warmup 1 --loop-steps 20 > $O/${R}_bench_n1.json 2> $O/${R}_bench_n1.err; tail -c 200 $O/${R}_bench_n1.json
timeout 1500 python tools/reference_table1.py 10 $O/${R}_reference_table1.txt > /dev/null 2>&1; tail -2 $O/${R}_reference_table1.txt
# launch lists (cold, serialised: shares, not absolutes)
python tools/c3_probe.py --horizon 20 --reps 2 --no-count > /dev/null 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_c3.csv \
    python tools/c3_probe.py --horizon 20 --reps 2 --no-count > /dev/null 2>&1
python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv --log-file $O/${R}_launches_c2.csv \
    python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# full captures of the dominant kernels
python tools/c3_probe.py --horizon 2 --reps 1 --no-count > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:bellman_wide2' -c 1 \
    -o $O/${R}_c3_wide2 python tools/c3_probe.py --horizon 2 --reps 1 --no-count > /dev/null 2>&1
python tools/profile_c2.py > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:bellman_stage' -s 40 -c 1 \
    -o $O/${R}_c2_stage python tools/profile_c2.py > /dev/null 2>&1
python tools/c4_probe.py 4096 > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:bellman_batch' -s 20 -c 1 \
    -o $O/${R}_c4_batch python tools/c4_probe.py 4096 > /dev/null 2>&1
ls -la $O | tail -25
