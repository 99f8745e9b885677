set -x
python tools/c3_probe.py --horizon 2 --reps 1 --no-count > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:bellman_wide2' -c 1 \
    -o gpurun_out/r02b_c3_wide2 python tools/c3_probe.py --horizon 2 --reps 1 --no-count > gpurun_out/ncu_b.log 2>&1
tail -2 gpurun_out/ncu_b.log
