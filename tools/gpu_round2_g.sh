set -x
for w in 1; do ECO_WIDE2=$w python tools/c3_probe.py --horizon 20 --reps 3 --no-count 2>&1 | tail -2; done
python -m pytest tests/test_gpu_parity.py -q -x -k "c3_full" 2>&1 | tail -3
python -m pytest tests/test_gpu_ties.py tests/test_gpu_slab.py -q -x 2>&1 | tail -3
python tools/c3_probe.py --horizon 2 --reps 1 --no-count > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:bellman_wide2' -c 1 \
    -o gpurun_out/r02c_c3_wide2 python tools/c3_probe.py --horizon 2 --reps 1 --no-count > gpurun_out/ncu_c.log 2>&1
tail -1 gpurun_out/ncu_c.log
