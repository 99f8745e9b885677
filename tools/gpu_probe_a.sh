set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for cm in 0 1; do ECO_CHUNK_MAJOR=$cm python tools/c3_probe.py --horizon 20 --reps 3 --no-count 2>&1 | tail -2; done
python tools/c3_probe.py --horizon 2 --reps 1 --no-count > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:bellman_wide' -c 1 \
    -o gpurun_out/r02a_c3_wide python tools/c3_probe.py --horizon 2 --reps 1 --no-count > gpurun_out/ncu_a.log 2>&1
tail -3 gpurun_out/ncu_a.log
