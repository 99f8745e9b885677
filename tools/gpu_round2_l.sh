python tools/c3_probe.py --horizon 2 --reps 1 --no-count > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:bellman_wide2' -c 1 \
    -o gpurun_out/r02e_c3_wide2 python tools/c3_probe.py --horizon 2 --reps 1 --no-count > gpurun_out/ncu_e.log 2>&1
tail -1 gpurun_out/ncu_e.log
python tools/c3_probe.py --horizon 20 --reps 2 --no-count > /dev/null 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3.csv \
    python tools/c3_probe.py --horizon 20 --reps 2 --no-count > /dev/null 2>&1
ls -la gpurun_out | tail -3
sha256sum paper_2104_01284_b200/_eco_b200.so | cut -c1-16 > gpurun_out/so_digest.txt
