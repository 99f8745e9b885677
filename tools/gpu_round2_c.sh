set -x
python -m pytest tests/test_gpu_finegrid.py -q -x -k "ring" 2>&1 | tail -5
python -m pytest tests/test_plugin.py -q -x 2>&1 | tail -3
ECO_DEBUG_IO=1 python tools/c3_probe.py --horizon 20 --reps 3 --no-count 2>&1 | tail -6
timeout 600 python bench.py --workload n1 --steps 2 --warmup 1 --loop-steps 5 --no-cpu-baseline > gpurun_out/b_n1.json 2> gpurun_out/b_n1.err; tail -c 2000 gpurun_out/b_n1.json; tail -5 gpurun_out/b_n1.err
