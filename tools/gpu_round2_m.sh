python tools/c3_probe.py --horizon 20 --reps 3 --no-count 2>&1 | tail -1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_ties.py tests/test_gpu_finegrid.py -q -x 2>&1 | tail -2
python tools/sanitize_cases.py 2>&1 | tail -2
