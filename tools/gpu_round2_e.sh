set -x
for w in 0 1; do ECO_WIDE2=$w ECO_DEBUG_IO=1 python tools/c3_probe.py --horizon 20 --reps 3 2>&1 | tail -4; done
python -m pytest tests/test_gpu_parity.py -q -x -k "c3" 2>&1 | tail -3
python -m pytest tests/test_gpu_ties.py tests/test_gpu_slab.py -q -x 2>&1 | tail -3
python -m pytest tests/test_gpu_parity.py -q -x -k "wide" 2>&1 | tail -3
