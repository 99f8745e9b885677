python -m pytest tests/test_gpu_finegrid.py -q -x 2>&1 | tail -15
