python -m pytest tests/test_gpu_ties.py tests/test_gpu_slab_ipc.py -q -x 2>&1 | tail -15
