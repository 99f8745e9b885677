ECO_B200_LIB=$PWD/paper_2104_01284_b200/_eco_b200_checked.so python tools/sanitize_cases.py 2>&1 | tail -4
python -m pytest tests/test_gpu_checked.py -q 2>&1 | tail -2
python tools/c3_probe.py --horizon 20 --reps 3 --no-count 2>&1 | tail -1
