python tools/c3_probe.py --horizon 20 --reps 3 --no-count 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
