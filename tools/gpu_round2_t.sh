PYTHONPATH=. python tools/solve_probe.py 2>&1 | tail -2
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
