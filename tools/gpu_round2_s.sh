PYTHONPATH=. python tools/solve_probe.py 2>&1 | tail -3
