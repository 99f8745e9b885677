python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['sweep_ms_per_stage'], d['roofline']['frac'])"
python bench.py --workload c4 --steps 2 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], d['ms_per_step'], d['roofline']['frac'])"
python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties.py tests/test_harness.py -q -x 2>&1 | tail -2
