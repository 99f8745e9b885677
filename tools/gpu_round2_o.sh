python -m pytest tests/test_gpu_checked.py -q 2>&1 | tail -2
ECO_B200_LIB=$PWD/paper_2104_01284_b200/_eco_b200_checked.so python tools/sanitize_cases.py 2>&1 | tail -2
python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['sweep_ms_per_stage'], d['roofline']['frac'])"
