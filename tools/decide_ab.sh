# closed-loop parity, then the C2 bench line twice
python -m pytest tests/test_gpu_parity.py tests/test_harness.py -m gpu -x -q -k "closed_loop or mpc_step or session or step_locked or byte" 2>&1 | tail -2
for V in 1 2; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['ms_per_solve'], d['sweep_ms_per_stage'], d['value'], d['e2e']['value'], d['roofline']['frac'])"
done
