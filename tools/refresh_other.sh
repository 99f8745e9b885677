#!/bin/bash
# CLI GPU test + the C3 / C4 / C5 bench lines
R=${1:-r01}
python -m pytest tests/test_cli.py -m gpu -q -x 2>&1 | tail -2
for W in c3 c4 c5; do
  python bench.py --workload $W > gpurun_out/${R}_bench_$W.json 2> gpurun_out/${R}_bench_$W.err
  tail -1 gpurun_out/${R}_bench_$W.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W', d['value'], d.get('ms_per_step'), d['e2e']['value'], d['roofline']['frac'])"
done
