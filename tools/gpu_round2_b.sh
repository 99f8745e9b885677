# round-2 check: new GPU tests, C3 default bench line, reference arm (short)
set -x
python -m pytest tests/test_gpu_ties.py tests/test_plugin.py -q -x 2>&1 | tail -5
python -m pytest tests/test_gpu_parity.py -q -x -k "c3" 2>&1 | tail -5
python bench.py --steps 5 --warmup 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; tail -c 3000 gpurun_out/b_c3.json; tail -5 gpurun_out/b_c3.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; tail -c 1500 gpurun_out/b_ref.json; tail -3 gpurun_out/b_ref.err
nproc; free -g | head -2
