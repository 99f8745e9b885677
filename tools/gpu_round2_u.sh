timeout 900 python tools/n1_full.py fp32 gpurun_out 2>&1 | tail -3
