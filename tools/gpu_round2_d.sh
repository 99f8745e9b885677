set -x
./tools/d2h_bw
nvidia-smi -q | grep -i -A3 "PCI\b\|Link Width\|Max Link Gen\|Current" | head -30
nvidia-smi topo -m | head -5
python -m pytest tests/test_gpu_slab.py -q -x 2>&1 | tail -5
