# geometry builder A/B: fit time, then parity of everything that reads the tile plans
for V in 1 0; do echo "== ECO_PLANE_TILES=$V"; ECO_PLANE_TILES=$V python tools/fit_probe.py | tail -2; done
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
ECO_PLANE_TILES=1 python tools/c3_probe.py --horizon 2 --reps 1 --no-count 2>&1 | tail -3
ECO_PLANE_TILES=0 python tools/c3_probe.py --horizon 2 --reps 1 --no-count 2>&1 | tail -3
