python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2104_01284_b200 import make_vehicle, load_fixture_route, GridSpec
from paper_2104_01284_b200.harness import run_bench
route, spat = load_fixture_route("urban", seed=0)
rep = run_bench(make_vehicle(), route, spat, grids=GridSpec(), horizon=20, backends=("b200", "b200-fp64"), reps=30, warmup=5)
print(rep.table())
PY
ECO_DEBUG_IO=1 python tools/c3_probe.py --horizon 20 --reps 3 --no-count 2>&1 | tail -3
