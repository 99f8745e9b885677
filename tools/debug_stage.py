"""One C2 urban solve with per-CTA timing of each stage kernel (ECO_DEBUG_STAGE=1)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ[os.environ.get("DBGVAR", "ECO_DEBUG_STAGE")] = "1"
from paper_2104_01284_b200 import GridSpec, PenaltyConfig, build_context, load_fixture_route, make_vehicle, solve_horizon
veh = make_vehicle(); route, spat = load_fixture_route("urban", seed=0)
ctx = build_context(veh, route, spat, 300, 100.0, grids=GridSpec(), penalty=PenaltyConfig(), gamma=0.5, horizon=20)
for _ in range(2):
    r = solve_horizon(ctx, backend="b200")
print(r.stats)
