"""C5 slab path on one GPU vs the plain C3 solve (same kernels): timing probe."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_01284_b200 import GridSpec, PenaltyConfig, build_context, load_fixture_route, make_vehicle
from paper_2104_01284_b200.dp import solve_stacks
from paper_2104_01284_b200.slab import SlabSolver
veh = make_vehicle(); route, spat = load_fixture_route("urban", seed=0)
ctx = build_context(veh, route, spat, 60, 30.0, grids=GridSpec(n_v=350, n_soc=260, n_t=400, dt=0.2),
                    penalty=PenaltyConfig(), gamma=0.5, horizon=20)
for i in range(3):
    st = solve_stacks(ctx, "b200")[2]
    print("solve_stacks", st["device_ms"], st["dominant_ms"], flush=True)
ss = SlabSolver(350, 260, 400, 20, rank=0, world=1, exchange=sys.argv[1] if len(sys.argv) > 1 else "p2p")
for i in range(3):
    st = ss.solve(ctx, return_P=False).stats
    print("slab", st["device_ms"], st["dominant_ms"], flush=True)
