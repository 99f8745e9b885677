"""Device runs of every kernel family through the public API, for the
self-checking build (compute-sanitizer is closed on this pool):

    ECO_B200_LIB=paper_2104_01284_b200/_eco_b200_checked.so python tools/sanitize_cases.py

prints the checked build's counters (gathers outside their buffers, stage
outputs not written exactly once) and exits 1 if either is nonzero; with the
regular build it only exercises the kernels.

Covers: toy tables (narrow stage kernel, per-state path), C1 (signal, red
wait), perturb_ties, a wide-row context (bellman_wide2_kernel + its per-state
fallback), the slab emulation (PEERS epilogue + copy-1 rebuild), the closed
loop (graph path and ring mode: seed / ladders / candidates / pick / field),
a small batch (bellman_batch_kernel)."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

from _toys import random_toy  # noqa: E402
from paper_2104_01284_b200 import (EcoDrivingMPC, GridSpec, PenaltyConfig, StateVector, build_context,  # noqa: E402
                                   load_fixture_route, make_vehicle, simulate_closed_loop, solve_horizon, solve_toy)
from paper_2104_01284_b200.mpc import MpcSession, clear_session_cache  # noqa: E402
from paper_2104_01284_b200.slab import emulate_slabs  # noqa: E402

pen = PenaltyConfig()
veh = make_vehicle()
short, sspat = load_fixture_route("short", seed=2)
urban, uspat = load_fixture_route("urban", seed=0)
for seed in (0, 3, 7):
    for b in ("b200", "b200-fp64"):
        solve_toy(random_toy(seed), backend=b)
print("toys ok", flush=True)
c1 = build_context(veh, short, sspat, 45, 50.0, grids=GridSpec(n_v=12, n_soc=8, n_t=40), penalty=pen, gamma=0.5,
                   horizon=6)
for b in ("b200", "b200-fp64"):
    solve_horizon(c1, backend=b)
    solve_horizon(c1, backend=b, perturb_ties=True)
print("c1 ok", flush=True)
wide = build_context(veh, urban, uspat, 150, 40.0, grids=GridSpec(n_v=16, n_soc=9, n_t=160, dt=0.5), penalty=pen,
                     gamma=0.5, horizon=3)
for b in ("b200", "b200-fp64"):
    solve_horizon(wide, backend=b)
J, P, _ = emulate_slabs(wide, 3, "b200")
print("wide + slab ok", flush=True)
small = GridSpec(n_v=12, n_soc=8, n_t=40, n_t_eng=8, n_t_bsg=10, horizon_steps=8)
mpc = EcoDrivingMPC(veh, gamma=0.5, grids=small, penalty=pen, horizon=8, backend="b200").fit(short, sspat)
simulate_closed_loop(short, sspat, mpc)
os.environ["ECO_RING"] = "1"
clear_session_cache()
sess = MpcSession(veh, short, sspat, gamma=0.5, grids=small, penalty=pen, horizon=8, backend="b200")
sess.fit(want_field=False)
sess.run(StateVector(0.0, 0.5, 0.0), 0, 12)
sess.close()
os.environ.pop("ECO_RING")
print("closed loops ok", flush=True)
from paper_2104_01284_b200.batch import BatchSolver  # noqa: E402
from paper_2104_01284_b200.fixtures import bench_schedule  # noqa: E402
sched = bench_schedule(urban, 6, 8, seed=0)
with BatchSolver(veh, urban, grids=GridSpec(n_v=10, n_soc=8, n_t=40), penalty=pen, gamma=0.5, horizon=6,
                 backend="b200") as bs:
    bs.solve([uspat] * len(sched), sched)
print("batch ok", flush=True)
# full-size stage kernels: C2 (narrow, staged band) and C3 (row blocks)
c2 = build_context(veh, urban, uspat, 60, 30.0, grids=GridSpec(), penalty=pen, gamma=0.5, horizon=4)
solve_horizon(c2, backend="b200")
c3 = build_context(veh, urban, uspat, 60, 30.0, grids=GridSpec(n_v=350, n_soc=260, n_t=400, dt=0.2), penalty=pen,
                   gamma=0.5, horizon=2)
solve_horizon(c3, backend="b200")
print("full-size stages ok", flush=True)
import ctypes as C  # noqa: E402
from paper_2104_01284_b200 import _abi  # noqa: E402
b, w = C.c_int64(0), C.c_int64(0)
_abi.check(_abi.lib().eco_debug_checks(C.byref(b), C.byref(w), 1), "eco_debug_checks")
print(f"checks bounds_violations={b.value} writer_violations={w.value}", flush=True)
sys.exit(1 if (b.value > 0 or w.value > 0) else 0)
