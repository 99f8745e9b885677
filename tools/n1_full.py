"""The north-star Target run end to end through the public API: the C3-grid
controller fitted on the 700-node urban route and driven over the whole route
(699 receding-horizon solves at 350 x 260 x 400 x 23 x 30, H = 20), with the
reference's experiment files written.  Usage: python tools/n1_full.py [fp32|fp64] [outdir]"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2104_01284_b200 import (EcoDrivingMPC, GridSpec, PenaltyConfig, load_fixture_route,  # noqa: E402
                                   make_vehicle, simulate_closed_loop)
from paper_2104_01284_b200 import io as eio  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
out = Path(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out")
out.mkdir(exist_ok=True)
backend = "b200" if prec == "fp32" else "b200-fp64"
route, spat = load_fixture_route("urban", seed=0)
t0 = time.perf_counter()
mpc = EcoDrivingMPC(make_vehicle(), gamma=0.5, grids=GridSpec(n_v=350, n_soc=260, n_t=400, dt=0.2),
                    penalty=PenaltyConfig(), horizon=20, backend=backend).fit(route, spat)
t1 = time.perf_counter()
traj = simulate_closed_loop(route, spat, mpc)
t2 = time.perf_counter()
eio.write_trajectory_csv(out / f"n1_{prec}_trajectory.csv", traj)
eio.write_timing_csv(out / f"n1_{prec}_timing.csv", traj)
summ = eio.summarize(traj)
eio.write_summary_json(out / f"n1_{prec}_summary.json", summ)
res = {"backend": backend, "status": traj.status, "n_steps": traj.n_steps, "fuel_g": traj.fuel_g,
       "travel_time_s": traj.travel_time_s, "soc_end": traj.soc_end,
       "fallbacks": int(sum(st.fallback for st in traj.steps)), "fit_wall_s": t1 - t0, "loop_wall_s": t2 - t1,
       "solve_ms_mean": 1e3 * sum(traj.solver_wall_s) / max(1, len(traj.solver_wall_s)),
       "solve_ms_max": 1e3 * max(traj.solver_wall_s) if traj.solver_wall_s else None,
       "loop_stats": traj.stats}
print(json.dumps(res))
(out / f"n1_{prec}_result.json").write_text(json.dumps(res, indent=1))
