"""Short C2 workload for profiling: fit + the first N receding-horizon steps
of the urban closed loop (default grid) on one session."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2104_01284_b200 import GridSpec, PenaltyConfig, StateVector, load_fixture_route, make_vehicle  # noqa
from paper_2104_01284_b200.mpc import MpcSession  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--start", type=int, default=60)
ap.add_argument("--precision", default="fp32")
a = ap.parse_args()
vehicle = make_vehicle()
route, spat = load_fixture_route("urban", seed=0)
sess = MpcSession(vehicle, route, spat, gamma=0.5, grids=GridSpec(), penalty=PenaltyConfig(), horizon=20,
                  backend="b200" if a.precision == "fp32" else "b200-fp64")
sess.fit(want_field=False)
rows, status, _, fin, st = sess.run(StateVector(8.0, 0.5, 30.0), start_node=a.start, max_steps=a.steps)
print("status", status, "rows", len(rows), st)
