"""Time EcoDrivingMPC.fit pieces on the C2 route (geometry + terminal field)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_01284_b200 import GridSpec, PenaltyConfig, load_fixture_route, make_vehicle
from paper_2104_01284_b200.mpc import MpcSession
veh = make_vehicle(); route, spat = load_fixture_route("urban", seed=0)
s = MpcSession(veh, route, spat, gamma=0.5, grids=GridSpec(), penalty=PenaltyConfig(), horizon=20, backend="b200")
for i in range(4):
    t0 = time.perf_counter()
    _, st = s.fit(want_field=False)
    print(f"fit wall {1e3 * (time.perf_counter() - t0):.2f} ms device {st['device_ms']:.2f} field sweeps {st['dominant_ms']:.2f} launches {st['kernel_launches']}", flush=True)
