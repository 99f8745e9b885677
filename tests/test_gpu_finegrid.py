"""North-star Target: the receding-horizon closed loop at the finest grid
(C3: 350 x 260 x 400 states, dt = 0.2 s, x 23 x 30 controls, H = 20) on one
B200, through the route session's ring of plan slots.

* ring mode is bitwise the all-route-geometry mode: forced on at C2
  (ECO_RING=1) the 699-step urban loop and the short-route loop (with its
  max-brake fallbacks and the shrinking horizon at the route end) equal the
  reference's trajectories row for row in fp64, and the chunked terminal
  field equals the reference's field;
* at C3 the fit (terminal field over the 700-node route, chunked) and the
  first 10 closed-loop nodes match the REFERENCE run
  (EcoDrivingMPC(C3 grid).fit(urban) + simulate_closed_loop's stepping,
  tests/golden/make_golden.py loop_c3): fp64 bitwise, fp32 within 0.1 % on
  fuel and travel time.
"""

import numpy as np
import pytest
from conftest import GOLDEN, golden_json, golden_npz

from paper_2104_01284_b200 import (EcoDrivingMPC, GridSpec, PenaltyConfig, StateVector, simulate_closed_loop,
                                   table_digest)
from paper_2104_01284_b200.mpc import MpcSession, clear_session_cache

pytestmark = pytest.mark.gpu

PEN = PenaltyConfig()
SMALL = GridSpec(n_v=12, n_soc=8, n_t=40, n_t_eng=8, n_t_bsg=10, horizon_steps=8)
C3 = GridSpec(n_v=350, n_soc=260, n_t=400, dt=0.2)
FIELDS = ("s", "v", "soc", "t", "t_eng", "t_bsg", "brake_force", "gear", "wait_s", "dt_move_s", "fuel_inc_g",
          "accel", "cost_to_go", "fallback")


def rows_of(rows) -> np.ndarray:
    return np.array([[float(r[f]) for f in FIELDS] for r in rows])


@pytest.fixture
def ring_on(monkeypatch):
    monkeypatch.setenv("ECO_RING", "1")
    clear_session_cache()
    yield
    clear_session_cache()


def test_ring_mode_short_loop_fp64_identical(ring_on, vehicle, short_route):
    route, spat = short_route
    g = golden_npz("loop_short_small.npz")
    sess = MpcSession(vehicle, route, spat, gamma=0.5, grids=SMALL, penalty=PEN, horizon=8, backend="b200-fp64")
    sess.fit(want_field=False)
    rows, status, _, fin, st = sess.run(StateVector(0.0, 0.5, 0.0))
    assert status == 0 and len(rows) == route.node_count - 1
    assert np.array_equal(rows_of(rows), g["rows"], equal_nan=True)
    assert np.array_equal(fin, g["final"])
    # single steps (EcoDrivingMPC.control) reuse the slots already built
    r1, *_ = sess.run(StateVector(*g["rows"][5, 1:4]), start_node=5, max_steps=1)
    assert np.array_equal(rows_of(r1)[0], g["rows"][5], equal_nan=True)
    sess.close()


def test_ring_mode_urban_c2_fp64_identical(ring_on, vehicle, urban_route):
    route, spat = urban_route
    g = golden_npz("loop_urban_c2.npz")
    fg = golden_json("fields_urban.json")
    mpc = EcoDrivingMPC(vehicle, gamma=0.5, grids=GridSpec(), penalty=PEN, horizon=20,
                        backend="b200-fp64").fit(route, spat)
    assert table_digest(mpc.terminal_field_.values) == fg["digest"]      # chunked field sweep
    traj = simulate_closed_loop(route, spat, mpc)
    assert traj.status == "ok"
    got = np.array([[float(getattr(st, f)) for f in FIELDS] for st in traj.steps])
    assert np.array_equal(got, g["rows"], equal_nan=True)


def _c3_prefix_golden():
    if not (GOLDEN / "loop_urban_c3_prefix.npz").exists():
        pytest.skip("C3 closed-loop golden not generated")
    return golden_npz("loop_urban_c3_prefix.npz"), golden_json("loop_urban_c3_prefix.json")


@pytest.fixture(scope="module")
def c3_fp64_session(vehicle, urban_route):
    route, spat = urban_route
    sess = MpcSession(vehicle, route, spat, gamma=0.5, grids=C3, penalty=PEN, horizon=20, backend="b200-fp64")
    field, fst = sess.fit(want_field=True)
    yield sess, field, fst
    sess.close()


def test_c3_terminal_field_fp64_equals_reference(c3_fp64_session):
    g, meta = _c3_prefix_golden()
    _, field, fst = c3_fp64_session
    assert list(field.shape) == meta["field_shape"]
    assert table_digest(field) == meta["field_digest"]
    fz = np.load(GOLDEN / "fields_c3.npz")
    assert np.array_equal(field[fz["urban_nodes"]], fz["urban_slices"])
    assert fst["stages"] == field.shape[0] - 1


def test_c3_closed_loop_prefix_fp64_identical(c3_fp64_session):
    """The north-star Target run: receding-horizon solves at the finest grid,
    the decision at the exact state and the plant step, node after node."""
    g, meta = _c3_prefix_golden()
    sess, _, _ = c3_fp64_session
    n = meta["steps"]
    rows, status, _, fin, st = sess.run(StateVector(0.0, 0.5, 0.0), start_node=0, max_steps=n)
    assert status == 0 and len(rows) == n
    assert np.array_equal(rows_of(rows), g["rows"], equal_nan=True)
    assert np.array_equal(fin, g["final"])
    assert st["stages"] == 20 * n


def test_c3_closed_loop_prefix_fp32_within_0p1pct(vehicle, urban_route):
    g, meta = _c3_prefix_golden()
    route, spat = urban_route
    n = meta["steps"]
    sess = MpcSession(vehicle, route, spat, gamma=0.5, grids=C3, penalty=PEN, horizon=20, backend="b200")
    sess.fit(want_field=False)
    rows, status, _, fin, st = sess.run(StateVector(0.0, 0.5, 0.0), start_node=0, max_steps=n)
    sess.close()
    assert status == 0 and len(rows) == n
    got = rows_of(rows)
    fuel, fuel_ref = got[:, FIELDS.index("fuel_inc_g")].sum(), g["rows"][:, FIELDS.index("fuel_inc_g")].sum()
    assert abs(fuel - fuel_ref) <= 1e-3 * fuel_ref, (fuel, fuel_ref)
    assert abs(fin[2] - g["final"][2]) <= 1e-3 * g["final"][2], (fin, g["final"])
    assert abs(fin[0] - g["final"][0]) <= 1e-3 * max(1.0, g["final"][0])
