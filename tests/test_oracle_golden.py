"""Pin the CPU oracle (oracle/eco_oracle.c) against reference-generated fixtures.

Every expected value below was produced by the reference package itself
(tests/golden/make_golden.py); tolerance is 0 everywhere — the oracle
restates the numba kernels with the same unfused double arithmetic.
"""

import math

import numpy as np
import pytest
from conftest import golden_json, golden_npz

from _toys import enumerate_costs, random_toy
from oracle import oracle as O
from paper_2104_01284_b200 import GridSpec, PenaltyConfig, build_context, table_digest

PEN = PenaltyConfig()
SMALL = GridSpec(n_v=12, n_soc=8, n_t=40, n_t_eng=8, n_t_bsg=10, horizon_steps=8)


def test_step_eval_matches_reference(vehicle):
    g = golden_npz("primitives.npz")
    for i in range(g["v"].size):
        got = O.step_eval(vehicle, g["v"][i], g["te"][i], g["tb"][i], 10.0, g["grade"][i], -3.0, 2.5, 0.0)
        exp = g["step"][i]
        assert got[0] == exp[0], i
        for j in range(1, 8):
            assert float(got[j]) == exp[j] or (math.isnan(exp[j]) and math.isnan(got[j])), (i, j)


def test_battery_and_locate_match_reference(vehicle):
    import ctypes as C
    from paper_2104_01284_b200 import _abi
    g = golden_npz("primitives.npz")
    p = _abi.pack_plant(vehicle.pack())
    for i in range(g["pb"].size):
        cur = C.c_double(0.0)
        ok = O.lib().oracle_battery_current(C.byref(p), g["pb"][i], g["soc"][i], C.byref(cur))
        assert (cur.value, float(ok)) == tuple(g["cur"][i])
    for i in range(g["xq"].size):
        assert tuple(map(float, O.locate_uniform(g["xq"][i], 0.0, 0.7, 35))) == tuple(g["loc"][i])


def test_signal_phase_matches_reference(short_route, urban_route):
    g = golden_npz("primitives.npz")
    _, spat = urban_route
    tm = spat.timing("tl1")
    for t, green, nxt in zip(g["ts"], g["green"], g["next_green"]):
        assert O.is_green(tm, t) == bool(green)
        if not green:
            assert O.next_green(tm, t) == nxt
    # Python floored remainder, not C fmod (route.py:69-70)
    assert O.pymod(-25.0, 60.0) == 35.0 == (-25.0 % 60.0)
    assert O.pymod(-1e-300, 60.0) == (-1e-300 % 60.0)


@pytest.mark.parametrize("seed", range(25))
def test_toys_serial_equal_reference_and_enumeration(seed):
    g = golden_npz("toys.npz")
    toy = random_toy(seed)
    J, P = O.solve_toy(toy)
    assert np.array_equal(J[0], g[f"enum_{seed}"])
    assert np.array_equal(enumerate_costs(random_toy(seed)), g[f"enum_{seed}"])
    for k in range(toy.horizon + 1):
        assert np.array_equal(J[k], g[f"J_{seed}_{k}"])
    for k in range(toy.horizon):
        assert np.array_equal(P[k], g[f"P_{seed}_{k}"])


@pytest.fixture(scope="module")
def c1_ctx(vehicle, short_route):
    route, spat = short_route
    return build_context(vehicle, route, spat, 45, 50.0, grids=GridSpec(n_v=12, n_soc=8, n_t=40), penalty=PEN,
                         gamma=0.5, horizon=20)


@pytest.mark.parametrize("parallel", [False, True])
def test_c1_solve_bitwise(c1_ctx, parallel):
    g = golden_npz("c1_short_s45_t50.npz")
    J, P = O.solve_context(c1_ctx, parallel=parallel, threads=4)
    assert np.array_equal(np.stack(J), g["J"])
    assert np.array_equal(np.stack(P), g["P"])


def test_c2_solves_match_reference_digests(vehicle, urban_route):
    route, spat = urban_route
    for case in golden_json("c2_urban_digests.json")[:3]:
        ctx = build_context(vehicle, route, spat, case["s"], case["t_start"], grids=GridSpec(), penalty=PEN,
                            gamma=0.5, horizon=20)
        J, P = O.solve_context(ctx, parallel=True)
        assert [table_digest(a) for a in J] == case["J"]
        assert [table_digest(a) for a in P] == case["P"]


def test_live_count_matches_survey(vehicle, urban_route):
    """U_live at C2 urban s=60 t=30: 114,537,119 (counted by the reference)."""
    route, spat = urban_route
    ctx = build_context(vehicle, route, spat, 60, 30.0, grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20)
    _, _, live_par = O.solve_context(ctx, parallel=True, with_live=True)
    assert live_par == 114_537_119


def test_field_short_small(vehicle, short_route):
    route, spat = short_route
    assert np.array_equal(O.field_build(vehicle, route, spat, SMALL, PEN, 0.5), golden_npz("fields.npz")["short_small"])


@pytest.mark.slow
def test_field_urban_default(vehicle, urban_route):
    route, spat = urban_route
    got = O.field_build(vehicle, route, spat, GridSpec(), PEN, 0.5)
    g = golden_npz("fields.npz")
    assert table_digest(got) == golden_json("fields_urban.json")["digest"]
    assert np.array_equal(got[g["urban_nodes"]], g["urban_slices"])


TRAJ_FIELDS = ("s", "v", "soc", "t", "t_eng", "t_bsg", "brake_force", "gear", "wait_s", "dt_move_s",
               "fuel_inc_g", "accel", "cost_to_go", "fallback")


def rows_as_matrix(rows) -> np.ndarray:
    return np.stack([rows[f].astype(np.float64) for f in TRAJ_FIELDS], axis=1)


def test_closed_loop_short_small(vehicle, short_route):
    route, spat = short_route
    g = golden_npz("loop_short_small.npz")
    fld = O.field_build(vehicle, route, spat, SMALL, PEN, 0.5)
    r = O.mpc_run(vehicle, route, spat, SMALL, PEN, 0.5, 8, (0.0, 0.5, 0.0), fld)
    assert r["status"] == 0
    assert np.array_equal(rows_as_matrix(r["rows"]), g["rows"], equal_nan=True)
    assert np.array_equal(r["final"], g["final"])
