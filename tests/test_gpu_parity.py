"""CUDA path vs the reference (golden fixtures) and the pinned CPU oracle.

Bar (north_star / SURVEY §8c):
  * backend "b200-fp64": bitwise equal — max |dJ| = 0, 0 policy mismatches,
    closed-loop trajectories identical row for row;
  * backend "b200" (f32 value path, f64 geometry): toys bitwise (dyadic
    arithmetic is exact in f32); on the plant, finite-mask agreement >= 99.9 %,
    both-finite |dJ| / max(1, |J|) <= 1e-4 at p99.9 and <= 1e-3 max, argmin
    agreement >= 99.9 %; closed-loop fuel and travel time within 0.1 %.
"""

import math

import numpy as np
import pytest
from conftest import golden_json, golden_npz

from _toys import random_toy
from oracle import oracle as O
from paper_2104_01284_b200 import (EcoDrivingMPC, GridSpec, PenaltyConfig, StartStateInfeasibleError, StateVector,
                                   backward_step, build_context, build_terminal_cost, mpc_step, simulate_closed_loop,
                                   solve_horizon, solve_toy, table_digest)

pytestmark = pytest.mark.gpu

PEN = PenaltyConfig()
SMALL = GridSpec(n_v=12, n_soc=8, n_t=40, n_t_eng=8, n_t_bsg=10, horizon_steps=8)
TRAJ_FIELDS = ("s", "v", "soc", "t", "t_eng", "t_bsg", "brake_force", "gear", "wait_s", "dt_move_s",
               "fuel_inc_g", "accel", "cost_to_go", "fallback")

# f32 tolerance of the cost-to-go (stated in DESIGN.md §5)
REL_P999 = 1e-4
REL_MAX = 1e-3


def fp32_agreement(J32, P32, J64, P64, j_inf=PEN.j_inf):
    f32, f64 = J32 < j_inf, J64 < j_inf
    mask_agree = float(np.mean(f32 == f64))
    both = f32 & f64
    rel = np.abs(J32[both] - J64[both]) / np.maximum(1.0, np.abs(J64[both]))
    pol = float(np.mean(P32[both] == P64[both])) if both.any() else 1.0
    return mask_agree, (float(np.quantile(rel, 0.999)) if rel.size else 0.0), \
        (float(rel.max()) if rel.size else 0.0), pol


# ------------------------------------------------------------------ toys

@pytest.mark.parametrize("backend", ["b200-fp64", "b200"])
@pytest.mark.parametrize("seed", range(25))
def test_toys_equal_reference(seed, backend):
    g = golden_npz("toys.npz")
    toy = random_toy(seed)
    J, P = solve_toy(toy, backend=backend)
    assert np.array_equal(J[0], g[f"enum_{seed}"])
    for k in range(toy.horizon + 1):
        assert np.array_equal(J[k], g[f"J_{seed}_{k}"])
    for k in range(toy.horizon):
        assert np.array_equal(P[k], g[f"P_{seed}_{k}"])


def test_toy_all_infeasible():
    toy = random_toy(13, horizon=1)
    toy.stage1[0]["ok"][:] = 0
    J, P = solve_toy(toy, backend="b200")
    assert np.all(J[0] >= toy.j_inf) and np.all(P[0] == -1)


def test_toy_tie_rule_lowest_flat_action():
    toy = random_toy(11, horizon=1)
    t = toy.stage1[0]
    t["ok"][:] = 1
    t["c1"][:] = 0.5
    t["pbat"][:] = 0.0
    t["dt"][:] = 2.0
    t["v2"][:] = 1.0 if toy.v_axis.shape[0] > 1 else 0.0
    toy.arr_green[0][:] = 1
    toy.dep_ok[0][:] = 1
    toy.wait[0][:] = 0.0
    toy.src_kinds[0] = 0
    toy.terminal[:] = 0.0
    for backend in ("b200", "b200-fp64"):
        _, P = solve_toy(toy, backend=backend)
        feas = P[0] >= 0
        assert feas.any() and np.all(P[0][feas] == 0)


def test_toy_red_arrival_gate():
    toy = random_toy(5, horizon=1)
    t = toy.stage1[0]
    t["ok"][:] = 1
    t["c1"][:] = 1.0
    t["pbat"][:] = 0.0
    t["dt"][:] = 2.0
    toy.src_kinds[0] = 0
    toy.dep_ok[0][:] = 1
    toy.wait[0][:] = 0.0
    toy.terminal[:] = 0.0
    toy.arr_green[0][:] = 0
    t["v2"][:] = 1.0
    J_moving, _ = solve_toy(toy, backend="b200")
    t["v2"][:] = 0.0
    J_stop, _ = solve_toy(toy, backend="b200")
    assert np.all(J_moving[0] >= toy.j_inf)
    assert (J_stop[0] < toy.j_inf).any()


# ------------------------------------------------------------- plant solves

@pytest.fixture(scope="module")
def c1_ctx(vehicle, short_route):
    route, spat = short_route
    return build_context(vehicle, route, spat, 45, 50.0, grids=GridSpec(n_v=12, n_soc=8, n_t=40), penalty=PEN,
                         gamma=0.5, horizon=20)


def test_c1_fp64_bitwise(c1_ctx):
    g = golden_npz("c1_short_s45_t50.npz")
    res = solve_horizon(c1_ctx, backend="b200-fp64")
    assert np.array_equal(np.stack([t.values for t in res.tables]), g["J"])
    assert np.array_equal(np.stack([p.values for p in res.policies]), g["P"])


def test_c1_fp32_within_tolerance(c1_ctx):
    g = golden_npz("c1_short_s45_t50.npz")
    res = solve_horizon(c1_ctx, backend="b200")
    J = np.stack([t.values for t in res.tables])
    P = np.stack([p.values for p in res.policies])
    mask, p999, mx, pol = fp32_agreement(J[:-1], P, g["J"][:-1], g["P"])
    assert mask >= 0.999 and p999 <= REL_P999 and mx <= REL_MAX and pol >= 0.999, (mask, p999, mx, pol)


def test_c1_backward_step_matches(c1_ctx):
    g = golden_npz("c1_short_s45_t50.npz")
    J, P = backward_step(c1_ctx, 7, g["J"][8], backend="b200-fp64")
    assert np.array_equal(J, g["J"][7]) and np.array_equal(P, g["P"][7])


def test_c2_fp64_digests_and_live_count(vehicle, urban_route):
    route, spat = urban_route
    for i, case in enumerate(golden_json("c2_urban_digests.json")):
        ctx = build_context(vehicle, route, spat, case["s"], case["t_start"], grids=GridSpec(), penalty=PEN,
                            gamma=0.5, horizon=20)
        res = solve_horizon(ctx, backend="b200-fp64", count_live=(i == 0))
        assert [table_digest(t.values) for t in res.tables] == case["J"]
        assert [table_digest(p.values) for p in res.policies] == case["P"]
        if i == 0:
            assert (case["s"], case["t_start"]) == (60, 30.0)
            assert res.stats["live_updates"] == 114_537_119


def test_c2_fp32_tolerance(vehicle, urban_route):
    route, spat = urban_route
    for case in golden_json("c2_urban_digests.json"):
        ctx = build_context(vehicle, route, spat, case["s"], case["t_start"], grids=GridSpec(), penalty=PEN,
                            gamma=0.5, horizon=20)
        r64 = solve_horizon(ctx, backend="b200-fp64")
        r32 = solve_horizon(ctx, backend="b200")
        J64 = np.stack([t.values for t in r64.tables[:-1]])
        J32 = np.stack([t.values for t in r32.tables[:-1]])
        P64 = np.stack([p.values for p in r64.policies])
        P32 = np.stack([p.values for p in r32.policies])
        mask, p999, mx, pol = fp32_agreement(J32, P32, J64, P64)
        assert mask >= 0.999 and p999 <= REL_P999 and mx <= REL_MAX and pol >= 0.999, (case["s"], mask, p999, mx, pol)


def test_c4_scenarios_fp64(vehicle):
    from paper_2104_01284_b200.fixtures import make_route_urban
    from paper_2104_01284_b200.route import load_route
    for case in golden_json("c4_batch_digests.json"):
        route, spat = load_route(make_route_urban(seed=case["seed"]))
        ctx = build_context(vehicle, route, spat, case["s"], case["t_start"], grids=GridSpec(), penalty=PEN,
                            gamma=0.5, horizon=20)
        res = solve_horizon(ctx, backend="b200-fp64")
        assert table_digest(res.tables[0].values) == case["J0"]
        assert table_digest(res.policies[0].values) == case["P0"]


def test_start_state_infeasible_raises(vehicle, short_route):
    route, spat = short_route
    ctx = build_context(vehicle, route, spat, 45, 50.0, grids=GridSpec(n_v=12, n_soc=8, n_t=40), penalty=PEN,
                        gamma=0.5, horizon=4)
    with pytest.raises(StartStateInfeasibleError):
        solve_horizon(ctx, StateVector(v=13.0, soc=0.31, t=200.0), backend="b200")


def test_solver_random_contexts_vs_oracle(vehicle, short_route):
    """Seeded start nodes / clocks incl. the signal and red waits (standstill relocation)."""
    route, spat = short_route
    rng = np.random.default_rng(7)
    grids = GridSpec(n_v=9, n_soc=7, n_t=24, n_t_eng=11, n_t_bsg=13)
    for _ in range(6):
        s = int(rng.integers(40, 70))
        t = float(rng.uniform(-30.0, 150.0))
        ctx = build_context(vehicle, route, spat, s, t, grids=grids, penalty=PEN, gamma=float(rng.uniform(0, 1)),
                            horizon=int(rng.integers(1, 9)), teleport=bool(rng.integers(0, 2)))
        J, P = O.solve_context(ctx)
        res = solve_horizon(ctx, backend="b200-fp64")
        for k in range(ctx.horizon):
            assert np.array_equal(res.tables[k].values, J[k]), (s, t, k)
            assert np.array_equal(res.policies[k].values, P[k]), (s, t, k)


# ---------------------------------------------------------- field and loop

def test_field_short_small_fp64(vehicle, short_route):
    route, spat = short_route
    f = build_terminal_cost(route, vehicle, gamma=0.5, grids=SMALL, penalty=PEN, backend="b200-fp64")
    assert np.array_equal(f.values, golden_npz("fields.npz")["short_small"])


def test_field_urban_default_fp64(vehicle, urban_route):
    route, spat = urban_route
    f = build_terminal_cost(route, vehicle, gamma=0.5, grids=GridSpec(), penalty=PEN, backend="b200-fp64")
    assert table_digest(f.values) == golden_json("fields_urban.json")["digest"]


def test_field_urban_fp32(vehicle, urban_route):
    route, spat = urban_route
    gz = golden_npz("fields.npz")
    g = gz["urban_slices"]
    f = build_terminal_cost(route, vehicle, gamma=0.5, grids=GridSpec(), penalty=PEN,
                            backend="b200").values[gz["urban_nodes"]]
    fin = g < PEN.j_inf
    assert np.mean((f < PEN.j_inf) == fin) >= 0.999
    both = fin & (f < PEN.j_inf)
    assert np.max(np.abs(f[both] - g[both]) / np.maximum(1, np.abs(g[both]))) <= REL_MAX


def rows_matrix(traj) -> np.ndarray:
    return np.array([[float(getattr(st, f)) for f in TRAJ_FIELDS] for st in traj.steps])


def test_closed_loop_short_fp64_identical(vehicle, short_route):
    route, spat = short_route
    g = golden_npz("loop_short_small.npz")
    mpc = EcoDrivingMPC(vehicle, gamma=0.5, grids=SMALL, penalty=PEN, horizon=8, backend="b200-fp64").fit(route, spat)
    traj = simulate_closed_loop(route, spat, mpc)
    assert traj.status == "ok" and traj.n_steps == route.node_count - 1
    assert np.array_equal(rows_matrix(traj), g["rows"], equal_nan=True)
    fs = traj.final_state
    assert np.array_equal([fs.v, fs.soc, fs.t], g["final"])


def test_closed_loop_short_fp32_totals(vehicle, short_route):
    route, spat = short_route
    g = golden_npz("loop_short_small.npz")
    mpc = EcoDrivingMPC(vehicle, gamma=0.5, grids=SMALL, penalty=PEN, horizon=8, backend="b200").fit(route, spat)
    traj = simulate_closed_loop(route, spat, mpc)
    assert traj.status == "ok"
    fuel_ref = g["rows"][:, TRAJ_FIELDS.index("fuel_inc_g")].sum()
    assert abs(traj.fuel_g - fuel_ref) <= 1e-3 * fuel_ref
    assert abs(traj.final_state.t - g["final"][2]) <= 1e-3 * g["final"][2]
    for st in traj.steps:
        sid = route.traffic_lights.get(st.s)
        if sid is not None and st.v > 0.0:
            assert spat.timing(sid).is_green(st.t)


def test_mpc_step_matches_gridded_policy(vehicle, short_route):
    """mpc.py:168-191 contract: on-grid state -> the solved policy's action."""
    route, spat = short_route
    fld = build_terminal_cost(route, vehicle, gamma=0.5, grids=SMALL, penalty=PEN, backend="b200-fp64")
    iv, jx = 4, 3
    x = StateVector(v=float(SMALL.v_axis(route, 0)[iv]), soc=float(SMALL.soc_axis(vehicle)[jx]), t=0.0)
    action, info = mpc_step(vehicle, route, spat, x, 0, gamma=0.5, grids=SMALL, penalty=PEN, horizon=8,
                            terminal=fld, backend="b200-fp64")
    ctx = build_context(vehicle, route, spat, 0, 0.0, grids=SMALL, penalty=PEN, gamma=0.5, horizon=8,
                        terminal_field=fld.node_slice(8))
    res = solve_horizon(ctx, backend="b200-fp64")
    assert (action.t_eng, action.t_bsg) == res.policies[0].action(iv, jx, 0)
    assert info.horizon == 8 and info.wait == 0.0 and math.isfinite(info.cost_to_go)


def test_mpc_step_errors(vehicle, short_route):
    route, spat = short_route
    with pytest.raises(ValueError):
        mpc_step(vehicle, route, spat, StateVector(5.0, 0.5, 0.0), route.node_count - 1, gamma=0.5, grids=SMALL,
                 penalty=PEN, horizon=8)
    _, info = mpc_step(vehicle, route, spat, StateVector(8.0, 0.5, 0.0), route.node_count - 2, gamma=0.5,
                       grids=SMALL, penalty=PEN, horizon=8)
    assert info.horizon == 1


@pytest.mark.slow
def test_closed_loop_urban_c2_fp64_identical(vehicle, urban_route):
    route, spat = urban_route
    g = golden_npz("loop_urban_c2.npz")
    mpc = EcoDrivingMPC(vehicle, gamma=0.5, grids=GridSpec(), penalty=PEN, horizon=20,
                        backend="b200-fp64").fit(route, spat)
    traj = simulate_closed_loop(route, spat, mpc)
    assert traj.status == "ok"
    assert np.array_equal(rows_matrix(traj), g["rows"], equal_nan=True)


def test_closed_loop_urban_c2_fp32_within_0p1pct(vehicle, urban_route):
    route, spat = urban_route
    ref = golden_json("loop_urban_c2.json")
    mpc = EcoDrivingMPC(vehicle, gamma=0.5, grids=GridSpec(), penalty=PEN, horizon=20, backend="b200").fit(route, spat)
    traj = simulate_closed_loop(route, spat, mpc)
    assert traj.status == "ok" and traj.n_steps == ref["n_steps"]
    assert abs(traj.fuel_g - ref["fuel_g"]) <= 1e-3 * ref["fuel_g"], (traj.fuel_g, ref["fuel_g"])
    assert abs(traj.travel_time_s - ref["travel_time_s"]) <= 1e-3 * ref["travel_time_s"]


# ------------------------------------------------------------ C3 fine grid

C3_GRID = GridSpec(n_v=350, n_soc=260, n_t=400, dt=0.2)


@pytest.fixture(scope="module")
def c3_short_ctx(vehicle, urban_route):
    route, spat = urban_route
    return build_context(vehicle, route, spat, 60, 30.0, grids=C3_GRID, penalty=PEN, gamma=0.5, horizon=2)


def test_c3_fine_grid_fp64_bitwise_vs_oracle(c3_short_ctx):
    """C3 (350 x 260 x 400, dt = 0.2): two stages against the OpenMP oracle."""
    from paper_2104_01284_b200.dp import solve_stacks
    J, P, _ = solve_stacks(c3_short_ctx, "b200-fp64")
    Jo, Po = O.solve_context(c3_short_ctx, parallel=True)
    for k in range(2):
        assert np.array_equal(J[k], Jo[k]), k
        assert np.array_equal(P[k], Po[k]), k


@pytest.fixture(scope="module")
def c3_full_ctx(vehicle, urban_route):
    route, spat = urban_route
    return build_context(vehicle, route, spat, 60, 30.0, grids=C3_GRID, penalty=PEN, gamma=0.5, horizon=20)


def test_c3_full_horizon_fp64_bitwise_vs_reference(c3_full_ctx):
    """C3 at the full H = 20 against the REFERENCE's own solve
    (solve_horizon(backend="parallel"), tests/golden/make_golden.py c3):
    blake2b digests of all 21 J and 20 P levels equal."""
    from paper_2104_01284_b200.dp import solve_stacks
    g = golden_json("c3_urban_s60_t30.json")
    J, P, st = solve_stacks(c3_full_ctx, "b200-fp64")
    assert st["stages"] == 20
    for k in range(21):
        assert table_digest(J[k]) == g["J"][k], f"J level {k}"
    for k in range(20):
        assert table_digest(P[k]) == g["P"][k], f"P level {k}"


def test_c3_full_horizon_fp32_within_tolerance_vs_reference(c3_full_ctx):
    """The fp32 production build at C3, every level, against the reference's
    values: finite counts and sums of every level, and the stated tolerances
    on 16,384 seeded state samples per level (golden c3 samples)."""
    from paper_2104_01284_b200.dp import solve_stacks
    g = golden_json("c3_urban_s60_t30.json")
    smp = golden_npz("c3_urban_s60_t30_samples.npz")
    idx = smp["idx"]
    J, P, st = solve_stacks(c3_full_ctx, "b200", count_live=True)
    assert st["live_updates"] > 0
    for k in range(21):
        lvl = g["levels"][k]
        fin = J[k] < PEN.j_inf
        n_fin = int(fin.sum())
        assert abs(n_fin - lvl["finite"]) <= 1e-3 * lvl["finite"], (k, n_fin, lvl["finite"])
        s = float(J[k][fin].sum())
        assert abs(s - lvl["sum_finite"]) <= 1e-4 * lvl["sum_finite"], (k, s, lvl["sum_finite"])
        Js = J[k].reshape(-1)[idx]
        Pk = P[k].reshape(-1)[idx] if k < 20 else np.zeros_like(idx, dtype=np.int32)
        Pr = smp["P"][k] if k < 20 else np.zeros_like(idx, dtype=np.int32)
        mask, p999, mx, pol = fp32_agreement(Js, Pk, smp["J"][k], Pr)
        assert mask >= 0.999 and p999 <= REL_P999 and mx <= REL_MAX and pol >= 0.999, (k, mask, p999, mx, pol)


# ------------------------------------------------------------- C4 batch

def _c4_scenarios(n, H=20):
    from paper_2104_01284_b200.fixtures import bench_schedule, make_route_urban
    from paper_2104_01284_b200.route import load_route
    routes = [load_route(make_route_urban(seed=i)) for i in range(n)]
    sched = [bench_schedule(r, H, 1, seed=i)[0] for i, (r, _) in enumerate(routes)]
    return routes, sched


def test_c4_batch_fp64_digests(vehicle):
    """The four golden C4 scenarios (reference solve_horizon digests) in one batch."""
    from paper_2104_01284_b200.batch import solve_batch
    cases = golden_json("c4_batch_digests.json")
    routes, sched = _c4_scenarios(len(cases))
    assert [(c["s"], c["t_start"]) for c in cases] == sched
    res = solve_batch(vehicle, routes[0][0], [sp for _, sp in routes], sched, grids=GridSpec(), penalty=PEN,
                      gamma=0.5, horizon=20, backend="b200-fp64")
    for i, case in enumerate(cases):
        assert table_digest(res.J0[i]) == case["J0"], i
        assert table_digest(res.P0[i]) == case["P0"], i


def test_c4_batch_matches_single_solves(vehicle):
    """fp32 batch == fp32 solve_horizon per scenario, bitwise (same geometry,
    same tiles), incl. horizons clipped at the route end and repeated solves."""
    from paper_2104_01284_b200.batch import BatchSolver
    routes, sched = _c4_scenarios(12)
    sched[3] = (690, 17.25)        # h = 9
    sched[7] = (698, 3.5)          # h = 1
    spats = [sp for _, sp in routes]
    with BatchSolver(vehicle, routes[0][0], grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20) as bs:
        res = bs.solve(spats, sched, count_live=True)
        res2 = bs.solve(spats[::-1], sched[::-1])
    assert list(res.horizons) == [20] * 3 + [9] + [20] * 3 + [1] + [20] * 4
    assert res.stats["live_updates"] > 0
    for i, ((route, spat), (s, t)) in enumerate(zip(routes, sched)):
        ctx = build_context(vehicle, route, spat, s, t, grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20)
        r = solve_horizon(ctx, backend="b200")
        assert np.array_equal(res.J0[i], r.tables[0].values), i
        assert np.array_equal(res.P0[i], r.policies[0].values), i
        assert np.array_equal(res2.J0[len(sched) - 1 - i], res.J0[i]), i


def test_c4_batch_fp32_tolerance(vehicle):
    from paper_2104_01284_b200.batch import BatchSolver
    routes, sched = _c4_scenarios(64)
    spats = [sp for _, sp in routes]
    kw = dict(grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20)
    with BatchSolver(vehicle, routes[0][0], backend="b200-fp64", **kw) as b64, \
            BatchSolver(vehicle, routes[0][0], backend="b200", **kw) as b32:
        r64, r32 = b64.solve(spats, sched), b32.solve(spats, sched)
    mask, p999, mx, pol = fp32_agreement(r32.J0, r32.P0, r64.J0, r64.P0)
    assert mask >= 0.999 and p999 <= REL_P999 and mx <= REL_MAX and pol >= 0.999, (mask, p999, mx, pol)


@pytest.fixture(scope="module")
def c4_all():
    from conftest import GOLDEN
    if not (GOLDEN / "c4_all_digests.json").exists():
        pytest.skip("C4 all-scenario golden not generated")
    g = golden_json("c4_all_digests.json")
    routes, sched = _c4_scenarios(len(g["rows"]))
    assert [(r[1], r[2]) for r in g["rows"]] == [(int(s), float(t)) for s, t in sched]
    return g["rows"], routes, sched


def test_c4_all_4096_scenarios_fp64_vs_reference(vehicle, c4_all):
    """All 4096 C4 scenarios in one batch against the REFERENCE's own
    solve_horizon(backend="parallel") per scenario: J0 / P0 digests equal."""
    from paper_2104_01284_b200.batch import BatchSolver
    rows, routes, sched = c4_all
    with BatchSolver(vehicle, routes[0][0], grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20,
                     backend="b200-fp64") as bs:
        res = bs.solve([sp for _, sp in routes], sched)
    bad = [r[0] for i, r in enumerate(rows)
           if table_digest(res.J0[i]) != r[3] or table_digest(res.P0[i]) != r[4]]
    assert not bad, bad[:20]


def test_c4_all_4096_scenarios_fp32_vs_reference(vehicle, c4_all):
    """The fp32 batch against the reference: every scenario's J0 finite count
    within 0.1 % and finite sum within 1e-4 of the reference's."""
    from paper_2104_01284_b200.batch import BatchSolver
    rows, routes, sched = c4_all
    with BatchSolver(vehicle, routes[0][0], grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20,
                     backend="b200") as bs:
        res = bs.solve([sp for _, sp in routes], sched)
    for i, r in enumerate(rows):
        fin = res.J0[i] < PEN.j_inf
        n, ssum = int(fin.sum()), float(res.J0[i][fin].sum())
        assert abs(n - r[5]) <= 1e-3 * max(1, r[5]), (i, n, r[5])
        assert abs(ssum - r[6]) <= 1e-4 * max(1.0, r[6]), (i, ssum, r[6])


def test_c4_batch_terminal_field_and_no_teleport(vehicle):
    """Options of build_context: the offline terminal field and teleport=False."""
    from paper_2104_01284_b200.batch import solve_batch
    routes, sched = _c4_scenarios(3)
    spats = [sp for _, sp in routes]
    field = build_terminal_cost(routes[0][0], vehicle, gamma=0.5, grids=GridSpec(), penalty=PEN,
                                backend="b200-fp64")
    res = solve_batch(vehicle, routes[0][0], spats, sched, grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20,
                      teleport=False, terminal_field=True, backend="b200-fp64")
    for i, ((route, spat), (s, t)) in enumerate(zip(routes, sched)):
        ctx = build_context(vehicle, route, spat, s, t, grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20,
                            teleport=False, terminal_field=field.values[s + min(20, route.node_count - 1 - s)])
        J, P = O.solve_context(ctx, parallel=True)
        assert np.array_equal(res.J0[i], J[0]) and np.array_equal(res.P0[i], P[0]), i


# ------------------------------------------------------- C5 slab (1 rank)

@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
@pytest.mark.parametrize("backend", ["b200-fp64", "b200"])
def test_slab_solver_single_rank_equals_solve_horizon(vehicle, urban_route, exchange, backend):
    """The slab path on one GPU (world 1) runs the same kernels with the
    plane-range tile order and the exchange plumbing; results must equal the
    unpartitioned solve bitwise.  (Multi-rank exchange: tests/test_slab_host.py.)"""
    from paper_2104_01284_b200.slab import SlabSolver
    route, spat = urban_route
    ctx = build_context(vehicle, route, spat, 60, 30.0, grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20)
    ref = solve_horizon(ctx, backend=backend)
    with SlabSolver(35, 26, 40, 20, backend=backend, exchange=exchange, rank=0, world=1) as ss:
        for _ in range(2):
            res = ss.solve(ctx, return_J=True)
            assert res.planes == (0, 35)
            for k in range(21):
                assert np.array_equal(res.J[k], ref.tables[k].values), k
            for k in range(20):
                assert np.array_equal(res.P[k], ref.policies[k].values), k


def test_closed_loop_files_byte_identical_to_reference(vehicle, short_route, tmp_path):
    """The fp64 device loop written with io.py's format: the trajectory CSV is
    byte-identical to the reference's file; the summary differs only in the
    backend name."""
    import json
    from conftest import GOLDEN
    from paper_2104_01284_b200.io import summarize, write_summary_json, write_trajectory_csv
    route, spat = short_route
    mpc = EcoDrivingMPC(vehicle, gamma=0.5, grids=SMALL, penalty=PEN, horizon=8, backend="b200-fp64").fit(route, spat)
    traj = simulate_closed_loop(route, spat, mpc)
    write_trajectory_csv(tmp_path / "t.csv", traj)
    assert (tmp_path / "t.csv").read_bytes() == (GOLDEN / "loop_short_small_traj.csv").read_bytes()
    write_summary_json(tmp_path / "s.json", summarize(traj))
    ours = json.loads((tmp_path / "s.json").read_text())
    ref = json.loads((GOLDEN / "loop_short_small_summary.json").read_text())
    assert ours.pop("backend") == "b200-fp64" and ref.pop("backend") == "parallel"
    assert ours == ref


def test_session_route_reupload_matches_fresh_session(vehicle):
    """A cached session fed another route's data (same node count) behaves
    exactly like a fresh session on that route (geometry, field, graphs)."""
    from paper_2104_01284_b200 import load_fixture_route
    from paper_2104_01284_b200.mpc import MpcSession
    r1, sp1 = load_fixture_route("short", seed=2)
    r2, sp2 = load_fixture_route("short", seed=5)
    kw = dict(gamma=0.5, grids=SMALL, penalty=PEN, horizon=8, backend="b200-fp64")
    x0 = StateVector(v=0.0, soc=0.5, t=0.0)
    with_fresh = MpcSession(vehicle, r2, sp2, **kw)
    with_fresh.fit(want_field=False)
    rows_f, st_f, _, fin_f, _ = with_fresh.run(x0)
    reused = MpcSession(vehicle, r1, sp1, **kw)
    reused.fit(want_field=False)
    reused.run(x0)                           # captures graphs on route 1
    reused.upload_route(r2, sp2)
    reused.fit(want_field=False)
    rows_r, st_r, _, fin_r, _ = reused.run(x0)
    assert st_f == st_r and np.array_equal(fin_f, fin_r)
    assert rows_f.tobytes() == rows_r.tobytes()
    with_fresh.close(); reused.close()


@pytest.mark.parametrize("nt", [128, 129, 130, 192, 256, 258, 322, 400, 434, 435, 512])
def test_wide_row_path_vs_oracle(vehicle, urban_route, nt):
    """Long ladders take the wide-row kernels: odd chunk counts, partial last
    chunks, ranges that end exactly on / one past a warp segment, the
    compiled n_t = 400 instantiation, the longest row-block ladder (7 warps x
    62 states = 434) and the first one past it; fp64 bitwise against the
    oracle, fp32 within tolerance (incl. the signal at node 80 inside the
    horizon: red gates, standstill relocation)."""
    route, spat = urban_route
    grids = GridSpec(n_v=7, n_soc=5, n_t=nt, dt=0.25)
    for s, t in [(62, 31.0), (76, 5.5)]:
        ctx = build_context(vehicle, route, spat, s, t, grids=grids, penalty=PEN, gamma=0.5, horizon=6)
        J, P = O.solve_context(ctx)
        r64 = solve_horizon(ctx, backend="b200-fp64")
        for k in range(ctx.horizon):
            assert np.array_equal(r64.tables[k].values, J[k]), (nt, s, k)
            assert np.array_equal(r64.policies[k].values, P[k]), (nt, s, k)
        r32 = solve_horizon(ctx, backend="b200")
        J32 = np.stack([x.values for x in r32.tables[:-1]])
        P32 = np.stack([x.values for x in r32.policies])
        mask, p999, mx, pol = fp32_agreement(J32, P32, np.stack(J[:-1]), np.stack(P))
        assert mask >= 0.999 and p999 <= REL_P999 and mx <= REL_MAX and pol >= 0.999, (nt, s, mask, p999, mx, pol)


@pytest.mark.slow
def test_c4_full_batch_fp32_vs_fp64(vehicle):
    """All 4096 C4 scenarios: the fp32 start-node tables against the fp64
    build (bitwise to the reference on the golden scenarios)."""
    from paper_2104_01284_b200 import _abi
    from paper_2104_01284_b200.batch import BatchSolver
    routes, sched = _c4_scenarios(4096)
    tim = _abi.signal_timings(routes[0][0], [sp for _, sp in routes])
    kw = dict(grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20)
    with BatchSolver(vehicle, routes[0][0], backend="b200-fp64", **kw) as b:
        r64 = b.solve(None, sched, timings=tim)
    with BatchSolver(vehicle, routes[0][0], backend="b200", **kw) as b:
        r32 = b.solve(None, sched, timings=tim)
    mask, p999, mx, pol = fp32_agreement(r32.J0, r32.P0, r64.J0, r64.P0)
    assert mask >= 0.999 and p999 <= REL_P999 and mx <= REL_MAX and pol >= 0.999, (mask, p999, mx, pol)


def test_closed_loop_step_clocks(vehicle, short_route):
    """Per-step solve clocks (device timestamps) behind the timing CSV."""
    route, spat = short_route
    mpc = EcoDrivingMPC(vehicle, gamma=0.5, grids=SMALL, penalty=PEN, horizon=8, backend="b200").fit(route, spat)
    traj = simulate_closed_loop(route, spat, mpc)
    w = np.asarray(traj.solver_wall_s)
    assert w.shape == (traj.n_steps,) and np.all(w > 0) and np.all(w < 0.05)
    assert abs(w.sum() * 1e3 - traj.stats["dominant_ms"]) <= 1e-6 * max(1.0, traj.stats["dominant_ms"])
    dec = mpc.control(StateVector(v=5.0, soc=0.5, t=0.0), 3)
    assert 0 < dec.solver_wall_s < 0.05


DIFF = GridSpec(n_v=20, n_soc=14, n_t=40, n_t_eng=16, n_t_bsg=20)


@pytest.mark.parametrize("kind,seed,grid,horizon,gamma,teleport", [
    ("short", 2, SMALL, 8, 0.0, True),        # max-brake fallbacks on the way
    ("short", 2, SMALL, 8, 1.0, False),       # red light without teleport: the plant step fails at node 54
    ("mixed", 1, DIFF, 20, 0.5, True),
    ("mixed", 1, DIFF, 20, 0.25, False),
    ("urban", 3, DIFF, 20, 0.8, True),
])
def test_closed_loop_variants_fp64_vs_oracle(vehicle, kind, seed, grid, horizon, gamma, teleport):
    """Whole closed loops (field, every solve, decision, plant step) on other
    routes, trade-offs and teleport settings: rows, status, failure node and
    final state bit for bit against the oracle's closed loop."""
    from paper_2104_01284_b200 import load_fixture_route
    route, spat = load_fixture_route(kind, seed=seed)
    fld = O.field_build(vehicle, route, spat, grid, PEN, gamma)
    ref = O.mpc_run(vehicle, route, spat, grid, PEN, gamma, horizon, (0.0, 0.5, 0.0), fld, teleport=teleport)
    mpc = EcoDrivingMPC(vehicle, gamma=gamma, grids=grid, penalty=PEN, horizon=horizon, backend="b200-fp64",
                        teleport=teleport).fit(route, spat)
    assert np.array_equal(mpc.terminal_field_.values, fld)
    rows, status, node, fin, _ = mpc.session_.run(StateVector(v=0.0, soc=0.5, t=0.0))
    assert (status, len(rows)) == (ref["status"], len(ref["rows"]))
    if status != 0:
        assert node == ref["status_node"]
    for f in rows.dtype.names:
        assert np.array_equal(rows[f], ref["rows"][f], equal_nan=True), f
    assert np.array_equal(fin, ref["final"])


@pytest.mark.parametrize("kind,seed,gamma", [("mixed", 1, 0.5), ("urban", 3, 0.8)])
def test_closed_loop_variants_fp32_within_0p1pct(vehicle, kind, seed, gamma):
    """fp32 production loop on other routes: fuel and travel time within 0.1 %
    of the oracle's fp64 closed loop (north_star's closed-loop bar)."""
    from paper_2104_01284_b200 import load_fixture_route
    route, spat = load_fixture_route(kind, seed=seed)
    fld = O.field_build(vehicle, route, spat, DIFF, PEN, gamma)
    ref = O.mpc_run(vehicle, route, spat, DIFF, PEN, gamma, 20, (0.0, 0.5, 0.0), fld)
    mpc = EcoDrivingMPC(vehicle, gamma=gamma, grids=DIFF, penalty=PEN, horizon=20, backend="b200").fit(route, spat)
    traj = simulate_closed_loop(route, spat, mpc)
    assert traj.status == "ok" and ref["status"] == 0
    fuel_ref = float(np.sum(ref["rows"]["fuel_inc_g"]))
    assert abs(traj.fuel_g - fuel_ref) <= 1e-3 * fuel_ref, (traj.fuel_g, fuel_ref)
    assert abs(traj.final_state.t - ref["final"][2]) <= 1e-3 * ref["final"][2], (traj.final_state.t, ref["final"][2])


def test_c3_compiled_ladder_equals_runtime_ladder(c3_short_ctx, monkeypatch):
    """The n_t = 400 instantiation of the row-block kernel (compile-time
    ladder length) and the runtime-n_t kernel (ECO_W2_NTC=0) give the same
    tables and policies bit for bit, fp64 and fp32."""
    from paper_2104_01284_b200.dp import solve_stacks
    for backend in ("b200-fp64", "b200"):
        monkeypatch.delenv("ECO_W2_NTC", raising=False)
        J1, P1, _ = solve_stacks(c3_short_ctx, backend)
        monkeypatch.setenv("ECO_W2_NTC", "0")
        J0, P0, _ = solve_stacks(c3_short_ctx, backend)
        assert np.array_equal(J1, J0) and np.array_equal(P1, P0), backend


def test_c3_host_widened_levels_equal_device_conversion(c3_short_ctx, monkeypatch):
    """Large fp32 solves send each level as f32 and widen it on the host
    (ECO_HOST_WIDEN): the tables equal the device-side f64 conversion bitwise."""
    from paper_2104_01284_b200.dp import solve_stacks
    J1, P1, _ = solve_stacks(c3_short_ctx, "b200")
    monkeypatch.setenv("ECO_HOST_WIDEN", "0")
    J0, P0, _ = solve_stacks(c3_short_ctx, "b200")
    assert np.array_equal(J1, J0) and np.array_equal(P1, P0)
    assert np.all(J1[J1 >= PEN.j_inf] == PEN.j_inf)
