"""Generate the golden fixtures under tests/golden/ from the REFERENCE package.

Run only in the build container, where the read-only reference is importable:

    NUMBA_CACHE_DIR=/tmp/nbc PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py [--skip-urban-loop]

Nothing here imports the product or the oracle: every number comes from
``ecodrive`` itself (serial / parallel numba backends), so the fixtures pin
both the C oracle and the CUDA path.  The GPU box never runs this script.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/tests")

from ecodrive import _kernels as K  # noqa: E402
from ecodrive.bench import bench_schedule  # noqa: E402
from ecodrive.dp import GridSpec, PenaltyConfig, build_context, solve_horizon, solve_toy  # noqa: E402
from ecodrive.fixtures import load_fixture_route, make_route_urban, make_vehicle  # noqa: E402
from ecodrive.mpc import EcoDrivingMPC, build_terminal_cost, simulate_closed_loop  # noqa: E402
from ecodrive.parallel import table_digest  # noqa: E402
from ecodrive.route import load_route  # noqa: E402
from enum_oracle import enumerate_costs, random_toy  # noqa: E402

PEN = PenaltyConfig()
SMALL = GridSpec(n_v=12, n_soc=8, n_t=40, n_t_eng=8, n_t_bsg=10, horizon_steps=8)
TRAJ_FIELDS = ("s", "v", "soc", "t", "t_eng", "t_bsg", "brake_force", "gear", "wait_s", "dt_move_s",
               "fuel_inc_g", "accel", "cost_to_go", "fallback")


def traj_array(traj) -> np.ndarray:
    return np.array([[float(getattr(st, f)) for f in TRAJ_FIELDS] for st in traj.steps], dtype=np.float64)


def toys():
    out = {}
    for seed in range(25):
        toy = random_toy(seed)
        J, P = solve_toy(toy, backend="serial")
        out[f"enum_{seed}"] = enumerate_costs(toy)
        for k, a in enumerate(J):
            out[f"J_{seed}_{k}"] = a
        for k, a in enumerate(P):
            out[f"P_{seed}_{k}"] = a
    np.savez_compressed(HERE / "toys.npz", **out)


def c1():
    vehicle = make_vehicle()
    route, spat = load_fixture_route("short", seed=2)
    ctx = build_context(vehicle, route, spat, 45, 50.0, grids=GridSpec(n_v=12, n_soc=8, n_t=40),
                        penalty=PEN, gamma=0.5, horizon=20)
    res = solve_horizon(ctx, backend="serial")
    np.savez_compressed(HERE / "c1_short_s45_t50.npz",
                        J=np.stack([t.values for t in res.tables]),
                        P=np.stack([p.values for p in res.policies]))


def c2_digests():
    vehicle = make_vehicle()
    route, spat = load_fixture_route("urban", seed=0)
    cases = [(60, 30.0), (300, 100.0)] + bench_schedule(route, 20, 3, seed=0)
    out = []
    for s, t in cases:
        ctx = build_context(vehicle, route, spat, s, t, grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20)
        t0 = time.perf_counter()
        res = solve_horizon(ctx, backend="parallel", workers=8)
        wall = time.perf_counter() - t0
        J0 = res.tables[0].values
        fin = J0 < PEN.j_inf
        out.append({
            "s": s, "t_start": t, "wall_s_reference_parallel": wall,
            "J": [table_digest(tb.values) for tb in res.tables],
            "P": [table_digest(p.values) for p in res.policies],
            "J0_finite": int(fin.sum()), "J0_sum_finite": float(J0[fin].sum()),
        })
        print("c2", s, t, f"{wall:.3f}s", flush=True)
    (HERE / "c2_urban_digests.json").write_text(json.dumps(out, indent=1))


def c2_batch_seeds():
    """C4-style scenarios (route_i = urban seed i, bench_schedule seed i)."""
    vehicle = make_vehicle()
    out = []
    for i in range(4):
        route, spat = load_route(make_route_urban(seed=i))
        s, t = bench_schedule(route, 20, 1, seed=i)[0]
        ctx = build_context(vehicle, route, spat, s, t, grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20)
        res = solve_horizon(ctx, backend="parallel", workers=8)
        out.append({"seed": i, "s": s, "t_start": t, "J0": table_digest(res.tables[0].values),
                    "P0": table_digest(res.policies[0].values)})
    (HERE / "c4_batch_digests.json").write_text(json.dumps(out, indent=1))


def fields():
    vehicle = make_vehicle()
    route, spat = load_fixture_route("short", seed=2)
    f_small = build_terminal_cost(route, vehicle, gamma=0.5, grids=SMALL, penalty=PEN)
    route_u, _ = load_fixture_route("urban", seed=0)
    t0 = time.perf_counter()
    f_urban = build_terminal_cost(route_u, vehicle, gamma=0.5, grids=GridSpec(), penalty=PEN)
    print(f"urban field {time.perf_counter() - t0:.1f}s", flush=True)
    nodes = np.array([0, 79, 80, 150, 349, 520, 610, 698, 699])
    np.savez_compressed(HERE / "fields.npz", short_small=f_small.values, urban_nodes=nodes,
                        urban_slices=f_urban.values[nodes])
    (HERE / "fields_urban.json").write_text(json.dumps({"digest": table_digest(f_urban.values),
                                                        "shape": list(f_urban.values.shape)}))


def loop_short():
    vehicle = make_vehicle()
    route, spat = load_fixture_route("short", seed=2)
    mpc = EcoDrivingMPC(vehicle, gamma=0.5, grids=SMALL, penalty=PEN, horizon=8, backend="parallel").fit(route, spat)
    traj = simulate_closed_loop(route, spat, mpc)
    np.savez_compressed(HERE / "loop_short_small.npz", rows=traj_array(traj),
                        final=np.array([traj.final_state.v, traj.final_state.soc, traj.final_state.t]))
    # the reference's own byte-deterministic writers (io.py) on this run
    from ecodrive import io as rio
    rio.write_trajectory_csv(HERE / "loop_short_small_traj.csv", traj)
    rio.write_summary_json(HERE / "loop_short_small_summary.json", rio.summarize(traj))


def loop_urban():
    vehicle = make_vehicle()
    route, spat = load_fixture_route("urban", seed=0)
    t0 = time.perf_counter()
    mpc = EcoDrivingMPC(vehicle, gamma=0.5, grids=GridSpec(), penalty=PEN, horizon=20, backend="parallel",
                        workers=8).fit(route, spat)
    t1 = time.perf_counter()
    traj = simulate_closed_loop(route, spat, mpc)
    t2 = time.perf_counter()
    np.savez_compressed(HERE / "loop_urban_c2.npz", rows=traj_array(traj),
                        final=np.array([traj.final_state.v, traj.final_state.soc, traj.final_state.t]))
    (HERE / "loop_urban_c2.json").write_text(json.dumps({
        "status": traj.status, "n_steps": traj.n_steps, "fuel_g": traj.fuel_g,
        "travel_time_s": traj.travel_time_s, "soc_end": traj.soc_end,
        "fallbacks": int(sum(st.fallback for st in traj.steps)),
        "fit_s_reference": t1 - t0, "loop_s_reference_parallel8": t2 - t1,
    }, indent=1))


def c4_all():
    """All 4096 C4 scenarios (route_i = urban seed i, bench_schedule seed i):
    digests of each scenario's start-node J / P levels from the reference's
    parallel backend, plus the finite count and finite sum of J0 (for the
    fp32 tolerance checks)."""
    vehicle = make_vehicle()
    out = []
    t0 = time.perf_counter()
    for i in range(4096):
        route, spat = load_route(make_route_urban(seed=i))
        s, t = bench_schedule(route, 20, 1, seed=i)[0]
        ctx = build_context(vehicle, route, spat, s, t, grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20)
        res = solve_horizon(ctx, backend="parallel", workers=8)
        J0 = res.tables[0].values
        fin = J0 < PEN.j_inf
        out.append([i, int(s), float(t), table_digest(J0), table_digest(res.policies[0].values), int(fin.sum()),
                    float(J0[fin].sum())])
        if i % 256 == 0:
            print(f"c4 {i} {time.perf_counter() - t0:.0f}s", flush=True)
    (HERE / "c4_all_digests.json").write_text(json.dumps(
        {"fields": ["seed", "s", "t_start", "J0", "P0", "J0_finite", "J0_sum_finite"], "rows": out}))


C3_GRID = dict(n_v=350, n_soc=260, n_t=400, dt=0.2)
C3_SAMPLES = 16384


def c3():
    """C3: urban s=60, t=30, the fine grid, all 21 J / 20 P levels (digests of
    every level + a seeded sample of states for the fp32 tolerance checks)."""
    vehicle = make_vehicle()
    route, spat = load_fixture_route("urban", seed=0)
    ctx = build_context(vehicle, route, spat, 60, 30.0, grids=GridSpec(**C3_GRID), penalty=PEN, gamma=0.5,
                        horizon=20)
    t0 = time.perf_counter()
    res = solve_horizon(ctx, backend="parallel", workers=8)
    wall = time.perf_counter() - t0
    ns = res.tables[0].values.size
    idx = np.random.default_rng(2104).choice(ns, C3_SAMPLES, replace=False).astype(np.int64)
    idx.sort()
    Js = np.stack([tb.values.reshape(-1)[idx] for tb in res.tables])
    Ps = np.stack([p.values.reshape(-1)[idx] for p in res.policies])
    summ = []
    for tb in res.tables:
        fin = tb.values < PEN.j_inf
        summ.append({"finite": int(fin.sum()), "sum_finite": float(tb.values[fin].sum())})
    np.savez_compressed(HERE / "c3_urban_s60_t30_samples.npz", idx=idx, J=Js, P=Ps)
    (HERE / "c3_urban_s60_t30.json").write_text(json.dumps({
        "s": 60, "t_start": 30.0, "grid": C3_GRID, "horizon": 20,
        "wall_s_reference_parallel8": wall,
        "J": [table_digest(tb.values) for tb in res.tables],
        "P": [table_digest(p.values) for p in res.policies],
        "P_infeasible": [int((p.values < 0).sum()) for p in res.policies],
        "levels": summ,
    }, indent=1))
    print(f"c3 solve {wall:.1f}s", flush=True)


C3_LOOP_STEPS = 10


def loop_c3():
    """North-star target at the finest grid: EcoDrivingMPC(C3 grid).fit(urban)
    (terminal field on) and the first C3_LOOP_STEPS nodes of the closed loop,
    stepped exactly as simulate_closed_loop (mpc.py:549-596) steps them."""
    from ecodrive.errors import StartStateInfeasibleError
    from ecodrive.mpc import _max_braking_decision
    from ecodrive.plant import StateVector, propagate_state_full
    from ecodrive.route import NODE_SIGNAL
    vehicle = make_vehicle()
    route, spat = load_fixture_route("urban", seed=0)
    t0 = time.perf_counter()
    mpc = EcoDrivingMPC(vehicle, gamma=0.5, grids=GridSpec(**C3_GRID), penalty=PEN, horizon=20,
                        backend="parallel", workers=8).fit(route, spat)
    t_fit = time.perf_counter() - t0
    print(f"c3 field {t_fit:.1f}s", flush=True)
    fv = mpc.terminal_field_.values
    nodes = np.array([0, 20, 21, 25, 30, 80, 150, 698, 699])
    np.savez_compressed(HERE / "fields_c3.npz", urban_nodes=nodes, urban_slices=fv[nodes])
    kinds = route.node_kinds()
    x = StateVector(v=0.0, soc=0.5, t=0.0)
    rows, walls = [], []
    for s in range(C3_LOOP_STEPS):
        t1 = time.perf_counter()
        try:
            dec = mpc.control(x, s)
        except StartStateInfeasibleError as exc:
            dec = _max_braking_decision(vehicle, route, x, s, str(exc))
        walls.append(time.perf_counter() - t1)
        src = int(kinds[s])
        sig = spat.timing(route.traffic_lights[s]) if src == NODE_SIGNAL else None
        x_next, info = propagate_state_full(vehicle, x, dec.action, route.delta_d, grade=float(route.grade[s]),
                                            source_kind=src, dest_kind=int(kinds[s + 1]), signal=sig,
                                            stop_dwell=route.stop_dwell, teleport=True,
                                            brake_force=dec.brake_force)
        rows.append([s, x.v, x.soc, x.t, dec.action.t_eng, dec.action.t_bsg, dec.brake_force, info.gear,
                     info.wait, info.dt_move, info.fuel_g, info.accel, dec.cost_to_go, float(dec.fallback)])
        x = x_next
        print(f"c3 loop step {s}: {walls[-1]:.1f}s", flush=True)
    np.savez_compressed(HERE / "loop_urban_c3_prefix.npz", rows=np.array(rows, dtype=np.float64),
                        final=np.array([x.v, x.soc, x.t]))
    (HERE / "loop_urban_c3_prefix.json").write_text(json.dumps({
        "steps": C3_LOOP_STEPS, "grid": C3_GRID, "horizon": 20,
        "field_digest": table_digest(fv), "field_shape": list(fv.shape),
        "fit_s_reference": t_fit, "step_s_reference_parallel8": walls,
    }, indent=1))


def primitives():
    rng = np.random.default_rng(1234)
    vehicle = make_vehicle()
    pack = vehicle.pack()
    n = 2000
    v = rng.uniform(0.0, 17.0, n)
    v[:50] = 0.0
    te = rng.uniform(-45.0, 185.0, n)
    tb = rng.uniform(-60.0, 62.0, n)
    tb[50:100] = 0.0
    grade = rng.choice([0.0, 0.015, -0.015], n)
    out = np.zeros((n, 8))
    for i in range(n):
        r = K.step_eval(pack, v[i], te[i], tb[i], 10.0, grade[i], -3.0, 2.5, 0.0)
        out[i] = [r[0], r[1], float(r[2]), r[3], r[4], r[5], r[6], r[7]]
    pb = rng.uniform(-15000.0, 60000.0, n)
    soc = rng.uniform(0.25, 0.85, n)
    cur = np.array([[*K.battery_current(pack, pb[i], soc[i])] for i in range(n)], dtype=np.float64)
    xq = rng.uniform(-1.0, 30.0, n)
    xq[:200] = np.round(xq[:200])          # node-exact queries
    loc = np.array([[*K.locate_uniform(xq[i], 0.0, 0.7, 35)] for i in range(n)], dtype=np.float64)
    route, spat = load_fixture_route("urban", seed=0)
    tm = spat.timing("tl1")
    ts = rng.uniform(-200.0, 400.0, n)
    ts[:100] = np.round(ts[:100])
    green = np.array([tm.is_green(t) for t in ts])
    nxt = np.array([tm.next_green_from(t) if not tm.is_green(t) else np.nan for t in ts])
    np.savez_compressed(HERE / "primitives.npz", v=v, te=te, tb=tb, grade=grade, step=out, pb=pb, soc=soc,
                        cur=cur, xq=xq, loc=loc, ts=ts, green=green, next_green=nxt,
                        sig=np.array([tm.cycle, tm.offset, *tm.green_windows[0]]))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-urban-loop", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    jobs = [("primitives", primitives), ("toys", toys), ("c1", c1), ("fields", fields), ("loop_short", loop_short),
            ("c2", c2_digests), ("c4", c2_batch_seeds), ("c3", c3), ("loop_c3", loop_c3), ("c4_all", c4_all)]
    if not a.skip_urban_loop:
        jobs.append(("loop_urban", loop_urban))
    for name, fn in jobs:
        if a.only and name not in a.only.split(","):
            continue
        t0 = time.perf_counter()
        fn()
        print(f"{name}: {time.perf_counter() - t0:.1f}s", flush=True)
