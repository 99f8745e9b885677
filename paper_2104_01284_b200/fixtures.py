"""Synthetic workloads: the 48 V P0 test vehicle, the urban / mixed / short
routes with seeded signal programs, and the seeded solve schedule.

These regenerate, value for value, the reference's synthetic inputs
(fixtures.py:32-251 and bench_schedule bench.py:76-94) so that benchmark and
parity workloads are the configurations BASELINE.json names.  Equality with
the reference generators is checked indirectly: every golden fixture under
tests/golden/ was produced by the reference from ITS generators, and the
tests rebuild the same inputs here and match those outputs bit for bit
(tests/test_oracle_golden.py, tests/test_gpu_parity.py).
"""

from __future__ import annotations

import numpy as np

from .plant import BatteryModel, BsgModel, EngineModel, Vehicle, VehicleParams
from .route import Route, SpatSchedule, load_route

# Willans-line synthetic fuel map (fixtures.py:25-29)
_WILLANS_EFF = 0.40
_LHV = 42.5e6
_LOSS_T0 = 14.0
_LOSS_T1 = 0.018


def make_vehicle() -> Vehicle:
    """Compact car with a belt starter-generator (fixtures.py:32-94)."""
    chassis = VehicleParams(
        mass=1530.0, c0=135.0, c1=3.2, c2=0.42, wheel_radius=0.307, final_drive=3.9,
        gear_ratios=(3.92, 2.29, 1.52, 1.13, 0.91, 0.77),
        gear_efficiencies=(0.95, 0.95, 0.96, 0.96, 0.965, 0.965),
        shift_speeds=(4.5, 8.0, 12.0, 16.5, 21.0),
        idle_speed=78.5,
    )
    w_f = np.linspace(78.5, 550.0, 10)
    t_f = np.linspace(0.0, 170.0, 12)
    W, T = np.meshgrid(w_f, t_f, indexing="ij")
    fuel = (T + (_LOSS_T0 + _LOSS_T1 * W)) * W / (_WILLANS_EFF * _LHV) * 1000.0
    engine = EngineModel(
        speed_axis=np.array([78.5, 120.0, 160.0, 200.0, 260.0, 320.0, 400.0, 480.0, 550.0]),
        torque_min=np.array([-12.0, -14.0, -16.0, -18.0, -21.0, -25.0, -30.0, -36.0, -42.0]),
        torque_max=np.array([95.0, 125.0, 150.0, 160.0, 160.0, 155.0, 145.0, 130.0, 110.0]),
        fuel_speed_axis=w_f, fuel_torque_axis=t_f, fuel_map=fuel,
    )
    w_b = np.array([210.0, 400.0, 700.0, 1000.0, 1500.0])
    t_cap = np.minimum(58.0, 13000.0 / w_b)
    w_e = np.array([210.0, 600.0, 1000.0, 1500.0])
    t_e = np.array([0.0, 15.0, 30.0, 45.0, 60.0])
    WE, TE = np.meshgrid(w_e, t_e, indexing="ij")
    eff = np.clip(0.91 - 0.035 * (WE / 1500.0) - 0.045 * (TE / 60.0), 0.80, 0.92)
    bsg = BsgModel(belt_ratio=2.7, speed_axis=w_b, torque_min=-t_cap, torque_max=t_cap,
                   eff_speed_axis=w_e, eff_torque_axis=t_e, eff_map=eff)
    battery = BatteryModel(
        r0=0.012, c_nom=36000.0,
        voc_soc_axis=np.array([0.20, 0.35, 0.50, 0.65, 0.80, 0.90]),
        voc=np.array([45.2, 46.4, 47.5, 48.6, 49.8, 50.6]),
        soc_min=0.30, soc_max=0.80,
    )
    return Vehicle(params=chassis, engine=engine, bsg=bsg, battery=battery,
                   name="synthetic-48v-p0")


def _signal_doc(rng: np.random.Generator, green_frac: float) -> dict:
    """One fixed-time program with every edge on the 2 s ladder (fixtures.py:97-103)."""
    cycle = float(rng.choice([60, 70, 80]))
    green = 2.0 * round(cycle * green_frac / 2.0)
    green = min(max(green, 10.0), cycle - 10.0)
    offset = 2.0 * float(rng.integers(0, int(cycle // 2)))
    return {"cycle_s": cycle, "offset_s": offset, "green_windows_s": [[0.0, green]]}


def _route_doc(name, n, v_max, grade, lights, stops, rng) -> dict:
    signals = {}
    for i in range(len(lights)):
        frac = rng.uniform(0.45, 0.62)
        signals[f"tl{i + 1}"] = _signal_doc(rng, frac)
    return {
        "name": name, "node_count": n, "delta_d_m": 10.0, "v_min_mps": 0.0,
        "v_max_mps": v_max, "grade_rad": grade,
        "accel_min_mps2": -3.0, "accel_max_mps2": 2.5, "stop_dwell_s": 2.0,
        "traffic_lights": [{"node": node, "signal": f"tl{i + 1}"} for i, node in enumerate(lights)],
        "stop_signs": list(stops), "signals": signals,
    }


def make_route_urban(seed: int = 0) -> dict:
    """7 km arterial, 5 signals, 2 stop signs (fixtures.py:106-132)."""
    v_max = np.full(700, 13.9)
    v_max[100:350] = 15.3
    v_max[350:550] = 16.7
    return _route_doc("urban-7km", 700, v_max.tolist(), 0.0, [80, 210, 330, 450, 610],
                      [150, 520], np.random.default_rng(seed))


def make_route_mixed(seed: int = 1) -> dict:
    """7.5 km mixed route with a graded rural middle (fixtures.py:135-164)."""
    rng = np.random.default_rng(seed)
    v_max = np.full(750, 15.3)
    v_max[:60] = 13.9
    v_max[250:550] = 22.2
    grade = np.zeros(750)
    grade[300:400] = 0.015
    grade[400:500] = -0.015
    return _route_doc("mixed-7p5km", 750, v_max.tolist(), grade.tolist(), [70, 180, 640], [230], rng)


def make_route_short(seed: int = 2) -> dict:
    """1.2 km single-signal route (fixtures.py:167-185)."""
    rng = np.random.default_rng(seed)
    doc = _route_doc("short-1p2km", 120, 13.9, 0.0, [], [], rng)
    doc["signals"] = {"tl1": _signal_doc(rng, 0.5)}
    doc["traffic_lights"] = [{"node": 60, "signal": "tl1"}]
    return doc


def load_fixture_route(kind: str, seed: int = 0):
    """(Route, SpatSchedule) of a bundled route (fixtures.py:243-251)."""
    makers = {"urban": (make_route_urban, 0), "mixed": (make_route_mixed, 1),
              "short": (make_route_short, 2)}
    if kind not in makers:
        raise ValueError(f"unknown fixture route kind: {kind!r}")
    fn, shift = makers[kind]
    return load_route(fn(seed + shift))


def bench_schedule(route: Route, horizon: int, count: int, seed: int = 0) -> list:
    """Seeded (start node, start time) pairs (bench.py:76-94)."""
    s_hi = route.node_count - 1 - horizon
    if s_hi < 0:
        raise ValueError(f"route of {route.node_count} nodes cannot host a {horizon}-step horizon")
    rng = np.random.default_rng(seed)
    nodes = rng.integers(0, s_hi + 1, size=count)
    times = rng.uniform(0.0, 120.0, size=count)
    return [(int(s), float(t)) for s, t in zip(nodes, times)]


__all__ = ["make_vehicle", "make_route_urban", "make_route_mixed", "make_route_short",
           "load_fixture_route", "bench_schedule", "Route", "SpatSchedule"]
