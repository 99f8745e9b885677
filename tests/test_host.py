"""CPU-side checks: host mirror of the reference interface, fixtures, the C ABI
library surface (loads and exports every declared symbol; no compute
without a GPU), and loud failure when no device is present."""

import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest
from conftest import ROOT, golden_npz

from oracle import oracle as O
from paper_2104_01284_b200 import (GridSpec, NativeLibraryError, PenaltyConfig, SignalTiming, SpatSchedule,
                                   build_context, dump_tables, load_tables, solve_horizon)
from paper_2104_01284_b200 import _abi
from paper_2104_01284_b200.dp import CostToGoTable, PolicyTable, SolveResult, locate_uniform, terminal_seed
from paper_2104_01284_b200.errors import RouteFormatError
from paper_2104_01284_b200.route import Route, load_route

PEN = PenaltyConfig()


def test_header_symbols_exported():
    lib = _abi.lib()
    names = re.findall(r"^\w[\w\s\*]*?\b(eco_\w+)\(", (ROOT / "include" / "eco_b200.h").read_text(), re.M)
    assert len(names) >= 9
    for n in names:
        assert hasattr(lib, n), n
    assert lib.eco_abi_version() == _abi.ABI_VERSION


def test_library_targets_sm100a():
    blob = (ROOT / "paper_2104_01284_b200" / "_eco_b200.so").read_bytes()
    assert b"sm_100a" in blob


def test_no_device_fails_loudly(vehicle, short_route):
    if _abi.lib().eco_device_count() > 0:
        pytest.skip("a GPU is visible")
    route, spat = short_route
    ctx = build_context(vehicle, route, spat, 45, 50.0, grids=GridSpec(n_v=4, n_soc=3, n_t=5), penalty=PEN,
                        gamma=0.5, horizon=2)
    with pytest.raises(NativeLibraryError, match="no CUDA device"):
        solve_horizon(ctx, backend="b200")


def test_unknown_backend_rejected(vehicle, short_route):
    route, spat = short_route
    ctx = build_context(vehicle, route, spat, 45, 50.0, grids=GridSpec(n_v=4, n_soc=3, n_t=5), penalty=PEN,
                        gamma=0.5, horizon=2)
    for bad in ("serial", "parallel", "cpu", ""):
        with pytest.raises(ValueError, match="unknown backend"):
            solve_horizon(ctx, backend=bad)


def test_context_validation(vehicle, short_route):
    route, spat = short_route
    with pytest.raises(ValueError):
        build_context(vehicle, route, spat, route.node_count - 1, 0.0, grids=GridSpec(), penalty=PEN, gamma=0.5)
    with pytest.raises(ValueError):
        build_context(vehicle, route, spat, 0, 0.0, grids=GridSpec(), penalty=PEN, gamma=1.5)
    with pytest.raises(ValueError):
        GridSpec(n_v=1)
    with pytest.raises(ValueError):
        PenaltyConfig(j_inf=0.0)
    ctx = build_context(vehicle, route, spat, route.node_count - 3, 0.0, grids=GridSpec(), penalty=PEN, gamma=0.5)
    assert ctx.horizon == 2                       # horizon clipped at the route end (dp.py:280-281)


def test_linspace_axes_match_numpy():
    for a, b, n in [(0.0, 13.9, 35), (0.3, 0.8, 26), (0.0, 16.7, 350), (-40.0, 180.0, 23), (0.0, 1.0, 2)]:
        assert np.array_equal(O.linspace(a, b, n), np.linspace(a, b, n))


def test_ladders_and_terminal_match_reference_semantics(vehicle, short_route):
    route, spat = short_route
    ctx = build_context(vehicle, route, spat, 45, 50.0, grids=GridSpec(n_v=12, n_soc=8, n_t=40), penalty=PEN,
                        gamma=0.5, horizon=20)
    tm = spat.timing("tl1")
    k = 60 - 45
    st = ctx.steps[k]                             # departure from the signal node
    for z, tz in enumerate(ctx.t_axis):
        if tm.is_green(tz):
            assert st.dep_ok[z] == 1 and st.wait[z] == 0.0 and st.t_dep[z] == tz
        else:
            assert st.t_dep[z] == tm.next_green_from(tz) and st.wait[z] == st.t_dep[z] - tz
    assert np.array_equal(ctx.steps[k - 1].arr_green, [1 if tm.is_green(t) else 0 for t in ctx.t_axis])
    g = golden_npz("c1_short_s45_t50.npz")
    assert np.array_equal(ctx.terminal, g["J"][-1])


def test_signal_timing_python_modulo():
    tm = SignalTiming(cycle=60.0, offset=20.0, green_windows=((0.0, 30.0),))
    assert tm.local_time(-25.0) == 15.0
    assert tm.is_green(-25.0)
    assert not tm.is_green(50.0)
    assert tm.next_green_from(50.0) == 80.0
    with pytest.raises(ValueError):
        tm.next_green_from(25.0)
    with pytest.raises(RouteFormatError):
        SignalTiming(cycle=60.0, offset=0.0, green_windows=((10.0, 5.0),))


def test_route_loader_errors():
    doc = {"node_count": 3, "delta_d_m": 10.0, "v_min_mps": 0.0, "v_max_mps": 10.0, "accel_min_mps2": -3.0,
           "accel_max_mps2": 2.5, "traffic_lights": [{"node": 1, "signal": "x"}], "signals": {}}
    with pytest.raises(RouteFormatError, match="unknown signal"):
        load_route(doc)
    doc["signals"] = {"x": {"cycle_s": 60.0, "green_windows_s": [[0.0, 30.0]]}}
    route, spat = load_route(doc)
    assert route.node_kind(1) == 1 and route.node_count == 3
    doc["v_min_mps"] = [0.0, 1.0, 0.0]
    with pytest.raises(RouteFormatError, match="must be 0 at traffic-light"):
        load_route(doc)


def test_cost_to_go_interpolate_absorbs():
    vals = np.ones((3, 3, 3))
    vals[0, 0, 0] = PEN.j_inf
    tab = CostToGoTable(values=vals, v_axis=np.linspace(0, 2, 3), soc_axis=np.linspace(0, 1, 3),
                        t_axis=np.arange(3.0), j_inf=PEN.j_inf)
    assert tab.interpolate(0.5, 0.25, 0.5) == PEN.j_inf
    assert tab.interpolate(1.0, 0.5, 1.0) == 1.0
    assert tab.interpolate(-0.1, 0.5, 1.0) == PEN.j_inf
    for q in (0.0, 0.7, 1.9999999999999, 2.0, 2.0000001):
        assert locate_uniform(q, 0.0, 1.0, 3)[:4] == O.locate_uniform(q, 0.0, 1.0, 3)


def test_policy_action_decoding():
    P = np.full((1, 1, 2), -1, dtype=np.int32)
    P[0, 0, 1] = 7
    pol = PolicyTable(values=P, te_axis=np.array([0.0, 10.0, 20.0]), tb_axis=np.array([-1.0, 0.0, 1.0, 2.0, 3.0]))
    assert pol.action(0, 0, 0) is None
    assert pol.action(0, 0, 1) == (10.0, 1.0)


def test_snapshot_round_trip(tmp_path):
    g = golden_npz("c1_short_s45_t50.npz")
    J, P = g["J"], g["P"]
    res = SolveResult(s=45, horizon=20, t_start=50.0, backend="b200-fp64", cost_at_start=math.nan,
                      tables=[CostToGoTable(J[k], None, None, None, PEN.j_inf) for k in range(21)],
                      policies=[PolicyTable(P[k], None, None) for k in range(20)], wall_time_s=0.0)
    path = tmp_path / "t.bin"
    dump_tables(str(path), res)
    h, t0, J2, P2 = load_tables(str(path))
    assert h == 20 and t0 == 50.0
    assert all(np.array_equal(a, b) for a, b in zip(J2, J))
    assert all(np.array_equal(a, b) for a, b in zip(P2, P))
    path.write_bytes(b"NOTATBL0" + b"\0" * 64)
    with pytest.raises(ValueError):
        load_tables(str(path))


def test_terminal_seed_matches_oracle_convention():
    soc = np.linspace(0.3, 0.8, 26)
    base = np.zeros((3, 26))
    base[1, 4] = PEN.j_inf
    base[2, 5] = PEN.j_inf - 10.0
    t = terminal_seed(base, soc, PEN, 4)
    assert t.shape == (3, 26, 4)
    assert t[1, 4, 0] == PEN.j_inf and t[2, 5, 3] == PEN.j_inf
    assert t[0, 0, 2] == 1500.0 * (0.3 - 0.5) ** 2
