"""The drop-in shim inside the reference package itself.

The reference is imported from /root/reference (build container) or, on the
GPU box where that tree does not exist, from the unmodified copy installed
into baseline/_ref (`pip install --no-deps --target baseline/_ref`, DESIGN.md
§8; git-ignored, it travels with the snapshot).  With a device present the
reference's own EcoDrivingMPC / simulate_closed_loop / run_bench run with
backend="b200" through plugin.install() and are checked against the
reference's own CPU backends and golden output.
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
_CANDIDATES = ("/root/reference/pkg/src", str(ROOT / "baseline" / "_ref"))
REF = next((p for p in _CANDIDATES if os.path.isdir(os.path.join(p, "ecodrive"))), None)
pytestmark = pytest.mark.skipif(REF is None, reason="reference package not present (install it into baseline/_ref)")


@pytest.fixture(scope="module")
def ecodrive():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_eco")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import ecodrive as E
    from paper_2104_01284_b200 import plugin
    plugin.install()
    yield E
    plugin.uninstall()


def _device():
    from paper_2104_01284_b200 import _abi
    return _abi.lib().eco_device_count() > 0


def _short_ctx(rdp, H=2, grids=None):
    from ecodrive.fixtures import load_fixture_route, make_vehicle
    route, spat = load_fixture_route("short", seed=2)
    return rdp.build_context(make_vehicle(), route, spat, 45, 50.0,
                             grids=grids or rdp.GridSpec(n_v=4, n_soc=3, n_t=6),
                             penalty=rdp.PenaltyConfig(), gamma=0.5, horizon=H)


def test_reference_backends_still_forwarded(ecodrive):
    import ecodrive.dp as rdp
    ctx = _short_ctx(rdp)
    res = rdp.solve_horizon(ctx, backend="serial")
    assert res.backend == "serial" and len(res.tables) == 3
    with pytest.raises(ValueError):
        rdp.solve_horizon(ctx, backend="nope")


def test_b200_names_route_to_the_device_library(ecodrive):
    import ecodrive.dp as rdp
    import ecodrive.mpc as rmpc
    from paper_2104_01284_b200 import NativeLibraryError
    assert rmpc.solve_horizon is rdp.solve_horizon is ecodrive.solve_horizon
    ctx = _short_ctx(rdp)
    if not _device():
        with pytest.raises(NativeLibraryError, match="no CUDA device"):
            rdp.solve_horizon(ctx, backend="b200")
        return
    res = rdp.solve_horizon(ctx, backend="b200-fp64")
    ref = rdp.solve_horizon(ctx, backend="serial")
    assert isinstance(res, rdp.SolveResult) and res.backend == "b200-fp64"
    for a, b in zip(res.tables, ref.tables):
        assert np.array_equal(a.values, b.values)


@pytest.mark.gpu
def test_reference_solve_horizon_on_b200_c1(ecodrive):
    """C1 through the reference's own solve_horizon (backend="b200-fp64"):
    every level bitwise equal to the reference's serial backend."""
    import ecodrive.dp as rdp
    ctx = _short_ctx(rdp, H=20, grids=rdp.GridSpec(n_v=12, n_soc=8, n_t=40))
    res = rdp.solve_horizon(ctx, backend="b200-fp64")
    ref = rdp.solve_horizon(ctx, backend="parallel", workers=4)
    for a, b in zip(res.tables, ref.tables):
        assert np.array_equal(a.values, b.values)
    for a, b in zip(res.policies, ref.policies):
        assert np.array_equal(a.values, b.values)
    # backward_step (the per-stage plug-in point, dp.py:365-404) too
    J, P = rdp.backward_step(ctx, 19, ctx.terminal, backend="b200-fp64")
    assert np.array_equal(J, ref.tables[19].values) and np.array_equal(P, ref.policies[19].values)


@pytest.mark.gpu
def test_reference_closed_loop_on_b200(ecodrive):
    """The reference's own EcoDrivingMPC + simulate_closed_loop (host argmin,
    host plant, bitwise prediction check at every node, mpc.py:513-596) with
    backend="b200-fp64": the trajectory equals the golden one the reference
    produced with its parallel backend."""
    from conftest import golden_npz
    from ecodrive.dp import GridSpec, PenaltyConfig
    from ecodrive.fixtures import load_fixture_route, make_vehicle
    route, spat = load_fixture_route("short", seed=2)
    grids = GridSpec(n_v=12, n_soc=8, n_t=40, n_t_eng=8, n_t_bsg=10, horizon_steps=8)
    mpc = ecodrive.EcoDrivingMPC(make_vehicle(), gamma=0.5, grids=grids, penalty=PenaltyConfig(), horizon=8,
                                 backend="b200-fp64").fit(route, spat)
    traj = ecodrive.simulate_closed_loop(route, spat, mpc)
    g = golden_npz("loop_short_small.npz")
    rows = np.array([[float(getattr(st, f)) for f in ("s", "v", "soc", "t", "t_eng", "t_bsg", "brake_force", "gear",
                                                       "wait_s", "dt_move_s", "fuel_inc_g", "accel", "cost_to_go",
                                                       "fallback")] for st in traj.steps])
    assert rows.shape == g["rows"].shape
    assert np.array_equal(rows, g["rows"], equal_nan=True)      # fallback rows carry cost_to_go = nan
    assert traj.final_state.v == g["final"][0] and traj.final_state.t == g["final"][2]


@pytest.mark.gpu
def test_reference_run_bench_on_b200(ecodrive):
    """The reference's Table-I harness (bench.py:97-150) timing the device
    backends next to its own parallel backend on identical contexts."""
    from ecodrive.bench import run_bench
    from ecodrive.dp import GridSpec
    from ecodrive.fixtures import load_fixture_route, make_vehicle
    route, spat = load_fixture_route("urban", seed=0)
    rep = run_bench(make_vehicle(), route, spat, grids=GridSpec(), horizon=20,
                    backends=("b200", "b200-fp64", "parallel"), workers=8, reps=4, warmup=1)
    by = {r.backend: r for r in rep.results}
    assert set(by) == {"b200", "b200-fp64", "parallel"}
    for r in rep.results:
        assert r.times_ms.shape == (4,) and np.all(r.times_ms > 0)
    assert by["b200"].times_ms.mean() < by["parallel"].times_ms.mean()
    assert "b200" in rep.table()


@pytest.mark.gpu
def test_reference_compare_solves_b200_vs_serial(ecodrive):
    """Acceptance criterion 1's per-context diff (bench.py:283-304) with the
    device backend seated where the reference puts its parallel backend."""
    import ecodrive.dp as rdp
    ctx = _short_ctx(rdp, H=8, grids=rdp.GridSpec(n_v=12, n_soc=8, n_t=40, n_t_eng=8, n_t_bsg=10))
    a = rdp.solve_horizon(ctx, backend="serial")
    b = rdp.solve_horizon(ctx, backend="b200-fp64")
    assert max(float(np.max(np.abs(x.values - y.values))) for x, y in zip(a.tables, b.tables)) == 0.0
    assert sum(int(np.count_nonzero(x.values != y.values)) for x, y in zip(a.policies, b.policies)) == 0


@pytest.mark.gpu
def test_reference_perturb_ties_matches_b200(ecodrive):
    """perturb_ties (reverse_ties, _kernels.py:630-632): the device's
    highest-index tie rule reproduces the reference parallel backend's
    perturbed policies exactly, costs unchanged (test_parallel.py:174-179)."""
    import ecodrive.dp as rdp
    ctx = _short_ctx(rdp, H=20, grids=rdp.GridSpec(n_v=12, n_soc=8, n_t=40))
    ref = rdp.solve_horizon(ctx, backend="parallel", workers=4, perturb_ties=True)
    res = rdp.solve_horizon(ctx, backend="b200-fp64", perturb_ties=True)
    plain = rdp.solve_horizon(ctx, backend="b200-fp64")
    for a, b, c in zip(res.tables, ref.tables, plain.tables):
        assert np.array_equal(a.values, b.values) and np.array_equal(a.values, c.values)
    for a, b in zip(res.policies, ref.policies):
        assert np.array_equal(a.values, b.values)
