"""Timing / comparison harness (``harness.py``, mirroring the reference's
bench.py).  CPU tests cover the report formatting and argument checks (with a
host callable standing in for a backend); GPU tests are the reference's
acceptance criteria 1 and 3 (tests/test_acceptance.py:115-200) restated for
the device backends, with the CPU oracle in the reference's "serial" seat."""

from types import SimpleNamespace

import numpy as np
import pytest

from oracle import oracle as O
from paper_2104_01284_b200 import GridSpec, PenaltyConfig, build_context
from paper_2104_01284_b200.harness import (BenchReport, BenchResult, DiffReport, StepDiff, _diff_tables,
                                           compare_solves, diff_backends_run, run_bench)

PEN = PenaltyConfig()
# the reference's reduced step-locked grid (test_acceptance.py:48-55)
DIFF_GRID = GridSpec(n_v=20, n_soc=14, n_t=40, n_t_eng=16, n_t_bsg=20)


def oracle_solver(ctx):
    """The CPU restatement as a backend callable (test infrastructure only)."""
    J, P = O.solve_context(ctx, parallel=True)
    return SimpleNamespace(tables=[SimpleNamespace(values=j) for j in J],
                           policies=[SimpleNamespace(values=p) for p in P])


oracle_solver.__name__ = "oracle"


# ----------------------------------------------------------------------- CPU

def _report():
    rs = [BenchResult("b200", 1, 3, 1, np.array([1.0, 2.0, 3.0])),
          BenchResult("oracle", 1, 3, 1, np.array([10.0, 20.0, 30.0]))]
    return BenchReport(results=rs, machine={"platform": "p", "cpu_count": 4, "device": "d", "python": "3"},
                       grids=GridSpec(), horizon=20, seed=0)


def test_bench_report_table_and_csv(tmp_path):
    rep = _report()
    assert rep.result("oracle").mean_ms == 20.0 and rep.result("b200").max_ms == 3.0
    with pytest.raises(KeyError):
        rep.result("serial")
    txt = rep.table()
    assert "speedup (b200 mean / oracle mean): 0.10x" in txt
    assert "solve size: (35 x 26 x 40) states, (23 x 30) actions, 20 steps" in txt
    rep.write_csv(tmp_path / "t.csv")
    lines = (tmp_path / "t.csv").read_text().splitlines()
    assert lines[0] == "backend,workers,rep,wall_ms" and len(lines) == 7 and lines[4] == "oracle,1,0,10.0"


def test_run_bench_argument_checks(vehicle, short_route):
    route, spat = short_route
    with pytest.raises(ValueError):
        run_bench(vehicle, route, spat, reps=0)
    with pytest.raises(ValueError):
        run_bench(vehicle, route, spat, warmup=-1)
    with pytest.raises(ValueError):
        run_bench(vehicle, route, spat, horizon=route.node_count, reps=1)


def test_run_bench_times_a_callable(vehicle, short_route):
    route, spat = short_route
    seen = []

    def probe(ctx):
        seen.append((ctx.s, ctx.t_start))

    probe.__name__ = "probe"
    rep = run_bench(vehicle, route, spat, grids=GridSpec(n_v=6, n_soc=5, n_t=8), horizon=4, backends=[probe],
                    reps=3, warmup=2, seed=5)
    assert len(seen) == 5 and rep.result("probe").times_ms.shape == (3,)


def test_diff_report_table_and_flags():
    rep = DiffReport(route_name="r", backends=("a", "b"))
    rep.steps = [StepDiff(s, 5, 0.0, 0) for s in range(6)]
    assert rep.identical and "(4 matching steps omitted)" in rep.table()
    rep.steps[3] = StepDiff(3, 5, 1e-9, 2)
    assert not rep.identical and rep.max_abs_dj == 1e-9 and rep.policy_mismatches == 2
    assert "    3       5   1.000000e-09" in rep.table()
    rep.steps[3] = StepDiff(3, 5, 0.0, 0)
    rep.status = "infeasible at node 4"
    assert not rep.identical


def test_diff_tables_counts():
    a = SimpleNamespace(tables=[SimpleNamespace(values=np.zeros((2, 2)))] * 2,
                        policies=[SimpleNamespace(values=np.zeros((2, 2), np.int32))])
    b = SimpleNamespace(tables=[SimpleNamespace(values=np.array([[0.0, 0.5], [0.0, -2.0]]))] * 2,
                        policies=[SimpleNamespace(values=np.array([[0, 1], [1, 0]], np.int32))])
    d = _diff_tables(a, b, 3, 2)
    assert (d.s, d.horizon, d.max_abs_dj, d.policy_mismatches) == (3, 2, 2.0, 2)


# ----------------------------------------------------------------------- GPU

@pytest.mark.gpu
def test_criterion_1_full_solve_equal_to_oracle(vehicle, urban_route):
    route, spat = urban_route
    ctx = build_context(vehicle, route, spat, 120, 37.0, grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20)
    d = compare_solves(ctx, a=oracle_solver, b="b200-fp64")
    assert d.max_abs_dj == 0.0 and d.policy_mismatches == 0, d


@pytest.mark.gpu
def test_criterion_1_step_locked_urban_loop(vehicle, urban_route):
    """Every receding-horizon context along the urban route: device fp64 vs
    the oracle, bit for bit, the plant advancing on the device controller."""
    route, spat = urban_route
    rep = diff_backends_run(vehicle, route, spat, a="b200-fp64", b=oracle_solver, grids=DIFF_GRID, horizon=20)
    assert rep.status == "ok" and len(rep.steps) == route.node_count - 1, rep.table()
    assert rep.identical, rep.table()


@pytest.mark.gpu
def test_step_locked_fp32_vs_fp64(vehicle, short_route):
    route, spat = short_route
    rep = diff_backends_run(vehicle, route, spat, a="b200-fp64", b="b200", grids=DIFF_GRID, horizon=20)
    assert rep.status == "ok" and len(rep.steps) == route.node_count - 1, rep.table()
    same = diff_backends_run(vehicle, route, spat, a="b200-fp64", b="b200-fp64", grids=DIFF_GRID, horizon=20)
    assert same.identical, same.table()


@pytest.mark.gpu
def test_criterion_3_solver_time(vehicle, urban_route):
    """The reference's solver-time gate (mean at most half the serial mean,
    variance no larger) with the device in the parallel seat."""
    route, spat = urban_route
    rep = run_bench(vehicle, route, spat, grids=GridSpec(), horizon=20, backends=[oracle_solver, "b200"],
                    reps=10, warmup=3, seed=0)
    print("\n" + rep.table())
    cpu, dev = rep.result("oracle"), rep.result("b200")
    assert dev.mean_ms <= 0.5 * cpu.mean_ms and dev.variance_ms2 <= cpu.variance_ms2, rep.table()


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not __import__("os").path.isdir(REF_SRC), reason="reference sources not present")
def test_reference_solver_accepts_our_contexts(vehicle, short_route):
    """The reference's own solve_horizon as a harness backend (build container
    only): it consumes this package's contexts and agrees with the oracle."""
    import sys
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import ecodrive.dp as RD

    def reference_serial(ctx):
        return RD.solve_horizon(ctx, None, backend="serial")

    route, spat = short_route
    ctx = build_context(vehicle, route, spat, 45, 50.0, grids=GridSpec(n_v=12, n_soc=8, n_t=40), penalty=PEN,
                        gamma=0.5, horizon=5)
    d = compare_solves(ctx, a=reference_serial, b=oracle_solver)
    assert d.max_abs_dj == 0.0 and d.policy_mismatches == 0
