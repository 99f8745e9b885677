"""The reference's timing / comparison harness for the device backends.

Mirrors ``pkg/src/ecodrive/bench.py``: ``run_bench`` (Table-I style timing of
full-horizon solves over ``bench_schedule``, bench.py:97-150), its
``BenchReport`` (table / CSV, bench.py:153-217), ``compare_solves`` (every
table level of one context from two backends, bench.py:296-304) and
``diff_backends_run`` (a step-locked closed loop comparing two backends at
every node, bench.py:307-384).  The reference hard-codes its CPU pair
(serial / parallel); here the pair is any two backend names of this package,
or callables ``ctx -> SolveResult`` (e.g. the reference's own
``ecodrive.solve_horizon`` through :mod:`plugin`).
"""

from __future__ import annotations

import csv
import os
import platform
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Optional, Sequence, Union

import numpy as np

from . import _abi
from .dp import GridSpec, PenaltyConfig, build_context, solve_horizon
from .fixtures import bench_schedule
from .mpc import EcoDrivingMPC
from .plant import StateVector, Vehicle
from .route import Route, SpatSchedule

Solver = Union[str, Callable]


def _solver(b: Solver) -> Callable:
    if callable(b):
        return b
    return lambda ctx: solve_horizon(ctx, backend=b)


def _name(b: Solver) -> str:
    return b if isinstance(b, str) else getattr(b, "__name__", "custom")


def machine_info() -> dict:
    import torch
    dev = torch.cuda.get_device_name(0) if torch.cuda.is_available() else "none"
    return {"platform": platform.platform(), "machine": platform.machine(), "cpu_count": os.cpu_count(),
            "python": platform.python_version(), "numpy": np.__version__, "device": dev}


@dataclass
class BenchResult:
    """Wall times of the timed repetitions of one backend (bench.py:55-75)."""

    backend: str
    workers: int
    reps: int
    warmup: int
    times_ms: np.ndarray

    @property
    def mean_ms(self) -> float:
        return float(np.mean(self.times_ms))

    @property
    def variance_ms2(self) -> float:
        return float(np.var(self.times_ms))

    @property
    def max_ms(self) -> float:
        return float(np.max(self.times_ms))


@dataclass
class BenchReport:
    results: list
    machine: dict
    grids: GridSpec
    horizon: int
    seed: int

    def result(self, backend: str) -> BenchResult:
        for r in self.results:
            if r.backend == backend:
                return r
        raise KeyError(backend)

    def table(self) -> str:
        head = f"{'backend':<10} {'workers':>7} {'reps':>5} {'mean (ms)':>12} {'variance (ms^2)':>16} {'max (ms)':>12}"
        rows = [head, "-" * len(head)]
        for r in self.results:
            rows.append(f"{r.backend:<10} {r.workers:>7d} {r.reps:>5d} {r.mean_ms:>12.3f} "
                        f"{r.variance_ms2:>16.3f} {r.max_ms:>12.3f}")
        if len(self.results) >= 2:
            base = self.results[0]
            rows.append("-" * len(head))
            for r in self.results[1:]:
                rows.append(f"speedup ({base.backend} mean / {r.backend} mean): {base.mean_ms / r.mean_ms:.2f}x")
                if base.variance_ms2 > 0.0:
                    rows.append(f"variance ratio ({r.backend} / {base.backend}): "
                                f"{r.variance_ms2 / base.variance_ms2:.3f}")
        g = self.grids
        rows += ["-" * len(head),
                 f"solve size: ({g.n_v} x {g.n_soc} x {g.n_t}) states, ({g.n_t_eng} x {g.n_t_bsg}) actions, "
                 f"{self.horizon} steps",
                 f"machine: {self.machine['platform']}, {self.machine['cpu_count']} cpu, "
                 f"device {self.machine['device']}, python {self.machine['python']}"]
        return "\n".join(rows)

    def write_csv(self, path: Union[str, Path]) -> None:
        with Path(path).open("w", newline="") as fh:
            out = csv.writer(fh)
            out.writerow(["backend", "workers", "rep", "wall_ms"])
            for r in self.results:
                for i, ms in enumerate(r.times_ms):
                    out.writerow([r.backend, r.workers, i, repr(float(ms))])


def run_bench(vehicle: Vehicle, route: Route, spat: SpatSchedule, *, gamma: float = 0.5,
              grids: Optional[GridSpec] = None, penalty: Optional[PenaltyConfig] = None, horizon: int = 20,
              backends: Sequence[Solver] = ("b200",), reps: int = 30, warmup: int = 5,
              seed: int = 0) -> BenchReport:
    """Wall time of ``reps`` full-horizon solves per backend on one shared
    schedule of precomputed contexts; the first ``warmup`` solves run on
    extra schedule entries and are not timed (bench.py:97-150)."""
    if reps < 1:
        raise ValueError("reps must be >= 1")
    if warmup < 0:
        raise ValueError("warmup must be >= 0")
    grids = grids if grids is not None else GridSpec()
    penalty = penalty if penalty is not None else PenaltyConfig()
    schedule = bench_schedule(route, horizon, warmup + reps, seed)
    contexts = [build_context(vehicle, route, spat, s, t, grids=grids, penalty=penalty, gamma=gamma,
                              horizon=horizon) for s, t in schedule]
    results = []
    for b in backends:
        solve = _solver(b)
        times = np.empty(reps)
        for i, ctx in enumerate(contexts):
            t0 = time.perf_counter()
            solve(ctx)
            wall = time.perf_counter() - t0
            if i >= warmup:
                times[i - warmup] = wall * 1.0e3
        results.append(BenchResult(backend=_name(b), workers=1, reps=reps, warmup=warmup, times_ms=times))
    return BenchReport(results=results, machine=machine_info(), grids=grids, horizon=horizon, seed=seed)


@dataclass
class StepDiff:
    """Table comparison at one node (bench.py:223-229)."""

    s: int
    horizon: int
    max_abs_dj: float
    policy_mismatches: int


@dataclass
class DiffReport:
    route_name: str
    backends: tuple
    steps: list = field(default_factory=list)
    status: str = "ok"
    fallback_steps: int = 0

    @property
    def max_abs_dj(self) -> float:
        return max((d.max_abs_dj for d in self.steps), default=0.0)

    @property
    def policy_mismatches(self) -> int:
        return sum(d.policy_mismatches for d in self.steps)

    @property
    def identical(self) -> bool:
        return self.status == "ok" and self.max_abs_dj == 0.0 and self.policy_mismatches == 0

    def table(self) -> str:
        head = f"{'node':>5} {'horizon':>7} {'max|dJ|':>14} {'policy mismatches':>18}"
        rows = [f"route: {self.route_name}  backends: {self.backends[0]} vs {self.backends[1]}", head,
                "-" * len(head)]
        flagged = [d for d in self.steps if d.max_abs_dj != 0.0 or d.policy_mismatches != 0]
        for d in (flagged if flagged else self.steps[:1] + self.steps[-1:]):
            rows.append(f"{d.s:>5d} {d.horizon:>7d} {d.max_abs_dj:>14.6e} {d.policy_mismatches:>18d}")
        if not flagged and len(self.steps) > 2:
            rows.insert(4, f"{'...':>5} ({len(self.steps) - 2} matching steps omitted)")
        rows += ["-" * len(head),
                 f"steps compared: {len(self.steps)}  max|dJ| overall: {self.max_abs_dj:.6e}  "
                 f"policy mismatches total: {self.policy_mismatches}  fallback steps: {self.fallback_steps}  "
                 f"status: {self.status}"]
        return "\n".join(rows)


def _diff_tables(res_a, res_b, s: int, h: int) -> StepDiff:
    max_dj = 0.0
    for ta, tb in zip(res_a.tables, res_b.tables):
        max_dj = max(max_dj, float(np.max(np.abs(ta.values - tb.values))))
    mism = sum(int(np.count_nonzero(pa.values != pb.values)) for pa, pb in zip(res_a.policies, res_b.policies))
    return StepDiff(s=s, horizon=h, max_abs_dj=max_dj, policy_mismatches=mism)


def compare_solves(ctx, a: Solver = "b200-fp64", b: Solver = "b200") -> StepDiff:
    """Every J / P level of one context from two backends (bench.py:296-304)."""
    return _diff_tables(_solver(a)(ctx), _solver(b)(ctx), ctx.s, ctx.horizon)


def diff_backends_run(vehicle: Vehicle, route: Route, spat: SpatSchedule, *, a: str = "b200-fp64",
                      b: Solver = "b200", gamma: float = 0.5, grids: Optional[GridSpec] = None,
                      penalty: Optional[PenaltyConfig] = None, horizon: int = 20, teleport: bool = True,
                      use_terminal_field: bool = True, x_start: Optional[StateVector] = None) -> DiffReport:
    """Step-locked closed loop (bench.py:307-384): at every node both backends
    solve the same context and all levels are compared; the plant advances on
    backend ``a``'s decision (its device controller, fallback included), so
    no divergence can accumulate."""
    grids = grids if grids is not None else GridSpec()
    penalty = penalty if penalty is not None else PenaltyConfig()
    x = x_start if x_start is not None else StateVector(v=0.0, soc=0.5, t=0.0)
    ctl = EcoDrivingMPC(vehicle, gamma=gamma, grids=grids, penalty=penalty, horizon=horizon, backend=a,
                        teleport=teleport, use_terminal_field=use_terminal_field).fit(route, spat)
    terminal = ctl.terminal_field_
    report = DiffReport(route_name=route.name, backends=(_name(a), _name(b)))
    solve_b = _solver(b)
    n = route.node_count
    for s in range(n - 1):
        h = min(horizon, n - 1 - s)
        ctx = build_context(vehicle, route, spat, s, x.t, grids=grids, penalty=penalty, gamma=gamma, horizon=h,
                            teleport=teleport,
                            terminal_field=None if terminal is None else terminal.node_slice(s + h))
        report.steps.append(_diff_tables(solve_horizon(ctx, backend=a), solve_b(ctx), s, h))
        # one device step of backend a's controller: its pick at x, or the
        # friction-only maximum-braking fallback, then the plant (mpc.py:513-596)
        rows, status, _, fin, _ = ctl.session_.run(x, start_node=s, max_steps=1)
        if status == _abi.RUN_MISMATCH:
            report.status = f"solver/plant mismatch at node {s}"
            break
        if status != _abi.RUN_OK or not len(rows):
            report.status = f"infeasible at node {s}"
            break
        report.fallback_steps += int(rows[0]["fallback"])
        x = StateVector(v=float(fin[0]), soc=float(fin[1]), t=float(fin[2]))
    return report


__all__ = ["BenchResult", "BenchReport", "run_bench", "StepDiff", "DiffReport", "compare_solves",
           "diff_backends_run", "machine_info"]
