"""Batch of independent receding-horizon solves on one route (C4).

The reference times many independent solves with ``run_bench``
(``pkg/src/ecodrive/bench.py:97-150``): one ``build_context`` (dp.py:255-341)
plus one ``solve_horizon`` (dp.py:425-475) per (start node, start time) of
``bench_schedule`` (bench.py:76-94), each with its own SPaT.  Scenarios on
the same road differ only in their clock and signal phasing, so the transition
geometry is shared: :class:`BatchSolver` keeps it resident on the device and
runs stage k of every scenario in one launch (``eco_batch_*`` in
``include/eco_b200.h``).  Per scenario the results are exactly those of
``solve_horizon(build_context(...))`` — bitwise in the fp64 build.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _abi
from .dp import GridSpec, PenaltyConfig, precision_of
from .mpc import _config
from .plant import Vehicle
from .route import Route, SpatSchedule


@dataclass
class BatchResult:
    """Start-node tables of every scenario (``None`` when not requested)."""

    J0: Optional[np.ndarray]          # (B, n_v, n_soc, n_t) f64, infeasible = j_inf
    P0: Optional[np.ndarray]          # (B, n_v, n_soc, n_t) int32 flat action, -1 infeasible
    horizons: np.ndarray              # (B,) horizon of each scenario (clipped at the route end)
    stats: dict = field(default_factory=dict)


class BatchSolver:
    """Route-resident batch solver.  ``solve`` may be called repeatedly with
    different scenario sets; the geometry is built on the first call."""

    def __init__(self, vehicle: Vehicle, route: Route, *, grids: Optional[GridSpec] = None,
                 penalty: Optional[PenaltyConfig] = None, gamma: float = 0.5, horizon: int = 20,
                 teleport: bool = True, terminal_field: bool = False, backend: str = "b200"):
        if not 0.0 <= gamma <= 1.0:
            raise ValueError("gamma must lie in [0, 1]")
        if horizon < 1:
            raise ValueError("horizon must be >= 1")
        precision_of(backend)
        self.route = route
        self.grids = grids if grids is not None else GridSpec()
        self.penalty = penalty if penalty is not None else PenaltyConfig()
        self.horizon = horizon
        self._rp = _abi.RoutePack(route, SpatSchedule(signals={}), signals_optional=True)
        self._cfg, self._keep = _config(vehicle, self.grids, self.penalty, gamma, horizon, teleport,
                                        terminal_field, backend)
        self._plant = _abi.pack_plant(vehicle.pack())
        self._lib = _abi.lib()
        self._h = C.c_void_p()
        _abi.check(self._lib.eco_batch_create(C.byref(self._plant), C.byref(self._rp.c), C.byref(self._cfg),
                                              C.byref(self._h)), "eco_batch_create")

    def horizons(self, starts: np.ndarray) -> np.ndarray:
        n = self.route.node_count
        return np.minimum(self.horizon, n - 1 - np.asarray(starts, dtype=np.int64)).astype(np.int32)

    def solve(self, spats: Sequence[SpatSchedule], schedule: Sequence, *, return_tables: bool = True,
              count_live: bool = False, timings: Optional[np.ndarray] = None) -> BatchResult:
        """Solve scenario i = (schedule[i] = (start node, start time), spats[i]).
        ``timings`` may carry a prebuilt :func:`_abi.signal_timings` array."""
        B = len(schedule)
        starts = np.ascontiguousarray([int(s) for s, _ in schedule], dtype=np.int32)
        clocks = np.ascontiguousarray([float(t) for _, t in schedule], dtype=np.float64)
        if timings is None:
            if len(spats) != B:
                raise ValueError("one SpatSchedule per scenario is required")
            timings = _abi.signal_timings(self.route, spats)
        timings = np.ascontiguousarray(timings, dtype=_abi.SIGNAL_TIMING_DTYPE)
        if timings.shape[0] != B:
            raise ValueError("signal timings do not match the schedule")
        g = self.grids
        shape = (B, g.n_v, g.n_soc, g.n_t)
        J0 = np.empty(shape) if return_tables else None
        P0 = np.empty(shape, dtype=np.int32) if return_tables else None
        st = _abi.EcoStats()
        _abi.check(self._lib.eco_batch_solve(
            self._h, B, timings.ctypes.data_as(C.c_void_p), _abi.ptr(starts, C.c_int32),
            _abi.ptr(clocks, C.c_double), None if J0 is None else _abi.ptr(J0, C.c_double),
            None if P0 is None else _abi.ptr(P0, C.c_int32), _abi.RUN_COUNT_LIVE if count_live else 0,
            C.byref(st)), "eco_batch_solve")
        stats = st.as_dict()
        stats["h2d_bytes"] = timings.nbytes + starts.nbytes + clocks.nbytes
        stats["d2h_bytes"] = 0 if J0 is None else J0.nbytes + P0.nbytes
        return BatchResult(J0=J0, P0=P0, horizons=self.horizons(starts), stats=stats)

    def close(self):
        if self._h:
            self._lib.eco_batch_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_batch(vehicle: Vehicle, route: Route, spats: Sequence[SpatSchedule], schedule: Sequence, **kw) -> BatchResult:
    """One-shot :class:`BatchSolver` (keyword arguments as its constructor,
    plus ``return_tables`` / ``count_live`` for ``solve``)."""
    solve_kw = {k: kw.pop(k) for k in ("return_tables", "count_live") if k in kw}
    with BatchSolver(vehicle, route, **kw) as bs:
        return bs.solve(spats, schedule, **solve_kw)


def shard(n_items: int, rank: int, world: int) -> range:
    """Contiguous block of scenarios owned by ``rank`` (C4 shards
    with no exchange; the first n % world ranks take one extra)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank / world size")
    q, r = divmod(n_items, world)
    lo = rank * q + min(rank, r)
    return range(lo, lo + q + (1 if rank < r else 0))


__all__ = ["BatchSolver", "BatchResult", "solve_batch", "shard"]
