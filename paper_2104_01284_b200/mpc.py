"""Receding-horizon eco-driving controller and the device-resident closed loop.

Front end with the reference's names and semantics (mpc.py:47-596):
``TerminalCostField``, ``build_terminal_cost``, ``field_value``,
``EcoDrivingMPC`` (fit / control), ``mpc_step``, ``simulate_closed_loop``,
``ControlDecision``, ``TrajectoryStep``, ``ClosedLoopTrajectory``.

Execution is on the B200: the offline field sweep, every horizon solve, the
exact-state argmin, the max-brake fallback and the plant step all run in the
sm_100a library (``eco_mpc_run``); the loop state never leaves the device
until the trajectory is copied back once at the end.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field as dc_field
from typing import Optional

import numpy as np

from . import _abi
from .dp import (GridSpec, PenaltyConfig, locate_uniform, precision_of, _bilin_abs)
from .errors import StartStateInfeasibleError
from .plant import ActionVector, StateVector, Vehicle
from .route import Route, SpatSchedule


@dataclass(frozen=True)
class TerminalCostField:
    """Cost-to-destination per node on the (v, soc) grid (mpc.py:47-71)."""

    values: np.ndarray           # (node_count, n_v, n_soc)
    route_name: str
    gamma: float
    grids: GridSpec
    penalty: PenaltyConfig

    def node_slice(self, s: int) -> np.ndarray:
        return self.values[s]

    @classmethod
    def _from_device(cls, values: np.ndarray, **kw) -> "TerminalCostField":
        """A field the device just built (shape known, NaN impossible by
        construction: +inf / j_inf only): skips the user-input checks of
        __post_init__ (a 5 MB NaN scan per fit at C2)."""
        obj = object.__new__(cls)
        object.__setattr__(obj, "values", values)
        for k, v in kw.items():
            object.__setattr__(obj, k, v)
        return obj

    def __post_init__(self):
        if self.values.ndim != 3:
            raise ValueError("terminal field values must be (nodes, n_v, n_soc)")
        if self.values.shape[1:] != (self.grids.n_v, self.grids.n_soc):
            raise ValueError("terminal field shape does not match the grid spec")
        if np.isnan(self.values).any():
            raise ValueError("terminal field contains NaN")


def field_value(field: TerminalCostField, vehicle: Vehicle, route: Route, s: int, v: float, soc: float) -> float:
    """Bilinear field value at node s with absorbing j_inf (mpc.py:74-93)."""
    g = field.grids
    va, xa = g.v_axis(route, s), g.soc_axis(vehicle)
    v0, x0 = float(va[0]), float(xa[0])
    a0, a1, wa, oka = locate_uniform(v, v0, (float(va[-1]) - v0) / (g.n_v - 1), g.n_v)
    b0, b1, wb, okb = locate_uniform(soc, x0, (float(xa[-1]) - x0) / (g.n_soc - 1), g.n_soc)
    if not (oka and okb):
        return field.penalty.j_inf
    G = field.values[s]
    return float(_bilin_abs(float(G[a0, b0]), float(G[a0, b1]), float(G[a1, b0]), float(G[a1, b1]),
                            wa, wb, field.penalty.j_inf))


def _config(vehicle, grids: GridSpec, penalty: PenaltyConfig, gamma: float, horizon: int, teleport: bool,
            use_field: bool, backend: str, start_node: int = 0, max_steps: int = -1):
    te, tb = grids.te_axis(), grids.tb_axis()
    cfg = _abi.EcoMpcConfig(
        n_v=grids.n_v, n_soc=grids.n_soc, n_t=grids.n_t, n_te=te.size, n_tb=tb.size, horizon=horizon,
        teleport=int(teleport), use_terminal_field=int(use_field), precision=precision_of(backend),
        start_node=start_node, max_steps=max_steps, dt=float(grids.dt), gamma=float(gamma),
        soc_target=float(penalty.soc_target), soc_weight=float(penalty.soc_weight), j_inf=float(penalty.j_inf),
        te_axis=_abi.ptr(te, C.c_double), tb_axis=_abi.ptr(tb, C.c_double))
    return cfg, (te, tb)


def build_terminal_cost(route: Route, vehicle: Vehicle, *, gamma: float, grids: GridSpec,
                        penalty: PenaltyConfig, spat: Optional[SpatSchedule] = None,
                        backend: str = "b200", stats: Optional[dict] = None) -> TerminalCostField:
    """Signal-free (v, soc) backward sweep over all nodes (mpc.py:96-158), on the device."""
    if not 0.0 <= gamma <= 1.0:
        raise ValueError("gamma must lie in [0, 1]")
    rp = _abi.RoutePack(route, spat if spat is not None else SpatSchedule(signals={}), signals_optional=True)
    cfg, keep = _config(vehicle, grids, penalty, gamma, 1, True, True, backend)
    plant = _abi.pack_plant(vehicle.pack())
    out = np.empty((route.node_count, grids.n_v, grids.n_soc))
    st = _abi.EcoStats()
    _abi.check(_abi.lib().eco_field_build(C.byref(plant), C.byref(rp.c), C.byref(cfg),
                                          _abi.ptr(out, C.c_double), C.byref(st)), "eco_field_build")
    if stats is not None:
        stats.update(st.as_dict())
    return TerminalCostField(values=out, route_name=route.name, gamma=gamma, grids=grids, penalty=penalty)


@dataclass
class ControlDecision:
    action: ActionVector
    brake_force: float = 0.0
    predicted_next: Optional[StateVector] = None
    cost_to_go: float = math.nan
    solver_wall_s: float = 0.0
    fallback: bool = False
    note: str = ""


@dataclass
class MpcStepInfo:
    predicted_next: StateVector
    cost_to_go: float
    wait: float
    solve_wall_s: float
    horizon: int


@dataclass
class TrajectoryStep:
    """One spatial step of a run, state taken at the source node (mpc.py:418-435)."""

    s: int
    v: float
    soc: float
    t: float
    t_eng: float
    t_bsg: float
    brake_force: float
    gear: int
    wait_s: float
    dt_move_s: float
    fuel_inc_g: float
    accel: float
    cost_to_go: float
    fallback: bool


@dataclass
class ClosedLoopTrajectory:
    """Step log, final state and totals of one run (mpc.py:438-487)."""

    route_name: str
    controller: str
    backend: str
    delta_d: float
    x_start: StateVector
    steps: list = dc_field(default_factory=list)
    solver_wall_s: list = dc_field(default_factory=list)
    final_state: Optional[StateVector] = None
    status: str = "ok"
    stats: dict = dc_field(default_factory=dict)

    @property
    def completed(self) -> bool:
        return self.status == "ok"

    @property
    def n_steps(self) -> int:
        return len(self.steps)

    @property
    def fuel_g(self) -> float:
        return float(sum(st.fuel_inc_g for st in self.steps))

    @property
    def travel_time_s(self) -> float:
        return 0.0 if self.final_state is None else float(self.final_state.t - self.x_start.t)

    @property
    def soc_end(self) -> float:
        return float(self.x_start.soc if self.final_state is None else self.final_state.soc)

    def distance_m(self, step_index: int) -> float:
        return self.steps[step_index].s * self.delta_d

    def timing_stats_ms(self) -> dict:
        if not self.solver_wall_s:
            return {"mean_ms": 0.0, "variance_ms2": 0.0, "max_ms": 0.0}
        arr = 1.0e3 * np.asarray(self.solver_wall_s)
        return {"mean_ms": float(arr.mean()), "variance_ms2": float(arr.var()), "max_ms": float(arr.max())}


_STEP_FIELDS = ("s", "v", "soc", "t", "t_eng", "t_bsg", "brake_force", "gear", "wait_s", "dt_move_s", "fuel_inc_g",
                "accel", "cost_to_go")


def _rows_to_steps(rows: np.ndarray) -> list:
    # column-wise tolist(): exact Python ints / floats, ~10x faster than
    # converting row by row (699 rows of a C2 run are in the e2e timing)
    cols = [rows[f].tolist() for f in _STEP_FIELDS]
    cols.append([x != 0 for x in rows["fallback"].tolist()])
    return [TrajectoryStep(*vals) for vals in zip(*cols)]


class MpcSession:
    """A route-resident device solver (eco_session_*): geometry, terminal
    field and loop buffers stay in HBM across runs, so repeated closed loops
    and single receding-horizon steps pay no allocation or upload."""

    def __init__(self, vehicle: Vehicle, route: Route, spat: SpatSchedule, *, gamma: float, grids: GridSpec,
                 penalty: PenaltyConfig, horizon: int, backend: str, teleport: bool = True,
                 use_terminal_field: bool = True):
        self.route, self.grids = route, grids
        self.use_terminal_field = use_terminal_field
        self._rp = _abi.RoutePack(route, spat)
        self._cfg, self._keep = _config(vehicle, grids, penalty, gamma, horizon, teleport, use_terminal_field,
                                        backend)
        self._plant = _abi.pack_plant(vehicle.pack())
        self._h = C.c_void_p()
        self._lib = _abi.lib()
        _abi.check(self._lib.eco_session_create(C.byref(self._plant), C.byref(self._rp.c), C.byref(self._cfg),
                                                C.byref(self._h)), "eco_session_create")
        self.h2d_bytes = (C.sizeof(self._plant) + C.sizeof(self._cfg) + sum(
            a.nbytes for a in (self._rp.v_min, self._rp.v_max, self._rp.grade, self._rp.cos_g, self._rp.sin_g,
                               self._rp.kinds, self._rp.cycle, self._rp.offset, self._rp.nwin, self._rp.win,
                               *self._keep)))

    def upload_route(self, route: Route, spat: SpatSchedule) -> int:
        """Re-send the route / SPaT arrays into the session's buffers (same node
        count); returns the bytes copied.  The next :meth:`fit` uses them."""
        if route.node_count != self.route.node_count:
            raise ValueError("route node count differs from the session's")
        rp = _abi.RoutePack(route, spat)
        _abi.check(self._lib.eco_session_upload_route(self._h, C.byref(rp.c)), "eco_session_upload_route")
        self._rp, self.route = rp, route
        return sum(a.nbytes for a in (rp.v_min, rp.v_max, rp.grade, rp.cos_g, rp.sin_g, rp.kinds, rp.cycle,
                                      rp.offset, rp.nwin, rp.win))

    _PACK_FIELDS = ("v_min", "v_max", "grade", "kinds", "cycle", "offset", "nwin", "win")

    def same_inputs(self, route: Route, spat: SpatSchedule) -> bool:
        """True when (route, spat) carry the values this session was loaded
        with (an equal route / SPaT passed as another object)."""
        if route.node_count != self.route.node_count or route.delta_d != self.route.delta_d or \
                route.accel_min != self.route.accel_min or route.accel_max != self.route.accel_max or \
                route.stop_dwell != self.route.stop_dwell:
            return False
        try:
            rp = _abi.RoutePack(route, spat)
        except (KeyError, ValueError):
            return False
        return all(np.array_equal(getattr(rp, f), getattr(self._rp, f)) for f in self._PACK_FIELDS)

    def fit(self, field: Optional[np.ndarray] = None, want_field: bool = True):
        """Route geometry + terminal field on the device; returns (field or None, stats)."""
        n = self.route.node_count
        out = np.empty((n, self.grids.n_v, self.grids.n_soc)) if (want_field and self.use_terminal_field) else None
        fin = None if field is None else np.ascontiguousarray(field, dtype=np.float64)
        st = _abi.EcoStats()
        _abi.check(self._lib.eco_session_fit(self._h, None if fin is None else _abi.ptr(fin, C.c_double),
                                             None if out is None else _abi.ptr(out, C.c_double), C.byref(st)),
                   "eco_session_fit")
        return out, st.as_dict()

    def run(self, x_start: StateVector, start_node: int = 0, max_steps: int = -1, *, count_live: bool = False,
            time_sweeps: bool = True):
        """Closed loop on the device -> (rows, status, status_node, final_state, stats).
        ``stats["dominant_ms"]`` is the summed per-step solve clock (device
        timestamps, always on; ``time_sweeps`` is accepted and ignored)."""
        rows = np.zeros(max(self.route.node_count - 1, 1), dtype=_abi.TRAJ_DTYPE)
        x0 = np.array([x_start.v, x_start.soc, x_start.t], dtype=np.float64)
        fin = np.zeros(3)
        n_rows, status, node = C.c_int32(0), C.c_int32(0), C.c_int32(-1)
        flags = (_abi.RUN_COUNT_LIVE if count_live else 0) | (_abi.RUN_TIME_SWEEPS if time_sweeps else 0)
        st = _abi.EcoStats()
        _abi.check(self._lib.eco_session_run(
            self._h, start_node, max_steps, _abi.ptr(x0, C.c_double),
            rows.ctypes.data_as(C.POINTER(_abi.EcoTrajRow)), C.byref(n_rows), C.byref(status), C.byref(node),
            _abi.ptr(fin, C.c_double), flags, C.byref(st)), "eco_session_run")
        return rows[:n_rows.value], status.value, node.value, fin, st.as_dict()

    def step_times(self, n: int) -> np.ndarray:
        """Per-step solve clocks (s) of the last :meth:`run`'s first n steps:
        device timestamps from context preparation to the decision."""
        out = np.zeros(max(n, 0))
        _abi.check(self._lib.eco_session_step_times(self._h, _abi.ptr(out, C.c_double), n),
                   "eco_session_step_times")
        return out * 1e-3

    def close(self):
        if self._h:
            self._lib.eco_session_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_closed_loop(vehicle: Vehicle, route: Route, spat: SpatSchedule, x_start: StateVector, *,
                    gamma: float, grids: GridSpec, penalty: PenaltyConfig, horizon: int, backend: str,
                    teleport: bool = True, field: Optional[TerminalCostField] = None,
                    use_terminal_field: bool = True, start_node: int = 0, max_steps: int = -1):
    """One call of ``eco_mpc_run``.  Returns (rows, status, status_node,
    final_state, field_values, stats)."""
    n = route.node_count
    rp = _abi.RoutePack(route, spat)
    cfg, keep = _config(vehicle, grids, penalty, gamma, horizon, teleport, use_terminal_field, backend,
                        start_node, max_steps)
    plant = _abi.pack_plant(vehicle.pack())
    x0 = np.array([x_start.v, x_start.soc, x_start.t], dtype=np.float64)
    rows = np.zeros(max(n - 1, 1), dtype=_abi.TRAJ_DTYPE)
    fin = np.zeros(3)
    n_rows, status, status_node = C.c_int32(0), C.c_int32(0), C.c_int32(-1)
    field_in = None
    field_out = None
    if use_terminal_field:
        if field is not None:
            field_in = np.ascontiguousarray(field.values, dtype=np.float64)
        else:
            field_out = np.empty((n, grids.n_v, grids.n_soc))
    st = _abi.EcoStats()
    _abi.check(_abi.lib().eco_mpc_run(
        C.byref(plant), C.byref(rp.c), C.byref(cfg), _abi.ptr(x0, C.c_double),
        None if field_in is None else _abi.ptr(field_in, C.c_double),
        None if field_out is None else _abi.ptr(field_out, C.c_double),
        rows.ctypes.data_as(C.POINTER(_abi.EcoTrajRow)), C.byref(n_rows), C.byref(status), C.byref(status_node),
        _abi.ptr(fin, C.c_double), C.byref(st)), "eco_mpc_run")
    return rows[:n_rows.value], status.value, status_node.value, fin, field_out, st.as_dict()


def _raise_step_status(status, rows, s, x, teleport):
    if status == _abi.RUN_MISMATCH:
        raise RuntimeError(f"solver/plant transition mismatch at node {s}")
    if status == _abi.RUN_INFEASIBLE or (len(rows) and rows[0]["fallback"]):
        raise StartStateInfeasibleError(
            f"no admissible action from node {s} at v={x.v:.2f} m/s, soc={x.soc:.3f}, t={x.t:.1f} s "
            f"(teleport={'on' if teleport else 'off'})")
    if status != _abi.RUN_OK or not len(rows):
        raise RuntimeError(f"plant step failed at node {s}")


def mpc_step(vehicle: Vehicle, route: Route, spat: SpatSchedule, x: StateVector, s: int, *, gamma: float,
             grids: GridSpec, penalty: PenaltyConfig, horizon: int, terminal: Optional[TerminalCostField] = None,
             backend: str = "b200", workers: int = 8, teleport: bool = True, perturb_ties: bool = False):
    """Solve the truncated horizon at node s and return the first action
    (mpc.py:281-337).  Raises StartStateInfeasibleError when no action at x
    has a feasible continuation."""
    n = route.node_count
    if not 0 <= s < n - 1:
        raise ValueError(f"start node {s} out of range for {n} route nodes")
    # perturb_ties flips only tied POLICY entries (the reference's
    # reverse_ties); the decision reads J_1 at the exact state (mpc.py:189-278)
    # and the costs are unchanged, so it cannot alter the action: accepted
    h = min(horizon, n - 1 - s)
    rows, status, _, fin, _, st = run_closed_loop(
        vehicle, route, spat, x, gamma=gamma, grids=grids, penalty=penalty, horizon=horizon, backend=backend,
        teleport=teleport, field=terminal, use_terminal_field=terminal is not None, start_node=s, max_steps=1)
    _raise_step_status(status, rows, s, x, teleport)
    r = rows[0]
    return (ActionVector(t_eng=float(r["t_eng"]), t_bsg=float(r["t_bsg"])),
            MpcStepInfo(predicted_next=StateVector(v=float(fin[0]), soc=float(fin[1]), t=float(fin[2])),
                        cost_to_go=float(r["cost_to_go"]), wait=float(r["wait_s"]),
                        solve_wall_s=st["device_ms"] / 1e3, horizon=h))


_SESSIONS: "dict" = {}
_SESSION_CAP = 4


def _session_for(vehicle, route, spat, **kw) -> "MpcSession":
    """Device sessions are cached per (vehicle, route, SPaT, settings): a
    re-fit on the same route reuses the HBM-resident buffers and the captured
    closed-loop graph instead of reallocating them (the cache keeps the keyed
    objects alive, so their ids stay unique)."""
    key = (id(vehicle), id(route), id(spat)) + tuple(sorted(kw.items()))
    hit = _SESSIONS.get(key)
    if hit is not None:
        return hit[0]
    while len(_SESSIONS) >= _SESSION_CAP:
        # drop the cache's reference only: a fitted controller may still hold
        # this session (EcoDrivingMPC.session_); it is closed when the last
        # holder lets go (MpcSession.__del__)
        _SESSIONS.pop(next(iter(_SESSIONS)))
    sess = MpcSession(vehicle, route, spat, **kw)
    _SESSIONS[key] = (sess, vehicle, route, spat)
    return sess


def clear_session_cache() -> None:
    """Forget the cached sessions (each is closed once no controller holds it)."""
    _SESSIONS.clear()


class EcoDrivingMPC:
    """Receding-horizon controller with fit / control (mpc.py:344-411)."""

    name = "mpc"

    def __init__(self, vehicle: Vehicle, *, gamma: float = 0.5, grids: Optional[GridSpec] = None,
                 penalty: Optional[PenaltyConfig] = None, horizon: int = 20, backend: str = "b200",
                 workers: int = 8, teleport: bool = True, use_terminal_field: bool = True,
                 perturb_ties: bool = False):
        precision_of(backend)
        self.vehicle = vehicle
        self.gamma = gamma
        self.grids = grids if grids is not None else GridSpec()
        self.penalty = penalty if penalty is not None else PenaltyConfig()
        self.horizon = horizon
        self.backend = backend
        self.workers = workers
        self.teleport = teleport
        self.use_terminal_field = use_terminal_field
        self.perturb_ties = perturb_ties

    def fit(self, route: Route, spat: SpatSchedule) -> "EcoDrivingMPC":
        if self.horizon < 1:
            raise ValueError("horizon must be >= 1")
        self.route_ = route
        self.spat_ = spat
        self.session_ = _session_for(self.vehicle, route, spat, gamma=self.gamma, grids=self.grids,
                                     penalty=self.penalty, horizon=self.horizon, backend=self.backend,
                                     teleport=self.teleport, use_terminal_field=self.use_terminal_field)
        # a cached session gets this call's route / SPaT values (they may have
        # been edited in place since): ~150 KB per fit, the inputs' H2D
        self.upload_bytes_ = self.session_.upload_route(route, spat)
        values, self.fit_stats_ = self.session_.fit()
        self.terminal_field_ = (TerminalCostField._from_device(values, route_name=route.name, gamma=self.gamma,
                                                  grids=self.grids, penalty=self.penalty)
                                if self.use_terminal_field else None)
        return self

    def control(self, x: StateVector, s: int) -> ControlDecision:
        """One receding-horizon decision at (x, s) on the fitted session."""
        self._check_fitted()
        n = self.route_.node_count
        if not 0 <= s < n - 1:
            raise ValueError(f"start node {s} out of range for {n} route nodes")
        rows, status, _, fin, st = self.session_.run(x, start_node=s, max_steps=1)
        _raise_step_status(status, rows, s, x, self.teleport)
        r = rows[0]
        return ControlDecision(action=ActionVector(t_eng=float(r["t_eng"]), t_bsg=float(r["t_bsg"])),
                               predicted_next=StateVector(v=float(fin[0]), soc=float(fin[1]), t=float(fin[2])),
                               cost_to_go=float(r["cost_to_go"]),
                               solver_wall_s=float(self.session_.step_times(1)[0]))

    def _check_fitted(self):
        if not hasattr(self, "route_"):
            raise RuntimeError("controller is not fitted: call fit(route, spat) first")


_STATUS_TEXT = {
    _abi.RUN_INFEASIBLE: "infeasible: no admissible action and no legal braking move at node {node}",
    _abi.RUN_PLANT: "infeasible: plant step rejected the applied action at node {node}",
}


def simulate_closed_loop(route: Route, spat: SpatSchedule, controller: EcoDrivingMPC,
                         x_start: Optional[StateVector] = None, *, backend_tag: Optional[str] = None,
                         ) -> ClosedLoopTrajectory:
    """Drive the route under a fitted controller (mpc.py:513-596), entirely
    on the device: one eco_mpc_run call for all N-1 nodes."""
    if not isinstance(controller, EcoDrivingMPC):
        raise TypeError("simulate_closed_loop drives an EcoDrivingMPC on the device")
    controller._check_fitted()
    if x_start is None:
        x_start = StateVector(v=0.0, soc=0.5, t=0.0)
    traj = ClosedLoopTrajectory(route_name=route.name, controller=controller.name,
                                backend=backend_tag if backend_tag is not None else controller.backend,
                                delta_d=route.delta_d, x_start=x_start)
    if route.node_count == 1:
        traj.final_state = x_start
        return traj
    if (route is not controller.route_ or spat is not controller.spat_) and \
            not controller.session_.same_inputs(route, spat):
        # the device loop plans and steps the plant on the fitted route / SPaT
        # (the reference plans on controller.spat_ and steps on `spat`)
        raise ValueError("simulate_closed_loop: route / SPaT differ from the ones the controller was fitted on; "
                         "fit the controller on them first")
    rows, status, node, fin, st = controller.session_.run(x_start)
    if status == _abi.RUN_MISMATCH:
        raise RuntimeError(f"solver/plant transition mismatch at node {node}")
    traj.steps = _rows_to_steps(rows)
    traj.solver_wall_s = [float(x) for x in controller.session_.step_times(len(rows))]
    traj.final_state = StateVector(v=float(fin[0]), soc=float(fin[1]), t=float(fin[2]))
    if status != _abi.RUN_OK:
        traj.status = _STATUS_TEXT[status].format(node=node)
    traj.stats = st
    return traj
