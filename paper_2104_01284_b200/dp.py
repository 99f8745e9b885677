"""Receding-horizon (v, SoC, t) dynamic program — the solver front end.

Same entry points, types and error behaviour as the reference's
``ecodrive.dp`` (dp.py:34-610): ``GridSpec``, ``PenaltyConfig``,
``build_context``, ``backward_step``, ``solve_horizon``, ``SolveResult``,
``CostToGoTable``, ``PolicyTable`` and the table-driven toy instances.  The
backend string selects the device precision instead of a CPU code path:

* ``"b200"``       — sm_100a kernels, transition geometry in f64, value
  gather / argmin in f32 (production);
* ``"b200-fp64"``  — the same kernels with an f64 value path and unfused
  arithmetic, bitwise equal to the reference's serial sweep.

Any other name raises ``ValueError`` exactly like dp.py:402-403.  There is no
CPU fallback: a missing or broken library raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
import struct
import time
from dataclasses import dataclass, field as dc_field
from typing import Optional, Sequence

import numpy as np

from . import _abi
from .errors import StartStateInfeasibleError
from .plant import PlantPack, StateVector, Vehicle
from .route import NODE_SIGNAL, NODE_STOP, Route, SpatSchedule

DEFAULT_J_INF = 1.0e6
BACKENDS = {"b200": _abi.FP32, "b200-fp64": _abi.FP64}
WEIGHT_SNAP = 1e-12


def precision_of(backend: str) -> int:
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend: {backend!r}")
    return BACKENDS[backend]


# ------------------------------------------------------------------- grids

@dataclass(frozen=True)
class GridSpec:
    """State / action resolution of a solve (dp.py:41-83)."""

    n_v: int = 35
    n_soc: int = 26
    n_t: int = 40
    n_t_eng: int = 23
    n_t_bsg: int = 30
    dt: float = 2.0
    horizon_steps: int = 20
    t_eng_lo: float = -40.0
    t_eng_hi: float = 180.0
    t_bsg_lo: float = -56.0
    t_bsg_hi: float = 60.0

    def __post_init__(self):
        for name in ("n_v", "n_soc", "n_t", "n_t_eng", "n_t_bsg", "horizon_steps"):
            if getattr(self, name) < 2:
                raise ValueError(f"{name} must be >= 2")
        if self.dt <= 0:
            raise ValueError("dt must be positive")

    @property
    def horizon_time(self) -> float:
        return self.dt * self.n_t

    def v_axis(self, route: Route, node: int) -> np.ndarray:
        return np.linspace(route.v_min[node], route.v_max[node], self.n_v)

    def soc_axis(self, vehicle: Vehicle) -> np.ndarray:
        return np.linspace(vehicle.battery.soc_min, vehicle.battery.soc_max, self.n_soc)

    def t_axis(self, t_start: float) -> np.ndarray:
        return self.dt * math.floor(t_start / self.dt) + self.dt * np.arange(self.n_t)

    def te_axis(self) -> np.ndarray:
        return np.linspace(self.t_eng_lo, self.t_eng_hi, self.n_t_eng)

    def tb_axis(self) -> np.ndarray:
        return np.linspace(self.t_bsg_lo, self.t_bsg_hi, self.n_t_bsg)


@dataclass(frozen=True)
class PenaltyConfig:
    """Terminal SoC penalty and the absorbing infeasibility cost (dp.py:86-98)."""

    soc_target: float = 0.5
    soc_weight: float = 1500.0
    j_inf: float = DEFAULT_J_INF

    def __post_init__(self):
        if self.soc_weight < 0:
            raise ValueError("soc_weight must be non-negative")
        if self.j_inf <= 0:
            raise ValueError("j_inf must be positive")


# ------------------------------------------------------------ host lookups

def locate_uniform(x: float, x0: float, dx: float, n: int):
    """Cell (lo, hi, w, ok) on a uniform axis with node snapping (K:284-306)."""
    f = (x - x0) / dx
    i = math.floor(f)
    w = f - i
    if w < WEIGHT_SNAP:
        w = 0.0
    elif w > 1.0 - WEIGHT_SNAP:
        i += 1
        w = 0.0
    if i < 0 or i > n - 1:
        return 0, 0, 0.0, False
    if w == 0.0:
        return i, i, 0.0, True
    if i == n - 1:
        return 0, 0, 0.0, False
    return i, i + 1, w, True


def _bilin_abs(c00, c01, c10, c11, wv, wx, j_inf):
    if c00 >= j_inf or c01 >= j_inf or c10 >= j_inf or c11 >= j_inf:
        return j_inf
    lo = c00 + wv * (c10 - c00)
    hi = c01 + wv * (c11 - c01)
    return lo + wx * (hi - lo)


@dataclass
class CostToGoTable:
    """Cost-to-go on one node's (v, soc, t) grid (dp.py:105-134)."""

    values: np.ndarray
    v_axis: np.ndarray
    soc_axis: np.ndarray
    t_axis: np.ndarray
    j_inf: float

    def interpolate(self, v: float, soc: float, t: float) -> float:
        """Trilinear value with absorbing infeasibility; j_inf off the hull."""
        def cell(axis, q):
            n = axis.shape[0]
            a0 = float(axis[0])
            return locate_uniform(q, a0, (float(axis[-1]) - a0) / (n - 1), n)
        a0, a1, wa, oka = cell(self.v_axis, v)
        b0, b1, wb, okb = cell(self.soc_axis, soc)
        c0, c1, wc, okc = cell(self.t_axis, t)
        if not (oka and okb and okc):
            return self.j_inf
        J, ji = self.values, self.j_inf

        def bil(k):
            return _bilin_abs(float(J[a0, b0, k]), float(J[a0, b1, k]), float(J[a1, b0, k]),
                              float(J[a1, b1, k]), wa, wb, ji)
        r0 = bil(c0)
        if r0 >= ji:
            return ji
        if c1 == c0:
            return r0
        r1 = bil(c1)
        if r1 >= ji:
            return ji
        return r0 + wc * (r1 - r0)


@dataclass
class PolicyTable:
    """Flat action index ``ite * n_tb + itb`` per state, -1 if none (dp.py:137-151)."""

    values: np.ndarray
    te_axis: np.ndarray
    tb_axis: np.ndarray

    def action(self, iv: int, jx: int, z: int):
        flat = int(self.values[iv, jx, z])
        if flat < 0:
            return None
        ntb = self.tb_axis.shape[0]
        return float(self.te_axis[flat // ntb]), float(self.tb_axis[flat % ntb])


def interpolate_value(table: CostToGoTable, x: StateVector) -> float:
    return table.interpolate(x.v, x.soc, x.t)


# ------------------------------------------------------------ solve context

@dataclass
class StepPlan:
    """Constants of one spatial step m -> m+1 (dp.py:173-188)."""

    node: int
    src_kind: int
    dest_kind: int
    grade: float
    v_src: np.ndarray
    v0_dest: float
    dv_dest: float
    arr_green: np.ndarray
    dep_ok: np.ndarray
    t_dep: np.ndarray
    wait: np.ndarray


@dataclass
class SolveContext:
    """Inputs of one horizon solve at node s, clock t_start (dp.py:191-214)."""

    vehicle: Vehicle
    route: Route
    s: int
    horizon: int
    t_start: float
    gamma: float
    teleport: bool
    grids: GridSpec
    penalty: PenaltyConfig
    soc_axis: np.ndarray
    t_axis: np.ndarray
    te_axis: np.ndarray
    tb_axis: np.ndarray
    v_axes: list
    steps: list
    terminal: np.ndarray

    @property
    def pack(self) -> PlantPack:
        return self.vehicle.pack()


def node_ladders(route: Route, spat: SpatSchedule, node: int, t_axis: np.ndarray, teleport: bool):
    """(green, dep_ok, t_dep, wait) of one node on the ladder (dp.py:217-252)."""
    nt = t_axis.shape[0]
    green = np.ones(nt, dtype=np.uint8)
    dep_ok = np.ones(nt, dtype=np.uint8)
    t_dep = np.array(t_axis, dtype=np.float64)
    wait = np.zeros(nt)
    kind = route.node_kind(node)
    if kind == NODE_SIGNAL:
        timing = spat.timing(route.traffic_lights[node])
        for z in range(nt):
            tz = float(t_axis[z])
            if timing.is_green(tz):
                continue
            green[z] = 0
            if teleport:
                t_dep[z] = timing.next_green_from(tz)
                wait[z] = t_dep[z] - tz
            else:
                dep_ok[z] = 0
    elif kind == NODE_STOP:
        t_dep = t_axis + route.stop_dwell
        wait[:] = route.stop_dwell
    return green, dep_ok, t_dep, wait


def terminal_seed(base2d: np.ndarray, soc_axis: np.ndarray, penalty: PenaltyConfig, n_t: int) -> np.ndarray:
    """min(base + w (xi - xi*)^2, j_inf), j_inf where base >= j_inf, repeated
    along t (dp.py:322-334)."""
    j_inf = penalty.j_inf
    quad = penalty.soc_weight * (soc_axis - penalty.soc_target) ** 2
    seed = np.where(base2d >= j_inf, j_inf, np.minimum(base2d + quad[None, :], j_inf))
    return np.ascontiguousarray(np.repeat(seed[:, :, None], n_t, axis=2))


def build_context(vehicle: Vehicle, route: Route, spat: SpatSchedule, s: int, t_start: float, *,
                  grids: GridSpec, penalty: PenaltyConfig, gamma: float, horizon: Optional[int] = None,
                  teleport: bool = True, terminal_field: Optional[np.ndarray] = None) -> SolveContext:
    """All per-step constants of one horizon solve (dp.py:255-341)."""
    n = route.node_count
    if not 0 <= s < n - 1:
        raise ValueError(f"start node {s} out of range for route of {n} nodes")
    if not 0.0 <= gamma <= 1.0:
        raise ValueError("gamma must lie in [0, 1]")
    h_max = n - 1 - s
    h = h_max if horizon is None else min(horizon, h_max)
    if h < 1:
        raise ValueError("horizon must cover at least one spatial step")
    kinds = route.node_kinds()
    soc_axis = grids.soc_axis(vehicle)
    t_axis = grids.t_axis(t_start)
    v_axes = [grids.v_axis(route, s + k) for k in range(h + 1)]
    lad = [node_ladders(route, spat, s + k, t_axis, teleport) for k in range(h + 1)]
    steps = []
    for k in range(h):
        vd = v_axes[k + 1]
        _, dep_ok, t_dep, wait = lad[k]
        steps.append(StepPlan(
            node=s + k, src_kind=int(kinds[s + k]), dest_kind=int(kinds[s + k + 1]),
            grade=float(route.grade[s + k]), v_src=v_axes[k], v0_dest=float(vd[0]),
            dv_dest=(float(vd[-1]) - float(vd[0])) / (grids.n_v - 1),
            arr_green=lad[k + 1][0], dep_ok=dep_ok, t_dep=t_dep, wait=wait))
    if terminal_field is None:
        base = np.zeros((grids.n_v, grids.n_soc))
    else:
        base = np.asarray(terminal_field, dtype=np.float64)
        if base.shape != (grids.n_v, grids.n_soc):
            raise ValueError("terminal_field shape does not match the state grid")
    return SolveContext(
        vehicle=vehicle, route=route, s=s, horizon=h, t_start=t_start, gamma=gamma, teleport=teleport,
        grids=grids, penalty=penalty, soc_axis=soc_axis, t_axis=t_axis, te_axis=grids.te_axis(),
        tb_axis=grids.tb_axis(), v_axes=v_axes, steps=steps,
        terminal=terminal_seed(base, soc_axis, penalty, grids.n_t))


# ----------------------------------------------------------- ABI marshaling

def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


_PLANT_CACHE: dict = {}


def _plant_of(pack) -> "_abi.EcoPlant":
    """EcoPlant of a PlantPack, cached by identity (a Vehicle keeps one pack;
    the cache holds the pack, so its id cannot be reused while cached)."""
    hit = _PLANT_CACHE.get(id(pack))
    if hit is not None and hit[0] is pack:
        return hit[1]
    if len(_PLANT_CACHE) > 64:
        _PLANT_CACHE.clear()
    plant = _abi.pack_plant(pack)
    _PLANT_CACHE[id(pack)] = (pack, plant)
    return plant


# EcoStepPlan as a numpy record (the plans of a solve are filled vectorised;
# ctypes pointer objects per field cost ~4 us each)
_PLAN_DTYPE = np.dtype([("node", "<i4"), ("src_kind", "<i4"), ("dest_kind", "<i4"), ("reserved", "<i4"),
                        ("grade", "<f8"), ("v0_dest", "<f8"), ("dv_dest", "<f8"), ("cos_grade", "<f8"),
                        ("sin_grade", "<f8"), ("v_src", "<u8"), ("arr_green", "<u8"), ("dep_ok", "<u8"),
                        ("t_dep", "<u8"), ("wait", "<u8")])
assert _PLAN_DTYPE.itemsize == C.sizeof(_abi.EcoStepPlan)


class _Marshal:
    """ctypes views of a SolveContext (keeps every numpy buffer alive)."""

    def __init__(self, ctx: SolveContext, steps: Sequence[StepPlan]):
        g = ctx.grids
        self.plant = _plant_of(ctx.pack)
        self.te, self.tb = _f64(ctx.te_axis), _f64(ctx.tb_axis)
        self.soc, self.tax = _f64(ctx.soc_axis), _f64(ctx.t_axis)
        self.prob = _abi.EcoProblem(
            n_v=g.n_v, n_soc=g.n_soc, n_t=g.n_t, n_te=self.te.size, n_tb=self.tb.size,
            delta_d=float(ctx.route.delta_d), a_min=float(ctx.route.accel_min),
            a_max=float(ctx.route.accel_max), gamma=float(ctx.gamma), j_inf=float(ctx.penalty.j_inf),
            t0=float(ctx.t_axis[0]), dtg=float(g.dt),
            te_axis=_abi.ptr(self.te, C.c_double), tb_axis=_abi.ptr(self.tb, C.c_double),
            soc_axis=_abi.ptr(self.soc, C.c_double), t_axis=_abi.ptr(self.tax, C.c_double))
        n = len(steps)
        # the plans' arrays stacked into one block each; per-plan pointers by
        # address arithmetic
        self.v = np.ascontiguousarray(np.stack([p.v_src for p in steps]), dtype=np.float64)
        self.green = np.ascontiguousarray(np.stack([p.arr_green for p in steps]), dtype=np.uint8)
        self.dep = np.ascontiguousarray(np.stack([p.dep_ok for p in steps]), dtype=np.uint8)
        self.tdep = np.ascontiguousarray(np.stack([p.t_dep for p in steps]), dtype=np.float64)
        self.wait = np.ascontiguousarray(np.stack([p.wait for p in steps]), dtype=np.float64)
        rec = np.zeros(n, dtype=_PLAN_DTYPE)
        rec["node"] = [p.node for p in steps]
        rec["src_kind"] = [p.src_kind for p in steps]
        rec["dest_kind"] = [p.dest_kind for p in steps]
        grade = np.array([p.grade for p in steps], dtype=np.float64)
        rec["grade"] = grade
        rec["v0_dest"] = [p.v0_dest for p in steps]
        rec["dv_dest"] = [p.dv_dest for p in steps]
        # libm cos / sin (road_load's trig is not recomputed on the device)
        rec["cos_grade"] = [math.cos(float(x)) for x in grade]
        rec["sin_grade"] = [math.sin(float(x)) for x in grade]
        idx = np.arange(n, dtype=np.uint64)
        for field, arr in (("v_src", self.v), ("arr_green", self.green), ("dep_ok", self.dep),
                           ("t_dep", self.tdep), ("wait", self.wait)):
            rec[field] = np.uint64(arr.ctypes.data) + idx * np.uint64(arr.strides[0])
        self.rec = rec
        self.plans = rec.ctypes.data_as(C.POINTER(_abi.EcoStepPlan))


def backward_step(ctx: SolveContext, k: int, J_next: np.ndarray, *, backend: str = "b200",
                  workers: int = 8, perturb_ties: bool = False, stats: Optional[dict] = None):
    """One Bellman update node s+k+1 -> s+k (dp.py:365-404) on the device.

    ``workers`` is accepted for signature compatibility and ignored (the
    device partition never changes results)."""
    prec = precision_of(backend)
    if perturb_ties:
        prec |= _abi.REVERSE_TIES
    g = ctx.grids
    m = _Marshal(ctx, [ctx.steps[k]])
    J_next = _f64(J_next)
    if J_next.shape != (g.n_v, g.n_soc, g.n_t):
        raise ValueError("J_next shape does not match the grid")
    # page-locked outputs (recycled): direct DMA / host widening
    J_out = _abi.PINNED.array(J_next.shape, np.float64)
    P_out = _abi.PINNED.array(J_next.shape, np.int32)
    st = _abi.EcoStats()
    _abi.check(_abi.lib().eco_bellman_step(
        C.byref(m.plant), C.byref(m.prob), m.plans, None, _abi.ptr(J_next, C.c_double),
        _abi.ptr(J_out, C.c_double), _abi.ptr(P_out, C.c_int32), prec, 0, C.byref(st)), "eco_bellman_step")
    if stats is not None:
        stats.update(st.as_dict())
    return J_out, P_out


@dataclass
class SolveResult:
    """Tables and diagnostics of one horizon solve (dp.py:407-422)."""

    s: int
    horizon: int
    t_start: float
    backend: str
    cost_at_start: float
    tables: list
    policies: list
    wall_time_s: float
    stats: dict = dc_field(default_factory=dict)

    @property
    def start_table(self) -> CostToGoTable:
        return self.tables[0]


def release_workspace():
    """Free the device workspace the stateless solvers keep between calls
    and the idle page-locked output blocks."""
    _abi.check(_abi.lib().eco_release_workspace(), "eco_release_workspace")
    _abi.PINNED.clear()


def solve_stacks(ctx, backend: str = "b200", count_live: bool = False, perturb_ties: bool = False):
    """Device solve of a context -> (J stack (H+1, n_v, n_soc, n_t) f64,
    P stack (H, ...) int32, stats).  ``ctx`` only needs the reference
    SolveContext's attributes (dp.py:191-214), so this also serves the
    reference's own objects (see plugin.py).  ``perturb_ties``: ties go to the
    highest flat action index (the reference's reverse_ties negative control,
    _kernels.py:630-632)."""
    prec = precision_of(backend) | (_abi.REVERSE_TIES if perturb_ties else 0)
    g, H = ctx.grids, ctx.horizon
    m = _Marshal(ctx, ctx.steps)
    terminal = _f64(ctx.terminal)
    # page-locked output blocks (recycled): the levels arrive by direct DMA
    # while the remaining stages still sweep
    J_stack = _abi.PINNED.array((H + 1, g.n_v, g.n_soc, g.n_t), np.float64)
    P_stack = _abi.PINNED.array((H, g.n_v, g.n_soc, g.n_t), np.int32)
    st = _abi.EcoStats()
    _abi.check(_abi.lib().eco_solve_horizon(
        C.byref(m.plant), C.byref(m.prob), m.plans, H, _abi.ptr(terminal, C.c_double),
        _abi.ptr(J_stack, C.c_double), _abi.ptr(P_stack, C.c_int32), prec, int(count_live), C.byref(st)),
        "eco_solve_horizon")
    return J_stack, P_stack, st.as_dict()


def solve_horizon(ctx: SolveContext, x_start: Optional[StateVector] = None, *, backend: str = "b200",
                  workers: int = 8, perturb_ties: bool = False, count_live: bool = False) -> SolveResult:
    """Backward recursion over the whole horizon on the device (dp.py:425-475).

    All H stages run back to back on the GPU from one upload of the context;
    the full J / P stacks come back in the reference's layout."""
    precision_of(backend)
    H = ctx.horizon
    j_inf = ctx.penalty.j_inf
    t0 = time.perf_counter()
    J_stack, P_stack, stats = solve_stacks(ctx, backend, count_live, perturb_ties)
    wall = time.perf_counter() - t0
    tables = [CostToGoTable(values=J_stack[k], v_axis=ctx.v_axes[k], soc_axis=ctx.soc_axis,
                            t_axis=ctx.t_axis, j_inf=j_inf) for k in range(H + 1)]
    policies = [PolicyTable(values=P_stack[k], te_axis=ctx.te_axis, tb_axis=ctx.tb_axis) for k in range(H)]
    cost0 = math.nan
    if x_start is not None:
        cost0 = tables[0].interpolate(x_start.v, x_start.soc, x_start.t)
        if cost0 >= j_inf:
            raise StartStateInfeasibleError(
                f"no feasible continuation from node {ctx.s} at v={x_start.v:.2f} m/s, "
                f"soc={x_start.soc:.3f}, t={x_start.t:.1f} s")
    return SolveResult(s=ctx.s, horizon=H, t_start=ctx.t_start, backend=backend, cost_at_start=cost0,
                       tables=tables, policies=policies, wall_time_s=wall, stats=stats)


# ------------------------------------------------------------- toy instances

@dataclass
class ToyInstance:
    """Table-driven instance with exact binary arithmetic (dp.py:482-535)."""

    v_axis: np.ndarray
    soc_axis: np.ndarray
    t_axis: np.ndarray
    n_actions_eng: int
    n_actions_bsg: int
    horizon: int
    pack: object
    src_kinds: Sequence[int]
    stage1: list = dc_field(default_factory=list)
    arr_green: list = dc_field(default_factory=list)
    dep_ok: list = dc_field(default_factory=list)
    t_dep: list = dc_field(default_factory=list)
    wait: list = dc_field(default_factory=list)
    terminal: Optional[np.ndarray] = None
    gamma: float = 0.5
    j_inf: float = DEFAULT_J_INF

    def finalize_step(self, step_idx: int) -> dict:
        """Destination speed cell and time shift of a step's raw tables."""
        t = self.stage1[step_idx]
        nv = self.v_axis.shape[0]
        v0 = float(self.v_axis[0])
        dv = (float(self.v_axis[-1]) - v0) / (nv - 1)
        dtg = (float(self.t_axis[-1]) - float(self.t_axis[0])) / (self.t_axis.shape[0] - 1)
        shape = t["ok"].shape
        cells = {k: np.zeros(shape, dtype=np.int32) for k in ("ivlo", "ivhi", "zoff")}
        cells.update(wv=np.zeros(shape), wz=np.zeros(shape))
        for idx in np.ndindex(shape):
            if not t["ok"][idx]:
                continue
            lo, hi, w, okv = locate_uniform(float(t["v2"][idx]), v0, dv, nv)
            if not okv:
                t["ok"][idx] = 0
                continue
            cells["ivlo"][idx], cells["ivhi"][idx], cells["wv"][idx] = lo, hi, w
            d = float(t["dt"][idx]) / dtg
            z = math.floor(d)
            wz = d - z
            if wz < WEIGHT_SNAP:
                wz = 0.0
            elif wz > 1.0 - WEIGHT_SNAP:
                z, wz = z + 1, 0.0
            cells["zoff"][idx], cells["wz"][idx] = z, wz
        t.update(cells)
        return t


def make_toy_pack(r0: float = 0.25, c_nom: float = 64.0, voc: float = 2.0) -> PlantPack:
    """Battery-only plant for toy instances (dp.py:538-554)."""
    one = np.array([0.0, 1.0])
    big = np.array([1.0e30, 1.0e30])
    return PlantPack(
        mass=1.0, c0=0.0, c1=0.0, c2=0.0, wheel_radius=1.0, final_drive=1.0,
        gear_ratios=np.array([1.0]), gear_eff=np.array([1.0]), shift_v=np.array([1.0e30]),
        idle_speed=1.0, belt_ratio=1.0, eng_w=one, eng_tmin=-big, eng_tmax=big,
        fuel_w=one, fuel_t=one, fuel_vals=np.zeros((2, 2)), bsg_w=one, bsg_tmin=-big, bsg_tmax=big,
        bsgeff_w=one, bsgeff_t=one, bsgeff_vals=np.ones((2, 2)), r0=r0, c_nom=c_nom,
        voc_soc=one, voc_v=np.array([voc, voc]), soc_min=0.0, soc_max=1.0,
        p_bat_max=voc * voc / (4.0 * r0))


def solve_toy(toy: ToyInstance, *, backend: str = "b200", workers: int = 4, perturb_ties: bool = False):
    """Backward recursion over a toy instance -> (J stack, P stack) (dp.py:557-610)."""
    prec = precision_of(backend) | (_abi.REVERSE_TIES if perturb_ties else 0)
    nv, nx, nt = toy.v_axis.shape[0], toy.soc_axis.shape[0], toy.t_axis.shape[0]
    nte, ntb = toy.n_actions_eng, toy.n_actions_bsg
    t0 = float(toy.t_axis[0])
    dtg = (float(toy.t_axis[-1]) - t0) / (nt - 1)
    H = toy.horizon
    keep = []
    tables = (_abi.EcoStage1Tables * H)()
    plans = (_abi.EcoStepPlan * H)()
    v_axis = _f64(toy.v_axis)
    for k in range(H):
        t = toy.finalize_step(k)
        arr = dict(ok=np.ascontiguousarray(t["ok"], dtype=np.uint8), v2=_f64(t["v2"]), dt=_f64(t["dt"]),
                   pbat=_f64(t["pbat"]), c1=_f64(t["c1"]),
                   ivlo=np.ascontiguousarray(t["ivlo"], dtype=np.int32),
                   ivhi=np.ascontiguousarray(t["ivhi"], dtype=np.int32), wv=_f64(t["wv"]),
                   zoff=np.ascontiguousarray(t["zoff"], dtype=np.int32), wz=_f64(t["wz"]))
        lad = (np.ascontiguousarray(toy.arr_green[k], dtype=np.uint8),
               np.ascontiguousarray(toy.dep_ok[k], dtype=np.uint8), _f64(toy.t_dep[k]), _f64(toy.wait[k]))
        keep.append((arr, lad))
        tables[k] = _abi.EcoStage1Tables(
            ok=_abi.ptr(arr["ok"], C.c_uint8), v2=_abi.ptr(arr["v2"], C.c_double),
            dt=_abi.ptr(arr["dt"], C.c_double), pbat=_abi.ptr(arr["pbat"], C.c_double),
            c1=_abi.ptr(arr["c1"], C.c_double), ivlo=_abi.ptr(arr["ivlo"], C.c_int32),
            ivhi=_abi.ptr(arr["ivhi"], C.c_int32), wv=_abi.ptr(arr["wv"], C.c_double),
            zoff=_abi.ptr(arr["zoff"], C.c_int32), wz=_abi.ptr(arr["wz"], C.c_double))
        plans[k] = _abi.EcoStepPlan(
            node=k, src_kind=int(toy.src_kinds[k]), dest_kind=0, grade=0.0, v0_dest=float(v_axis[0]),
            dv_dest=(float(v_axis[-1]) - float(v_axis[0])) / (nv - 1), cos_grade=1.0, sin_grade=0.0,
            v_src=_abi.ptr(v_axis, C.c_double), arr_green=_abi.ptr(lad[0], C.c_uint8),
            dep_ok=_abi.ptr(lad[1], C.c_uint8), t_dep=_abi.ptr(lad[2], C.c_double),
            wait=_abi.ptr(lad[3], C.c_double))
    plant = _abi.pack_plant(toy.pack)
    te, tb = np.zeros(nte), np.zeros(ntb)
    soc, tax = _f64(toy.soc_axis), _f64(toy.t_axis)
    prob = _abi.EcoProblem(
        n_v=nv, n_soc=nx, n_t=nt, n_te=nte, n_tb=ntb, delta_d=1.0, a_min=-1.0e30, a_max=1.0e30,
        gamma=float(toy.gamma), j_inf=float(toy.j_inf), t0=t0, dtg=dtg,
        te_axis=_abi.ptr(te, C.c_double), tb_axis=_abi.ptr(tb, C.c_double),
        soc_axis=_abi.ptr(soc, C.c_double), t_axis=_abi.ptr(tax, C.c_double))
    terminal = _f64(toy.terminal)
    J = np.empty((H + 1, nv, nx, nt))
    P = np.empty((H, nv, nx, nt), dtype=np.int32)
    _abi.check(_abi.lib().eco_solve_tables(
        C.byref(plant), C.byref(prob), plans, tables, H, _abi.ptr(terminal, C.c_double),
        _abi.ptr(J, C.c_double), _abi.ptr(P, C.c_int32), prec), "eco_solve_tables")
    return [J[k] for k in range(H + 1)], [P[k] for k in range(H)]


# ------------------------------------------------- digests and snapshots

_MAGIC = b"ECODPT01"


def table_digest(arr: np.ndarray) -> str:
    """blake2b-64 over dtype, shape and bytes (parallel.py:165-171)."""
    h = hashlib.blake2b(digest_size=8)
    h.update(str(arr.dtype).encode())
    h.update(struct.pack("<%dq" % arr.ndim, *arr.shape))
    h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def solve_digests(result: SolveResult) -> list:
    out = []
    for k, tab in enumerate(result.tables):
        pd = table_digest(result.policies[k].values) if k < len(result.policies) else "-"
        out.append((k, table_digest(tab.values), pd))
    return out


def dump_tables(path: str, result: SolveResult) -> None:
    """ECODPT01 little-endian snapshot (parallel.py:183-198)."""
    g0 = result.tables[0].values
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(struct.pack("<IIII", result.horizon, *g0.shape))
        fh.write(struct.pack("<d", result.t_start))
        for tab in result.tables:
            fh.write(np.ascontiguousarray(tab.values, dtype="<f8").tobytes())
        for pol in result.policies:
            fh.write(np.ascontiguousarray(pol.values, dtype="<i4").tobytes())


def load_tables(path: str):
    """Read an ECODPT01 snapshot -> (horizon, t_start, [J], [P])."""
    with open(path, "rb") as fh:
        magic = fh.read(8)
        if magic != _MAGIC:
            raise ValueError(f"not a table snapshot: bad magic {magic!r}")
        horizon, n_v, n_soc, n_t = struct.unpack("<IIII", fh.read(16))
        (t_start,) = struct.unpack("<d", fh.read(8))
        cnt = n_v * n_soc * n_t
        J = [np.frombuffer(fh.read(cnt * 8), dtype="<f8").reshape(n_v, n_soc, n_t).copy()
             for _ in range(horizon + 1)]
        P = [np.frombuffer(fh.read(cnt * 4), dtype="<i4").reshape(n_v, n_soc, n_t).copy()
             for _ in range(horizon)]
    return horizon, t_start, J, P
