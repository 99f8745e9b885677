"""ctypes front end of the CPU oracle (eco_oracle.c).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product.  It
reuses the product's ABI struct *layouts* (paper_2104_01284_b200._abi) to
marshal inputs; every number it returns is computed by eco_oracle.c, a
restatement of the reference's numba kernels (see that file's header).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from paper_2104_01284_b200 import _abi
from paper_2104_01284_b200.dp import _Marshal

HERE = Path(__file__).resolve().parent
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = HERE / "_eco_oracle.so"
        if not path.exists():
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        L = C.CDLL(str(path))
        P = C.POINTER
        D, I, PD, PI = C.c_double, C.c_int, P(C.c_double), P(C.c_int)
        L.oracle_sweep_serial.restype = C.c_int64
        L.oracle_sweep_serial.argtypes = [P(_abi.EcoPlant), P(_abi.EcoProblem), P(_abi.EcoStepPlan),
                                          P(_abi.EcoStage1Tables), PD, PD, P(C.c_int32)]
        L.oracle_sweep_parallel.restype = C.c_int64
        L.oracle_sweep_parallel.argtypes = [P(_abi.EcoPlant), P(_abi.EcoProblem), P(_abi.EcoStepPlan), PD, PD,
                                            P(C.c_int32), I]
        L.oracle_field_build.restype = None
        L.oracle_field_build.argtypes = [P(_abi.EcoPlant), P(_abi.EcoRoute), P(_abi.EcoMpcConfig), PD]
        L.oracle_mpc_run.restype = I
        L.oracle_mpc_run.argtypes = [P(_abi.EcoPlant), P(_abi.EcoRoute), P(_abi.EcoMpcConfig), PD, PD, I, I, I,
                                     P(_abi.EcoTrajRow), PI, PI, PD, PD, P(C.c_int64)]
        L.oracle_step_eval.restype = I
        L.oracle_step_eval.argtypes = [P(_abi.EcoPlant), D, D, D, D, D, D, D, D, PD]
        L.oracle_battery_current.restype = I
        L.oracle_battery_current.argtypes = [P(_abi.EcoPlant), D, D, PD]
        L.oracle_locate_uniform.restype = I
        L.oracle_locate_uniform.argtypes = [D, D, D, I, PI, PI, PD]
        L.oracle_tcell_shift.restype = None
        L.oracle_tcell_shift.argtypes = [D, D, PI, PD]
        L.oracle_interp3_abs.restype = D
        L.oracle_interp3_abs.argtypes = [PD, I, I, I, I, D, I, I, D, I, I, D, D]
        L.oracle_pymod.restype = D
        L.oracle_pymod.argtypes = [D, D]
        L.oracle_is_green.restype = I
        L.oracle_is_green.argtypes = [D, D, PD, I, D]
        L.oracle_next_green.restype = D
        L.oracle_next_green.argtypes = [D, D, PD, I, D]
        L.oracle_linspace.restype = None
        L.oracle_linspace.argtypes = [D, D, I, PD]
        _LIB = L
    return _LIB


def threads_available() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ solves

def sweep(ctx, k: int, J_next: np.ndarray, parallel: bool = False, threads: int = 0):
    """One backward step of a SolveContext -> (J, P, live_count)."""
    m = _Marshal(ctx, [ctx.steps[k]])
    g = ctx.grids
    Jn = np.ascontiguousarray(J_next, dtype=np.float64)
    J = np.empty((g.n_v, g.n_soc, g.n_t))
    P = np.empty((g.n_v, g.n_soc, g.n_t), dtype=np.int32)
    if parallel:
        live = lib().oracle_sweep_parallel(C.byref(m.plant), C.byref(m.prob), m.plans,
                                           _abi.ptr(Jn, C.c_double), _abi.ptr(J, C.c_double),
                                           _abi.ptr(P, C.c_int32), threads)
    else:
        live = lib().oracle_sweep_serial(C.byref(m.plant), C.byref(m.prob), m.plans, None,
                                         _abi.ptr(Jn, C.c_double), _abi.ptr(J, C.c_double),
                                         _abi.ptr(P, C.c_int32))
    return J, P, int(live)


def solve_context(ctx, parallel: bool = False, threads: int = 0, with_live: bool = False):
    """solve_horizon restated on the CPU -> ([J_0..J_H], [P_0..P_{H-1}])."""
    J = [None] * (ctx.horizon + 1)
    P = [None] * ctx.horizon
    J[ctx.horizon] = np.array(ctx.terminal, dtype=np.float64)
    live = 0
    for k in range(ctx.horizon - 1, -1, -1):
        J[k], P[k], lv = sweep(ctx, k, J[k + 1], parallel, threads)
        live += lv
    return (J, P, live) if with_live else (J, P)


def solve_toy(toy):
    """Serial sweep in table mode (dp_sweep_serial use_tables=1) over a toy."""
    nv, nx, nt = toy.v_axis.shape[0], toy.soc_axis.shape[0], toy.t_axis.shape[0]
    nte, ntb = toy.n_actions_eng, toy.n_actions_bsg
    t0 = float(toy.t_axis[0])
    dtg = (float(toy.t_axis[-1]) - t0) / (nt - 1)
    plant = _abi.pack_plant(toy.pack)
    te, tb = np.zeros(nte), np.zeros(ntb)
    soc, tax = np.ascontiguousarray(toy.soc_axis, dtype=np.float64), np.ascontiguousarray(toy.t_axis, dtype=np.float64)
    prob = _abi.EcoProblem(n_v=nv, n_soc=nx, n_t=nt, n_te=nte, n_tb=ntb, delta_d=1.0, a_min=-1e30, a_max=1e30,
                           gamma=float(toy.gamma), j_inf=float(toy.j_inf), t0=t0, dtg=dtg,
                           te_axis=_abi.ptr(te, C.c_double), tb_axis=_abi.ptr(tb, C.c_double),
                           soc_axis=_abi.ptr(soc, C.c_double), t_axis=_abi.ptr(tax, C.c_double))
    v_axis = np.ascontiguousarray(toy.v_axis, dtype=np.float64)
    J = [None] * (toy.horizon + 1)
    P = [None] * toy.horizon
    J[toy.horizon] = np.array(toy.terminal, dtype=np.float64)
    for k in range(toy.horizon - 1, -1, -1):
        t = toy.finalize_step(k)
        arr = dict(ok=np.ascontiguousarray(t["ok"], dtype=np.uint8),
                   **{n: np.ascontiguousarray(t[n], dtype=np.float64) for n in ("v2", "dt", "pbat", "c1", "wv", "wz")},
                   **{n: np.ascontiguousarray(t[n], dtype=np.int32) for n in ("ivlo", "ivhi", "zoff")})
        tab = _abi.EcoStage1Tables(
            ok=_abi.ptr(arr["ok"], C.c_uint8), v2=_abi.ptr(arr["v2"], C.c_double), dt=_abi.ptr(arr["dt"], C.c_double),
            pbat=_abi.ptr(arr["pbat"], C.c_double), c1=_abi.ptr(arr["c1"], C.c_double),
            ivlo=_abi.ptr(arr["ivlo"], C.c_int32), ivhi=_abi.ptr(arr["ivhi"], C.c_int32),
            wv=_abi.ptr(arr["wv"], C.c_double), zoff=_abi.ptr(arr["zoff"], C.c_int32), wz=_abi.ptr(arr["wz"], C.c_double))
        lad = (np.ascontiguousarray(toy.arr_green[k], dtype=np.uint8), np.ascontiguousarray(toy.dep_ok[k], dtype=np.uint8),
               np.ascontiguousarray(toy.t_dep[k], dtype=np.float64), np.ascontiguousarray(toy.wait[k], dtype=np.float64))
        plan = _abi.EcoStepPlan(node=k, src_kind=int(toy.src_kinds[k]), dest_kind=0, grade=0.0,
                                v0_dest=float(v_axis[0]), dv_dest=(float(v_axis[-1]) - float(v_axis[0])) / (nv - 1),
                                cos_grade=1.0, sin_grade=0.0, v_src=_abi.ptr(v_axis, C.c_double),
                                arr_green=_abi.ptr(lad[0], C.c_uint8), dep_ok=_abi.ptr(lad[1], C.c_uint8),
                                t_dep=_abi.ptr(lad[2], C.c_double), wait=_abi.ptr(lad[3], C.c_double))
        Jn = J[k + 1]
        Jo = np.empty((nv, nx, nt))
        Po = np.empty((nv, nx, nt), dtype=np.int32)
        lib().oracle_sweep_serial(C.byref(plant), C.byref(prob), C.byref(plan), C.byref(tab),
                                  _abi.ptr(Jn, C.c_double), _abi.ptr(Jo, C.c_double), _abi.ptr(Po, C.c_int32))
        J[k], P[k] = Jo, Po
    return J, P


def _cfg(grids, penalty, gamma, horizon, teleport=True, use_field=True):
    te, tb = grids.te_axis(), grids.tb_axis()
    cfg = _abi.EcoMpcConfig(n_v=grids.n_v, n_soc=grids.n_soc, n_t=grids.n_t, n_te=te.size, n_tb=tb.size,
                            horizon=horizon, teleport=int(teleport), use_terminal_field=int(use_field),
                            precision=1, start_node=0, max_steps=-1, dt=float(grids.dt), gamma=float(gamma),
                            soc_target=float(penalty.soc_target), soc_weight=float(penalty.soc_weight),
                            j_inf=float(penalty.j_inf), te_axis=_abi.ptr(te, C.c_double),
                            tb_axis=_abi.ptr(tb, C.c_double))
    return cfg, (te, tb)


def field_build(vehicle, route, spat, grids, penalty, gamma):
    """build_terminal_cost restated -> (node_count, n_v, n_soc)."""
    rp = _abi.RoutePack(route, spat, signals_optional=True)
    cfg, keep = _cfg(grids, penalty, gamma, 1)
    plant = _abi.pack_plant(vehicle.pack())
    out = np.empty((route.node_count, grids.n_v, grids.n_soc))
    lib().oracle_field_build(C.byref(plant), C.byref(rp.c), C.byref(cfg), _abi.ptr(out, C.c_double))
    return out


def mpc_run(vehicle, route, spat, grids, penalty, gamma, horizon, x_start, field=None, *, teleport=True,
            parallel=True, threads=0, max_steps=-1):
    """simulate_closed_loop(EcoDrivingMPC) restated.  field=None runs without a
    terminal field.  Returns dict(rows, status, status_node, final, solve_s, live)."""
    rp = _abi.RoutePack(route, spat)
    cfg, keep = _cfg(grids, penalty, gamma, horizon, teleport, field is not None)
    plant = _abi.pack_plant(vehicle.pack())
    x0 = np.array(x_start, dtype=np.float64)
    rows = np.zeros(max(route.node_count - 1, 1), dtype=_abi.TRAJ_DTYPE)
    st, node = C.c_int(0), C.c_int(-1)
    fin = np.zeros(3)
    secs = C.c_double(0.0)
    live = C.c_int64(0)
    fld = None if field is None else np.ascontiguousarray(field, dtype=np.float64)
    n = lib().oracle_mpc_run(C.byref(plant), C.byref(rp.c), C.byref(cfg), _abi.ptr(x0, C.c_double),
                             None if fld is None else _abi.ptr(fld, C.c_double), 1 if parallel else 0, threads,
                             max_steps, rows.ctypes.data_as(C.POINTER(_abi.EcoTrajRow)), C.byref(st),
                             C.byref(node), _abi.ptr(fin, C.c_double), C.byref(secs), C.byref(live))
    if n < 0:
        raise RuntimeError("oracle: solver/plant prediction mismatch")
    return dict(rows=rows[:n], status=st.value, status_node=node.value, final=fin, solve_s=secs.value,
                live=live.value)


# ------------------------------------------------------------- primitives

def step_eval(vehicle, v, te, tb, dd, grade, a_min, a_max, brake):
    out = np.zeros(7)
    p = _abi.pack_plant(vehicle.pack() if hasattr(vehicle, "pack") else vehicle)
    feas = lib().oracle_step_eval(C.byref(p), v, te, tb, dd, grade, a_min, a_max, brake, _abi.ptr(out, C.c_double))
    return (feas, out[0], bool(out[1]), out[2], out[3], out[4], out[5], out[6])


def locate_uniform(x, x0, dx, n):
    lo, hi, w = C.c_int(0), C.c_int(0), C.c_double(0.0)
    ok = lib().oracle_locate_uniform(x, x0, dx, n, C.byref(lo), C.byref(hi), C.byref(w))
    return lo.value, hi.value, w.value, bool(ok)


def pymod(a, b):
    return lib().oracle_pymod(a, b)


def is_green(timing, t):
    w = np.ascontiguousarray(np.asarray(timing.green_windows, dtype=np.float64).reshape(-1))
    return bool(lib().oracle_is_green(timing.cycle, timing.offset, _abi.ptr(w, C.c_double),
                                      len(timing.green_windows), t))


def next_green(timing, t):
    w = np.ascontiguousarray(np.asarray(timing.green_windows, dtype=np.float64).reshape(-1))
    return lib().oracle_next_green(timing.cycle, timing.offset, _abi.ptr(w, C.c_double),
                                   len(timing.green_windows), t)


def linspace(a, b, n):
    out = np.empty(n)
    lib().oracle_linspace(a, b, n, _abi.ptr(out, C.c_double))
    return out
