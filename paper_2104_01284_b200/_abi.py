"""ctypes mirror of include/eco_b200.h and the loader of the sm_100a library.

The shared library ``_eco_b200.so`` is built in-tree by
``__graft_entry__.build()`` (nvcc, ``-gencode arch=compute_100a,code=sm_100a``).
There is no fallback: if it is missing or fails to load, every solver call
raises :class:`NativeLibraryError`.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from pathlib import Path

import numpy as np

from .errors import NativeLibraryError

MAX_GEARS = 16
MAX_AXIS = 32
MAX_MAP = MAX_AXIS * MAX_AXIS
MAX_WINDOWS = 8
ABI_VERSION = 6
XCHG_P2P, XCHG_NCCL = 0, 1
SLAB_INFO_BYTES = 256

OK, ERR_ARG, ERR_CUDA, ERR_NODEV = 0, 1, 2, 3
FP32, FP64 = 0, 1
REVERSE_TIES = 0x100          # OR-ed into the precision argument (perturb_ties)
RUN_OK, RUN_INFEASIBLE, RUN_PLANT, RUN_MISMATCH = 0, 1, 2, 3
RUN_COUNT_LIVE, RUN_TIME_SWEEPS = 1, 2

_D = C.c_double
_I = C.c_int32
_PD = C.POINTER(C.c_double)
_PU8 = C.POINTER(C.c_uint8)
_PI = C.POINTER(C.c_int32)
_PI8 = C.POINTER(C.c_int8)


class EcoPlant(C.Structure):
    _fields_ = [(n, _D) for n in ("mass", "c0", "c1", "c2", "wheel_radius", "final_drive",
                                  "idle_speed", "belt_ratio", "r0", "c_nom", "soc_min", "soc_max",
                                  "p_bat_max")] + \
               [(n, _I) for n in ("n_gears", "n_eng", "n_fuel_w", "n_fuel_t", "n_bsg", "n_eff_w",
                                  "n_eff_t", "n_voc")] + \
               [("gear_ratios", _D * MAX_GEARS), ("gear_eff", _D * MAX_GEARS), ("shift_v", _D * MAX_GEARS)] + \
               [(n, _D * MAX_AXIS) for n in ("eng_w", "eng_tmin", "eng_tmax", "fuel_w", "fuel_t",
                                             "bsg_w", "bsg_tmin", "bsg_tmax", "eff_w", "eff_t",
                                             "voc_soc", "voc_v")] + \
               [("fuel_vals", _D * MAX_MAP), ("eff_vals", _D * MAX_MAP)]


class EcoProblem(C.Structure):
    _fields_ = [("n_v", _I), ("n_soc", _I), ("n_t", _I), ("n_te", _I), ("n_tb", _I), ("reserved", _I),
                ("delta_d", _D), ("a_min", _D), ("a_max", _D), ("gamma", _D), ("j_inf", _D),
                ("t0", _D), ("dtg", _D),
                ("te_axis", _PD), ("tb_axis", _PD), ("soc_axis", _PD), ("t_axis", _PD)]


class EcoStepPlan(C.Structure):
    _fields_ = [("node", _I), ("src_kind", _I), ("dest_kind", _I), ("reserved", _I),
                ("grade", _D), ("v0_dest", _D), ("dv_dest", _D), ("cos_grade", _D), ("sin_grade", _D),
                ("v_src", _PD), ("arr_green", _PU8), ("dep_ok", _PU8), ("t_dep", _PD), ("wait", _PD)]


class EcoStage1Tables(C.Structure):
    _fields_ = [("ok", _PU8), ("v2", _PD), ("dt", _PD), ("pbat", _PD), ("c1", _PD),
                ("ivlo", _PI), ("ivhi", _PI), ("wv", _PD), ("zoff", _PI), ("wz", _PD)]


class EcoRoute(C.Structure):
    _fields_ = [("node_count", _I), ("reserved", _I),
                ("delta_d", _D), ("accel_min", _D), ("accel_max", _D), ("stop_dwell", _D),
                ("v_min", _PD), ("v_max", _PD), ("grade", _PD), ("cos_grade", _PD), ("sin_grade", _PD),
                ("kinds", _PI8), ("sig_cycle", _PD), ("sig_offset", _PD), ("sig_nwin", _PI),
                ("sig_win", _PD)]


class EcoMpcConfig(C.Structure):
    _fields_ = [("n_v", _I), ("n_soc", _I), ("n_t", _I), ("n_te", _I), ("n_tb", _I), ("horizon", _I),
                ("teleport", _I), ("use_terminal_field", _I), ("precision", _I), ("start_node", _I),
                ("max_steps", _I), ("reserved", _I),
                ("dt", _D), ("gamma", _D), ("soc_target", _D), ("soc_weight", _D), ("j_inf", _D),
                ("te_axis", _PD), ("tb_axis", _PD)]


class EcoTrajRow(C.Structure):
    _fields_ = [("s", _I), ("gear", _I), ("fallback", _I), ("horizon", _I)] + \
               [(n, _D) for n in ("v", "soc", "t", "t_eng", "t_bsg", "brake_force", "wait_s",
                                  "dt_move_s", "fuel_inc_g", "accel", "cost_to_go")]


class EcoStats(C.Structure):
    _fields_ = [("device_ms", _D), ("dominant_ms", _D), ("dense_updates", C.c_int64),
                ("live_updates", C.c_int64), ("stages", C.c_int64), ("kernel_launches", C.c_int64)]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}


TRAJ_DTYPE = np.dtype([("s", "<i4"), ("gear", "<i4"), ("fallback", "<i4"), ("horizon", "<i4")] +
                      [(n, "<f8") for n in ("v", "soc", "t", "t_eng", "t_bsg", "brake_force", "wait_s",
                                            "dt_move_s", "fuel_inc_g", "accel", "cost_to_go")])
assert TRAJ_DTYPE.itemsize == C.sizeof(EcoTrajRow)

# ------------------------------------------------------------------ packing


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def _fill(dst, src, cap: int, name: str) -> int:
    src = np.ascontiguousarray(src, dtype=np.float64).ravel()
    if src.size > cap:
        raise ValueError(f"{name}: {src.size} entries exceed the ABI capacity {cap}")
    C.memmove(dst, src.ctypes.data, src.size * 8)
    return int(src.size)


def pack_plant(pack) -> EcoPlant:
    """PlantPack (plant.py / _kernels.py:31-53 field set) -> EcoPlant."""
    p = EcoPlant()
    for n in ("mass", "c0", "c1", "c2", "wheel_radius", "final_drive", "idle_speed", "belt_ratio",
              "r0", "c_nom", "soc_min", "soc_max", "p_bat_max"):
        setattr(p, n, float(getattr(pack, n)))
    p.n_gears = _fill(p.gear_ratios, pack.gear_ratios, MAX_GEARS, "gear_ratios")
    _fill(p.gear_eff, pack.gear_eff, MAX_GEARS, "gear_eff")
    _fill(p.shift_v, pack.shift_v, MAX_GEARS, "shift_v")
    p.n_eng = _fill(p.eng_w, pack.eng_w, MAX_AXIS, "eng_w")
    _fill(p.eng_tmin, pack.eng_tmin, MAX_AXIS, "eng_tmin")
    _fill(p.eng_tmax, pack.eng_tmax, MAX_AXIS, "eng_tmax")
    p.n_fuel_w = _fill(p.fuel_w, pack.fuel_w, MAX_AXIS, "fuel_w")
    p.n_fuel_t = _fill(p.fuel_t, pack.fuel_t, MAX_AXIS, "fuel_t")
    _fill(p.fuel_vals, pack.fuel_vals, MAX_MAP, "fuel_vals")
    p.n_bsg = _fill(p.bsg_w, pack.bsg_w, MAX_AXIS, "bsg_w")
    _fill(p.bsg_tmin, pack.bsg_tmin, MAX_AXIS, "bsg_tmin")
    _fill(p.bsg_tmax, pack.bsg_tmax, MAX_AXIS, "bsg_tmax")
    p.n_eff_w = _fill(p.eff_w, pack.bsgeff_w, MAX_AXIS, "bsgeff_w")
    p.n_eff_t = _fill(p.eff_t, pack.bsgeff_t, MAX_AXIS, "bsgeff_t")
    _fill(p.eff_vals, pack.bsgeff_vals, MAX_MAP, "bsgeff_vals")
    p.n_voc = _fill(p.voc_soc, pack.voc_soc, MAX_AXIS, "voc_soc")
    _fill(p.voc_v, pack.voc_v, MAX_AXIS, "voc_v")
    return p


class RoutePack:
    """EcoRoute plus the numpy arrays it points into (kept alive here)."""

    def __init__(self, route, spat, signals_optional: bool = False):
        n = route.node_count
        self.kinds = np.ascontiguousarray(route.node_kinds(), dtype=np.int8)
        self.v_min = np.ascontiguousarray(route.v_min, dtype=np.float64)
        self.v_max = np.ascontiguousarray(route.v_max, dtype=np.float64)
        self.grade = np.ascontiguousarray(route.grade, dtype=np.float64)
        # libm cos/sin on the host: road_load's trig is not recomputed on the device
        self.cos_g = np.array([math.cos(float(g)) for g in self.grade])
        self.sin_g = np.array([math.sin(float(g)) for g in self.grade])
        self.cycle = np.ones(n)
        self.offset = np.zeros(n)
        self.nwin = np.zeros(n, dtype=np.int32)
        self.win = np.zeros((n, MAX_WINDOWS, 2))
        for node, sid in route.traffic_lights.items():
            if signals_optional and sid not in spat.signals:
                continue      # the always-green field sweep never reads phases
            tm = spat.timing(sid)
            if len(tm.green_windows) > MAX_WINDOWS:
                raise ValueError(f"signal {sid}: more than {MAX_WINDOWS} green windows")
            self.cycle[node] = tm.cycle
            self.offset[node] = tm.offset
            self.nwin[node] = len(tm.green_windows)
            for i, (a, b) in enumerate(tm.green_windows):
                self.win[node, i] = (a, b)
        self.c = EcoRoute(
            node_count=n, reserved=0, delta_d=float(route.delta_d), accel_min=float(route.accel_min),
            accel_max=float(route.accel_max), stop_dwell=float(route.stop_dwell),
            v_min=ptr(self.v_min, C.c_double), v_max=ptr(self.v_max, C.c_double),
            grade=ptr(self.grade, C.c_double), cos_grade=ptr(self.cos_g, C.c_double),
            sin_grade=ptr(self.sin_g, C.c_double), kinds=ptr(self.kinds, C.c_int8),
            sig_cycle=ptr(self.cycle, C.c_double), sig_offset=ptr(self.offset, C.c_double),
            sig_nwin=ptr(self.nwin, C.c_int32), sig_win=ptr(self.win, C.c_double))


# EcoSignalTiming as a numpy record (arrays of them are passed as void*)
SIGNAL_TIMING_DTYPE = np.dtype([("cycle", "<f8"), ("offset", "<f8"), ("nwin", "<i4"), ("reserved", "<i4"),
                                ("win", "<f8", (MAX_WINDOWS, 2))])
assert SIGNAL_TIMING_DTYPE.itemsize == 152


def signal_timings(route, spats) -> np.ndarray:
    """(len(spats), n_signal_nodes) EcoSignalTiming records: scenario i's
    phase plan at each signal node of ``route`` (node order)."""
    nodes = sorted(route.traffic_lights)
    out = np.zeros((len(spats), len(nodes)), dtype=SIGNAL_TIMING_DTYPE)
    for i, spat in enumerate(spats):
        for j, node in enumerate(nodes):
            tm = spat.timing(route.traffic_lights[node])
            if len(tm.green_windows) > MAX_WINDOWS:
                raise ValueError(f"signal {route.traffic_lights[node]}: more than {MAX_WINDOWS} green windows")
            rec = out[i, j]
            rec["cycle"] = tm.cycle
            rec["offset"] = tm.offset
            rec["nwin"] = len(tm.green_windows)
            for w, (a, b) in enumerate(tm.green_windows):
                rec["win"][w] = (a, b)
    return out


# ------------------------------------------------------------------ loading

LIB_NAME = "_eco_b200.so"
_LIB = None


def library_path() -> Path:
    return Path(__file__).resolve().parent / LIB_NAME


def _declare(lib):
    P = C.POINTER
    sig = {
        "eco_abi_version": (_I, []),
        "eco_last_error": (C.c_char_p, []),
        "eco_device_count": (_I, []),
        "eco_release_workspace": (_I, []),
        "eco_host_alloc": (_I, [C.c_uint64, P(C.c_void_p)]),
        "eco_debug_checks": (_I, [P(C.c_int64), P(C.c_int64), _I]),
        "eco_host_free": (_I, [C.c_void_p]),
        "eco_bellman_step": (_I, [P(EcoPlant), P(EcoProblem), P(EcoStepPlan), P(EcoStage1Tables),
                                  _PD, _PD, _PI, _I, _I, P(EcoStats)]),
        "eco_solve_horizon": (_I, [P(EcoPlant), P(EcoProblem), P(EcoStepPlan), _I, _PD, _PD, _PI, _I, _I,
                                   P(EcoStats)]),
        "eco_solve_tables": (_I, [P(EcoPlant), P(EcoProblem), P(EcoStepPlan), P(EcoStage1Tables), _I, _PD,
                                  _PD, _PI, _I]),
        "eco_field_build": (_I, [P(EcoPlant), P(EcoRoute), P(EcoMpcConfig), _PD, P(EcoStats)]),
        "eco_mpc_run": (_I, [P(EcoPlant), P(EcoRoute), P(EcoMpcConfig), _PD, _PD, _PD, P(EcoTrajRow), _PI,
                             _PI, _PI, _PD, P(EcoStats)]),
        "eco_session_create": (_I, [P(EcoPlant), P(EcoRoute), P(EcoMpcConfig), P(C.c_void_p)]),
        "eco_session_fit": (_I, [C.c_void_p, _PD, _PD, P(EcoStats)]),
        "eco_session_upload_route": (_I, [C.c_void_p, P(EcoRoute)]),
        "eco_session_run": (_I, [C.c_void_p, _I, _I, _PD, P(EcoTrajRow), _PI, _PI, _PI, _PD, _I, P(EcoStats)]),
        "eco_session_step_times": (_I, [C.c_void_p, _PD, _I]),
        "eco_session_destroy": (_I, [C.c_void_p]),
        "eco_batch_create": (_I, [P(EcoPlant), P(EcoRoute), P(EcoMpcConfig), P(C.c_void_p)]),
        "eco_batch_solve": (_I, [C.c_void_p, _I, C.c_void_p, _PI, _PD, _PD, _PI, _I, P(EcoStats)]),
        "eco_batch_destroy": (_I, [C.c_void_p]),
        "eco_slab_create": (_I, [_I, _I, _I, _PI, _I, _I, _I, _I, _I, P(C.c_void_p)]),
        "eco_slab_info": (_I, [C.c_void_p, C.c_void_p]),
        "eco_slab_connect": (_I, [C.c_void_p, C.c_void_p]),
        "eco_slab_solve": (_I, [C.c_void_p, P(EcoPlant), P(EcoProblem), P(EcoStepPlan), _I, _PD, _PD, _PI, _I,
                                P(EcoStats)]),
        "eco_slab_destroy": (_I, [C.c_void_p]),
        "eco_slab_set_host_barrier": (_I, [C.c_void_p, C.c_void_p, C.c_void_p]),
        "eco_slab_emulate": (_I, [_I, _PI, _I, P(EcoPlant), P(EcoProblem), P(EcoStepPlan), _I, _PD, _PD, _PI,
                                  P(EcoStats)]),
        "eco_solve_batch": (_I, [P(EcoPlant), P(EcoRoute), P(EcoMpcConfig), _I, C.c_void_p, _PI, _PD, _PD, _PI,
                                 P(EcoStats)]),
    }
    # ECO_B200_LIB (a variant build under study) may predate newer entry points
    lenient = "ECO_B200_LIB" in os.environ
    for name, (res, args) in sig.items():
        if lenient and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The loaded sm_100a library (raises NativeLibraryError, never falls back)."""
    global _LIB
    if _LIB is None:
        path = Path(os.environ.get("ECO_B200_LIB", library_path()))
        if not path.exists():
            raise NativeLibraryError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            _LIB = _declare(C.CDLL(str(path)))
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
        if _LIB.eco_abi_version() != ABI_VERSION and "ECO_B200_LIB" not in os.environ:
            raise NativeLibraryError("ABI version mismatch between eco_b200.h and the Python bindings")
    return _LIB


def check(status: int, what: str):
    if status == OK:
        return
    msg = lib().eco_last_error().decode(errors="replace")
    if status == ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    raise NativeLibraryError(f"{what} failed (status {status}): {msg}")


# ------------------------------------------------------------ pinned outputs

class _PinnedBuf:
    """One page-locked block exposed as a numpy array (via the array
    interface); returns the block to its pool when the last view dies."""

    def __init__(self, pool, ptr: int, cap: int, shape, dtype):
        self._pool, self._ptr, self._cap = pool, ptr, cap
        self.__array_interface__ = {"data": (ptr, False), "shape": tuple(shape),
                                    "typestr": np.dtype(dtype).str, "version": 3}

    def __del__(self):
        try:
            self._pool._give_back(self._ptr, self._cap)
        except Exception:       # interpreter shutdown
            pass


class PinnedPool:
    """Recycled page-locked host blocks for solver outputs (eco_host_alloc).

    Tables written into them arrive by direct DMA, overlapped level by level
    with the remaining sweep (eco_solve_horizon), instead of through a staging
    copy into pageable numpy memory.  Arrays handed out are ordinary numpy
    arrays; when a result is dropped its block goes back to the pool.  Idle
    blocks beyond ``keep_bytes`` are unpinned."""

    def __init__(self, keep_bytes: int = 24 << 30):
        import threading
        self._lock = threading.Lock()
        self._free = []               # (capacity, ptr)
        self._keep = keep_bytes

    def array(self, shape, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        need = max(nbytes, 1)
        with self._lock:
            best = None
            for i, (cap, ptr) in enumerate(self._free):
                if need <= cap <= 2 * need + (64 << 20) and (best is None or cap < self._free[best][0]):
                    best = i
            blk = self._free.pop(best) if best is not None else None
        if blk is None:
            cap = (need + (2 << 20) - 1) & ~((2 << 20) - 1)
            out = C.c_void_p()
            if lib().eco_host_alloc(cap, C.byref(out)) != OK or not out.value:
                # host memory could not be page-locked (or there is no
                # device, which the solver call reports): an ordinary array;
                # the library then copies through its pinned staging
                return np.empty(shape, dtype)
            blk = (cap, out.value)
        return np.asarray(_PinnedBuf(self, blk[1], blk[0], shape, dtype))

    def _give_back(self, ptr: int, cap: int):
        with self._lock:
            self._free.append((cap, ptr))
            total = sum(c for c, _ in self._free)
            drop = []
            while total > self._keep and self._free:
                c, p = self._free.pop(0)
                total -= c
                drop.append(p)
        for p in drop:
            lib().eco_host_free(p)

    def clear(self):
        with self._lock:
            drop, self._free = self._free, []
        for _, p in drop:
            lib().eco_host_free(p)


PINNED = PinnedPool()
