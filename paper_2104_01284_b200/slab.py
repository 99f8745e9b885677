"""Slab-partitioned horizon solve across GPUs (C5).

The reference parallelises one Bellman stage by giving each worker a
contiguous run of whole speed planes (``WorkPartition`` / ``make_partition``,
``pkg/src/ecodrive/parallel.py:59-106``; ``dp_stage2_sweep`` workers own
v-plane slabs, ``_kernels.py:649-651``).  Here each GPU (one process per GPU,
``torch.distributed`` for the host-side rendezvous) owns such a slab of every
level: it sweeps its planes reading the full J_{k+1}, then the slabs are
exchanged so every rank holds the full J_k before the next stage:

* ``exchange="p2p"`` -- the stage kernel's epilogue stores its outputs into
  every peer's replica of the level over NVLink (CUDA IPC handles exchanged
  here) and a GPU-side flag barrier closes the stage: no separate collective;
* ``exchange="nccl"`` -- one grouped ``ncclBroadcast`` per slab after the
  stage kernel (the library baseline).

Policies stay sharded: :meth:`SlabSolver.solve` returns this rank's planes;
:func:`gather_policies` assembles the full tables on one rank.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _abi
from .dp import _Marshal, _f64, precision_of

EXCHANGES = {"p2p": _abi.XCHG_P2P, "nccl": _abi.XCHG_NCCL}


def make_partition(n_v: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous speed-plane runs per rank, exactly parallel.py:87-101:
    rint(linspace(0, n_v, world + 1)); every rank must own >= 1 plane."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    if world > n_v:
        raise ValueError(f"{world} ranks but only {n_v} speed planes")
    edges = np.rint(np.linspace(0, n_v, world + 1)).astype(np.int64)
    return [(int(edges[g]), int(edges[g + 1])) for g in range(world)]


@dataclass
class SlabResult:
    planes: Tuple[int, int]               # [lo, hi) speed planes of this rank
    P: Optional[np.ndarray]               # (H, hi - lo, n_soc, n_t) int32
    J: Optional[np.ndarray]               # (H + 1, n_v, n_soc, n_t) f64 (full: every rank holds it)
    stats: dict = field(default_factory=dict)


def _dist():
    try:
        import torch.distributed as dist
    except ImportError:        # pragma: no cover
        return None
    return dist if dist.is_available() and dist.is_initialized() else None


class SlabSolver:
    """One rank of a slab-partitioned solver (collective: every rank of the
    process group constructs it and calls :meth:`solve` with the same context)."""

    def __init__(self, n_v: int, n_soc: int, n_t: int, max_horizon: int, *, backend: str = "b200",
                 exchange: str = "p2p", rank: Optional[int] = None, world: Optional[int] = None, group=None,
                 host_barrier: bool = False):
        """``host_barrier`` (tests): close each P2P stage with a stream sync +
        a barrier of the process group on the host instead of the GPU-side
        flag barrier, so several ranks can share ONE GPU (their kernels must
        not wait on one another there); the data path -- CUDA IPC replicas,
        epilogue stores into peers, local copy-1 rebuild -- is unchanged."""
        if exchange not in EXCHANGES:
            raise ValueError(f"unknown exchange {exchange!r} (p2p | nccl)")
        dist = _dist()
        if rank is None or world is None:
            rank, world = (dist.get_rank(group), dist.get_world_size(group)) if dist else (0, 1)
        self.rank, self.world, self.exchange = rank, world, exchange
        self.partition = make_partition(n_v, world)
        self.grid = (n_v, n_soc, n_t)
        self.max_horizon = max_horizon
        self._lib = _abi.lib()
        self._h = C.c_void_p()
        bounds = np.array([lo for lo, _ in self.partition] + [n_v], dtype=np.int32)
        _abi.check(self._lib.eco_slab_create(world, rank, EXCHANGES[exchange], _abi.ptr(bounds, C.c_int32),
                                             precision_of(backend), n_v, n_soc, n_t, max_horizon,
                                             C.byref(self._h)), "eco_slab_create")
        info = (C.c_uint8 * _abi.SLAB_INFO_BYTES)()
        _abi.check(self._lib.eco_slab_info(self._h, info), "eco_slab_info")
        infos = [bytes(info)]
        if world > 1:
            if dist is None:
                raise RuntimeError("a multi-rank SlabSolver needs an initialised torch.distributed group")
            infos = [None] * world
            dist.all_gather_object(infos, bytes(info), group=group)
        allinfo = (C.c_uint8 * (_abi.SLAB_INFO_BYTES * world)).from_buffer_copy(b"".join(infos))
        _abi.check(self._lib.eco_slab_connect(self._h, allinfo), "eco_slab_connect")
        self._barrier_cb = None
        if host_barrier and world > 1:
            grp = group

            def _barrier(_user):
                dist.barrier(group=grp)

            self._barrier_cb = C.CFUNCTYPE(None, C.c_void_p)(_barrier)
            _abi.check(self._lib.eco_slab_set_host_barrier(self._h, C.cast(self._barrier_cb, C.c_void_p), None),
                       "eco_slab_set_host_barrier")

    def solve(self, ctx, *, return_J: bool = False, return_P: bool = True, count_live: bool = False) -> SlabResult:
        g = ctx.grids
        if (g.n_v, g.n_soc, g.n_t) != self.grid:
            raise ValueError("context grid differs from the solver's")
        H = ctx.horizon
        lo, hi = self.partition[self.rank]
        m = _Marshal(ctx, ctx.steps)
        terminal = _f64(ctx.terminal)
        J = np.empty((H + 1, g.n_v, g.n_soc, g.n_t)) if return_J else None
        P = np.empty((H, hi - lo, g.n_soc, g.n_t), dtype=np.int32) if return_P else None
        st = _abi.EcoStats()
        _abi.check(self._lib.eco_slab_solve(
            self._h, C.byref(m.plant), C.byref(m.prob), m.plans, H, _abi.ptr(terminal, C.c_double),
            None if J is None else _abi.ptr(J, C.c_double), None if P is None else _abi.ptr(P, C.c_int32),
            int(count_live), C.byref(st)), "eco_slab_solve")
        return SlabResult(planes=(lo, hi), P=P, J=J, stats=st.as_dict())

    def close(self):
        if self._h:
            self._lib.eco_slab_destroy(self._h)
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


def emulate_slabs(ctx, world: int, backend: str = "b200"):
    """The ``world``-rank slab decomposition of one solve emulated on ONE GPU
    (eco_slab_emulate): every rank's replica of the J stack, (world, H + 1,
    n_v, n_soc, n_t), and the policy stack assembled from the slabs.  GPU-count
    invariance (test_parallel.py:164-171) means every replica equals the
    unpartitioned solve_horizon."""
    g, H = ctx.grids, ctx.horizon
    part = make_partition(g.n_v, world)
    bounds = np.array([lo for lo, _ in part] + [g.n_v], dtype=np.int32)
    m = _Marshal(ctx, ctx.steps)
    terminal = _f64(ctx.terminal)
    J = np.empty((world, H + 1, g.n_v, g.n_soc, g.n_t))
    P = np.empty((H, g.n_v, g.n_soc, g.n_t), dtype=np.int32)
    st = _abi.EcoStats()
    _abi.check(_abi.lib().eco_slab_emulate(world, _abi.ptr(bounds, C.c_int32), precision_of(backend),
                                           C.byref(m.plant), C.byref(m.prob), m.plans, H,
                                           _abi.ptr(terminal, C.c_double), _abi.ptr(J, C.c_double),
                                           _abi.ptr(P, C.c_int32), C.byref(st)), "eco_slab_emulate")
    return J, P, st.as_dict()


def gather_policies(res: SlabResult, n_v: int, dst: int = 0, group=None) -> Optional[np.ndarray]:
    """Assemble the full (H, n_v, n_soc, n_t) policy stack on rank ``dst``
    from every rank's slab (host transport of the process group)."""
    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        return res.P
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, (res.planes, res.P), group=group)
    if dist.get_rank(group) != dst:
        return None
    H, _, nx, nt = res.P.shape
    out = np.empty((H, n_v, nx, nt), dtype=np.int32)
    for (lo, hi), p in parts:
        out[:, lo:hi] = p
    return out


__all__ = ["SlabSolver", "SlabResult", "make_partition", "gather_policies", "emulate_slabs", "EXCHANGES"]
