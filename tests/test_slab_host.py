"""C5 host side on CPU: the slab partition mirrors the reference's
make_partition, and the slab decomposition + per-stage exchange reproduces
the unpartitioned solve (oracle sweeps per rank, gloo world_size 2)."""

import numpy as np
import pytest

from _dist import run_gloo
from paper_2104_01284_b200 import NativeLibraryError, _abi
from paper_2104_01284_b200.slab import SlabResult, SlabSolver, gather_policies, make_partition


def _ref_partition(n_v, world):
    # parallel.py:87-101 restated: rint(linspace(0, n_v, w + 1)), planes not split
    edges = np.unique(np.rint(np.linspace(0, n_v, min(world, n_v) + 1)).astype(np.int64))
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]


@pytest.mark.parametrize("n_v,world", [(35, 1), (35, 2), (35, 3), (35, 8), (350, 8), (350, 7), (12, 12)])
def test_partition_matches_reference(n_v, world):
    part = make_partition(n_v, world)
    assert part == _ref_partition(n_v, world)
    assert part[0][0] == 0 and part[-1][1] == n_v
    assert all(b > a for a, b in part) and all(part[i][1] == part[i + 1][0] for i in range(world - 1))


def test_partition_against_reference_package():
    par = pytest.importorskip("ecodrive.parallel")
    for n_v, w in [(35, 2), (35, 8), (350, 8), (12, 5)]:
        b = par.make_partition(n_v, 26, 40, w).bounds // (26 * 40)
        assert make_partition(n_v, w) == [(int(x), int(y)) for x, y in zip(b[:-1], b[1:])]


def test_partition_rejects_more_ranks_than_planes():
    with pytest.raises(ValueError):
        make_partition(4, 5)


def test_slab_solver_fails_loudly_without_device():
    if _abi.lib().eco_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(NativeLibraryError):
        SlabSolver(12, 8, 40, 4, rank=0, world=1)


def _slab_solve_rank(rank, world):
    """Each rank owns make_partition's planes of every level; after a stage
    it contributes only its slab and rebuilds the full level from the
    all-gather (gloo) before the next stage -- the C5 data flow."""
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2104_01284_b200 import (GridSpec, PenaltyConfig, build_context, load_fixture_route,
                                       make_vehicle)
    veh = make_vehicle()
    route, spat = load_fixture_route("short", seed=2)
    ctx = build_context(veh, route, spat, 45, 50.0, grids=GridSpec(n_v=12, n_soc=8, n_t=40),
                        penalty=PenaltyConfig(), gamma=0.5, horizon=6)
    lo, hi = make_partition(ctx.grids.n_v, world)[rank]
    J_next = np.array(ctx.terminal)
    P_slab = []
    for k in range(ctx.horizon - 1, -1, -1):
        J_full, P_full, _ = O.sweep(ctx, k, J_next)
        mine = torch.from_numpy(np.ascontiguousarray(J_full[lo:hi]))
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, mine.numpy()))
        J_next = np.empty_like(J_full)
        for a, b, blk in parts:
            J_next[a:b] = blk
        P_slab.insert(0, P_full[lo:hi])
    res = SlabResult(planes=(lo, hi), P=np.stack(P_slab), J=None)
    P_all = gather_policies(res, ctx.grids.n_v)
    return J_next, P_all


def test_slab_exchange_reproduces_full_solve_gloo():
    from oracle import oracle as O
    from paper_2104_01284_b200 import (GridSpec, PenaltyConfig, build_context, load_fixture_route,
                                       make_vehicle)
    out = run_gloo(_slab_solve_rank, world=2)
    veh = make_vehicle()
    route, spat = load_fixture_route("short", seed=2)
    ctx = build_context(veh, route, spat, 45, 50.0, grids=GridSpec(n_v=12, n_soc=8, n_t=40),
                        penalty=PenaltyConfig(), gamma=0.5, horizon=6)
    J, P = O.solve_context(ctx)
    for J0, _ in out:
        assert np.array_equal(J0, J[0])               # every rank ends with the full level 0
    assert np.array_equal(out[0][1], np.stack(P))     # policies assembled on rank 0
    assert out[1][1] is None
