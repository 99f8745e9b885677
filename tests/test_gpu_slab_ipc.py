"""The C5 P2P slab path as shipped -- CUDA IPC replicas exchanged through the
process group, the stage kernel's PEERS epilogue storing each rank's slab
into the other processes' replicas, the local copy-1 rebuild -- with two
rank processes sharing the ONE GPU of this lease.  The only substitution is
the stage barrier: a stream sync + a gloo barrier on the host
(SlabSolver(host_barrier=True)) instead of the GPU-side spin barrier, because
kernels that wait on one another must not run as separate launches on one
GPU.  Every rank's replica of every level and the assembled policies equal
the unpartitioned solve bitwise (test_parallel.py:164-171)."""

import numpy as np
import pytest

from _dist import run_gloo

pytestmark = pytest.mark.gpu


GRIDS = {
    "c2": dict(),                                            # narrow tiles (the default grid)
    "fine": dict(n_v=20, n_soc=30, n_t=400, dt=0.2),         # row-block kernel, compiled n_t = 400
    "wide": dict(n_v=20, n_soc=30, n_t=256, dt=0.3),         # row-block kernel, runtime n_t
}


def _ctx(grid="c2"):
    from paper_2104_01284_b200 import GridSpec, PenaltyConfig, build_context, load_fixture_route, make_vehicle
    route, spat = load_fixture_route("urban", seed=0)
    h = 20 if grid == "c2" else 4
    return build_context(make_vehicle(), route, spat, 60, 30.0, grids=GridSpec(**GRIDS[grid]),
                         penalty=PenaltyConfig(), gamma=0.5, horizon=h)


def _rank(rank, world, backend, grid="c2"):
    import torch
    torch.cuda.set_device(0)                     # both ranks on the lease's one GPU
    from paper_2104_01284_b200.slab import SlabSolver, gather_policies
    ctx = _ctx(grid)
    g = ctx.grids
    with SlabSolver(g.n_v, g.n_soc, g.n_t, ctx.horizon, backend=backend, exchange="p2p", host_barrier=True) as ss:
        out = []
        for _ in range(2):                       # a second solve reuses the connected replicas
            res = ss.solve(ctx, return_J=True)
            P = gather_policies(res, g.n_v)
            out.append((res.J, P, res.planes, res.stats["stages"]))
    return out


@pytest.mark.parametrize("backend", ["b200-fp64", "b200"])
def test_p2p_slab_two_processes_one_gpu(backend):
    from paper_2104_01284_b200 import solve_horizon
    outs = run_gloo(_rank, world=2, args=(backend,), timeout=600)
    ref = solve_horizon(_ctx(), backend=backend)
    assert outs[0][0][2] == (0, 18) and outs[1][0][2] == (18, 35)
    for rank, runs in enumerate(outs):
        for J, P, planes, stages in runs:
            assert stages == 20
            for k in range(21):
                assert np.array_equal(J[k], ref.tables[k].values), (rank, k)
            if rank == 0:
                for k in range(20):
                    assert np.array_equal(P[k], ref.policies[k].values), k
            else:
                assert P is None


@pytest.mark.parametrize("grid", ["fine", "wide"])
@pytest.mark.parametrize("backend", ["b200-fp64", "b200"])
def test_p2p_slab_two_processes_wide_rows(backend, grid):
    """The row-block kernel's PEERS epilogue (the compiled n_t = 400 and the
    runtime-n_t instantiations) between two rank processes: every replica
    and the assembled policies equal the unpartitioned solve bitwise."""
    from paper_2104_01284_b200 import solve_horizon
    outs = run_gloo(_rank, world=2, args=(backend, grid), timeout=600)
    ctx = _ctx(grid)
    ref = solve_horizon(ctx, backend=backend)
    H = ctx.horizon
    assert outs[0][0][2] == (0, 10) and outs[1][0][2] == (10, 20)
    for rank, runs in enumerate(outs):
        for J, P, planes, stages in runs:
            assert stages == H
            for k in range(H + 1):
                assert np.array_equal(J[k], ref.tables[k].values), (rank, k)
            if rank == 0:
                for k in range(H):
                    assert np.array_equal(P[k], ref.policies[k].values), k
