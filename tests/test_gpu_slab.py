"""C5 slab decomposition on the device with several ranks.

The reference's contract is that tables do not depend on the worker count
(test_parallel.py:164-171, test_dp_oracle.py:48-56; partition
parallel.py:87-101).  This lease has one GPU, and ranks whose kernels wait on
one another may not run as separate launches on one GPU, so the G ranks are
emulated in one launch per stage (eco_slab_emulate): each rank reads its own
replica of J_{k+1}, writes its slab, stores it into every peer replica
through the PEERS epilogue (copy 0 only) and rebuilds its shifted copy 1
locally -- the data path of the multi-GPU exchange.  Every replica of every
level must equal the unpartitioned solve bitwise, for G = 1..8."""

import numpy as np
import pytest

from paper_2104_01284_b200 import GridSpec, PenaltyConfig, build_context, solve_horizon
from paper_2104_01284_b200.slab import emulate_slabs, make_partition

pytestmark = pytest.mark.gpu

PEN = PenaltyConfig()


@pytest.fixture(scope="module")
def c2_ctx(vehicle, urban_route):
    route, spat = urban_route
    return build_context(vehicle, route, spat, 60, 30.0, grids=GridSpec(), penalty=PEN, gamma=0.5, horizon=20)


@pytest.mark.parametrize("backend", ["b200-fp64", "b200"])
@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_slab_ranks_invariant_c2(c2_ctx, backend, world):
    ref = solve_horizon(c2_ctx, backend=backend)
    J, P, st = emulate_slabs(c2_ctx, world, backend)
    assert J.shape[0] == world and st["stages"] == 20
    for g in range(world):
        for k in range(21):
            assert np.array_equal(J[g, k], ref.tables[k].values), (g, k)
    for k in range(20):
        assert np.array_equal(P[k], ref.policies[k].values), k


@pytest.mark.parametrize("world", [2, 4, 7])
def test_slab_ranks_invariant_wide_rows(vehicle, urban_route, world):
    """The wide-row kernel (n_t >= 128, the C3 / C5 path) with the exchange."""
    route, spat = urban_route
    ctx = build_context(vehicle, route, spat, 150, 40.0, grids=GridSpec(n_v=28, n_soc=12, n_t=160, dt=0.5),
                        penalty=PEN, gamma=0.5, horizon=4)
    ref = solve_horizon(ctx, backend="b200-fp64")
    J, P, _ = emulate_slabs(ctx, world, "b200-fp64")
    for g in range(world):
        for k in range(5):
            assert np.array_equal(J[g, k], ref.tables[k].values), (g, k)
    for k in range(4):
        assert np.array_equal(P[k], ref.policies[k].values), k


def test_slab_emulation_rejects_bad_partitions(c2_ctx):
    with pytest.raises(ValueError):
        emulate_slabs(c2_ctx, 9, "b200")              # > 8 emulated ranks
    with pytest.raises(ValueError):
        make_partition(35, 36)


def test_slab_ranks_invariant_c3_shape(vehicle, urban_route):
    """The row-block wide kernel's PEERS epilogue at the real C3 grid
    (350 x 260 x 400): 4 emulated ranks, 3 stages, every replica bitwise
    equal to the unpartitioned fp64 solve."""
    route, spat = urban_route
    ctx = build_context(vehicle, route, spat, 60, 30.0, grids=GridSpec(n_v=350, n_soc=260, n_t=400, dt=0.2),
                        penalty=PEN, gamma=0.5, horizon=3)
    ref = solve_horizon(ctx, backend="b200-fp64")
    J, P, _ = emulate_slabs(ctx, 4, "b200-fp64")
    for g in range(4):
        for k in range(4):
            assert np.array_equal(J[g, k], ref.tables[k].values), (g, k)
    for k in range(3):
        assert np.array_equal(P[k], ref.policies[k].values), k
