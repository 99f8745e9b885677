"""CPU checks of the C4 batch host side: signal-timing packing, scenario
sharding, argument validation and loud failure without a device."""

import numpy as np
import pytest

from paper_2104_01284_b200 import GridSpec, NativeLibraryError, PenaltyConfig
from paper_2104_01284_b200 import _abi
from paper_2104_01284_b200.batch import BatchSolver, shard
from paper_2104_01284_b200.fixtures import bench_schedule, make_route_urban
from paper_2104_01284_b200.route import load_route


def test_signal_timings_match_route_pack():
    routes = [load_route(make_route_urban(seed=i)) for i in range(5)]
    base = routes[0][0]
    tim = _abi.signal_timings(base, [sp for _, sp in routes])
    nodes = sorted(base.traffic_lights)
    assert tim.shape == (5, len(nodes)) and tim.dtype.itemsize == 152
    for i, (route, spat) in enumerate(routes):
        rp = _abi.RoutePack(route, spat)
        for j, node in enumerate(nodes):
            assert tim[i, j]["cycle"] == rp.cycle[node] and tim[i, j]["offset"] == rp.offset[node]
            assert tim[i, j]["nwin"] == rp.nwin[node]
            assert np.array_equal(tim[i, j]["win"], rp.win[node])


def test_c4_geometry_is_seed_independent():
    """The batch shares one route geometry: seeds only change signal phasing."""
    a, _ = load_route(make_route_urban(seed=0))
    for seed in (1, 17, 4095):
        b, _ = load_route(make_route_urban(seed=seed))
        assert np.array_equal(a.v_max, b.v_max) and np.array_equal(a.grade, b.grade)
        assert np.array_equal(a.node_kinds(), b.node_kinds())
        assert a.traffic_lights == b.traffic_lights and a.stop_signs == b.stop_signs


@pytest.mark.parametrize("n,world", [(4096, 8), (4096, 3), (5, 8), (0, 2), (7, 1)])
def test_shard_covers_each_scenario_once(n, world):
    seen = []
    for r in range(world):
        blk = shard(n, r, world)
        assert blk.step == 1
        seen.extend(blk)
    assert seen == list(range(n))
    sizes = [len(shard(n, r, world)) for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_shard_rejects_bad_rank():
    with pytest.raises(ValueError):
        shard(10, 2, 2)


def test_batch_fails_loudly_without_device(vehicle):
    if _abi.lib().eco_device_count() > 0:
        pytest.skip("a GPU is visible")
    route, _ = load_route(make_route_urban(seed=0))
    with pytest.raises(NativeLibraryError):
        BatchSolver(vehicle, route, grids=GridSpec(n_v=4, n_soc=3, n_t=5), penalty=PenaltyConfig())


def test_batch_argument_validation(vehicle):
    route, _ = load_route(make_route_urban(seed=0))
    with pytest.raises(ValueError):
        BatchSolver(vehicle, route, gamma=1.5)
    with pytest.raises(ValueError):
        BatchSolver(vehicle, route, horizon=0)
    with pytest.raises(ValueError, match="unknown backend"):
        BatchSolver(vehicle, route, backend="cpu")
    sched = bench_schedule(route, 20, 3, seed=1)
    assert all(0 <= s <= route.node_count - 21 for s, _ in sched)
