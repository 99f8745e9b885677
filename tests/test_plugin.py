"""The drop-in shim inside the reference package (build container only:
the reference is not present on the GPU box, where this module skips)."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def ecodrive():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_eco")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import ecodrive as E
    from paper_2104_01284_b200 import plugin
    plugin.install()
    yield E
    plugin.uninstall()


def test_reference_backends_still_forwarded(ecodrive):
    import ecodrive.dp as rdp
    from ecodrive.fixtures import load_fixture_route, make_vehicle
    route, spat = load_fixture_route("short", seed=2)
    ctx = rdp.build_context(make_vehicle(), route, spat, 45, 50.0, grids=rdp.GridSpec(n_v=4, n_soc=3, n_t=6),
                            penalty=rdp.PenaltyConfig(), gamma=0.5, horizon=2)
    res = rdp.solve_horizon(ctx, backend="serial")
    assert res.backend == "serial" and len(res.tables) == 3
    with pytest.raises(ValueError):
        rdp.solve_horizon(ctx, backend="nope")


def test_b200_names_route_to_the_device_library(ecodrive):
    import ecodrive.dp as rdp
    import ecodrive.mpc as rmpc
    from ecodrive.fixtures import load_fixture_route, make_vehicle
    from paper_2104_01284_b200 import NativeLibraryError, _abi
    assert rmpc.solve_horizon is rdp.solve_horizon is ecodrive.solve_horizon
    route, spat = load_fixture_route("short", seed=2)
    ctx = rdp.build_context(make_vehicle(), route, spat, 45, 50.0, grids=rdp.GridSpec(n_v=4, n_soc=3, n_t=6),
                            penalty=rdp.PenaltyConfig(), gamma=0.5, horizon=2)
    if _abi.lib().eco_device_count() == 0:
        with pytest.raises(NativeLibraryError, match="no CUDA device"):
            rdp.solve_horizon(ctx, backend="b200")
    else:
        res = rdp.solve_horizon(ctx, backend="b200-fp64")
        ref = rdp.solve_horizon(ctx, backend="serial")
        assert isinstance(res, rdp.SolveResult)
        for a, b in zip(res.tables, ref.tables):
            assert np.array_equal(a.values, b.values)
