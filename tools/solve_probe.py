"""Wall-time breakdown of one solve_horizon call at the C2 grid (marshal /
ABI call / device time / table objects)."""

import time

import numpy as np

from paper_2104_01284_b200 import GridSpec, PenaltyConfig, build_context, load_fixture_route, make_vehicle
from paper_2104_01284_b200 import _abi, dp
from paper_2104_01284_b200.fixtures import bench_schedule
import ctypes as C

veh = make_vehicle()
route, spat = load_fixture_route("urban", seed=0)
sched = bench_schedule(route, 20, 30, 0)
ctxs = [build_context(veh, route, spat, s, t, grids=GridSpec(), penalty=PenaltyConfig(), gamma=0.5, horizon=20)
        for s, t in sched]
for backend in ("b200", "b200-fp64"):
    rows = []
    for i, ctx in enumerate(ctxs):
        t0 = time.perf_counter()
        m = dp._Marshal(ctx, ctx.steps)
        term = dp._f64(ctx.terminal)
        g, H = ctx.grids, ctx.horizon
        t1 = time.perf_counter()
        J = _abi.PINNED.array((H + 1, g.n_v, g.n_soc, g.n_t), np.float64)
        P = _abi.PINNED.array((H, g.n_v, g.n_soc, g.n_t), np.int32)
        t2 = time.perf_counter()
        st = _abi.EcoStats()
        _abi.check(_abi.lib().eco_solve_horizon(C.byref(m.plant), C.byref(m.prob), m.plans, H,
                                                _abi.ptr(term, C.c_double), _abi.ptr(J, C.c_double),
                                                _abi.ptr(P, C.c_int32), dp.precision_of(backend), 0, C.byref(st)),
                   "x")
        t3 = time.perf_counter()
        res = dp.solve_horizon(ctx, backend=backend)
        t4 = time.perf_counter()
        if i >= 5:
            rows.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, st.device_ms, (t4 - t3) * 1e3))
    a = np.array(rows)
    print(backend, "marshal %.3f  alloc %.3f  abi %.3f  device %.3f  full solve_horizon %.3f ms" % tuple(a.mean(0)))
