"""Drop-in registration of the B200 backends inside the reference package.

The reference dispatches on a backend *string* (``backward_step``
dp.py:365-404: serial / parallel / ValueError) and binds ``solve_horizon`` by
name in three modules (``ecodrive.dp``, ``ecodrive.mpc`` mpc.py:25-32,
``ecodrive.bench`` bench.py:25).  ``install()`` wraps those names so that
``backend="b200"`` / ``"b200-fp64"`` run on the sm_100a library while every
other backend string is forwarded untouched to the original functions::

    import ecodrive
    from paper_2104_01284_b200 import plugin
    plugin.install()
    res = ecodrive.solve_horizon(ctx, backend="b200")          # GPU
    mpc = ecodrive.EcoDrivingMPC(vehicle, backend="b200")      # GPU solves,
    traj = ecodrive.simulate_closed_loop(route, spat, mpc.fit(route, spat))

Results come back as the reference's own ``CostToGoTable`` / ``PolicyTable``
/ ``SolveResult`` objects, and an infeasible start raises the reference's
``StartStateInfeasibleError``, so callers cannot tell the backends apart.
"""

from __future__ import annotations

import math
import time

from .dp import BACKENDS, solve_stacks

_INSTALLED = {}


def _ref():
    import ecodrive.bench as rbench
    import ecodrive.dp as rdp
    import ecodrive.errors as rerr
    import ecodrive.mpc as rmpc
    return rdp, rmpc, rbench, rerr


def install(names=tuple(BACKENDS)) -> None:
    """Register the B200 backend names in an importable ``ecodrive``."""
    rdp, rmpc, rbench, rerr = _ref()
    if _INSTALLED:
        return
    orig_step, orig_solve = rdp.backward_step, rdp.solve_horizon
    _INSTALLED.update(backward_step=orig_step, solve_horizon=orig_solve,
                      mpc_solve=rmpc.solve_horizon, bench_solve=rbench.solve_horizon)

    def backward_step(ctx, k, J_next, *, backend="serial", workers=8, perturb_ties=False):
        if backend not in names:
            return orig_step(ctx, k, J_next, backend=backend, workers=workers, perturb_ties=perturb_ties)
        from . import dp as mdp
        return mdp.backward_step(ctx, k, J_next, backend=backend, perturb_ties=perturb_ties)

    def solve_horizon(ctx, x_start=None, *, backend="serial", workers=8, perturb_ties=False):
        if backend not in names:
            return orig_solve(ctx, x_start, backend=backend, workers=workers, perturb_ties=perturb_ties)
        t0 = time.perf_counter()
        J, P, _ = solve_stacks(ctx, backend, perturb_ties=perturb_ties)
        wall = time.perf_counter() - t0
        j_inf = ctx.penalty.j_inf
        tables = [rdp.CostToGoTable(values=J[k], v_axis=ctx.v_axes[k], soc_axis=ctx.soc_axis,
                                    t_axis=ctx.t_axis, j_inf=j_inf) for k in range(ctx.horizon + 1)]
        policies = [rdp.PolicyTable(values=P[k], te_axis=ctx.te_axis, tb_axis=ctx.tb_axis)
                    for k in range(ctx.horizon)]
        cost0 = math.nan
        if x_start is not None:
            cost0 = tables[0].interpolate(x_start.v, x_start.soc, x_start.t)
            if cost0 >= j_inf:
                raise rerr.StartStateInfeasibleError(
                    f"no feasible continuation from node {ctx.s} at v={x_start.v:.2f} m/s, "
                    f"soc={x_start.soc:.3f}, t={x_start.t:.1f} s")
        return rdp.SolveResult(s=ctx.s, horizon=ctx.horizon, t_start=ctx.t_start, backend=backend,
                               cost_at_start=cost0, tables=tables, policies=policies, wall_time_s=wall)

    rdp.backward_step = backward_step
    rdp.solve_horizon = solve_horizon
    rmpc.solve_horizon = solve_horizon
    rbench.solve_horizon = solve_horizon
    import ecodrive
    ecodrive.solve_horizon = solve_horizon


def uninstall() -> None:
    if not _INSTALLED:
        return
    rdp, rmpc, rbench, _ = _ref()
    rdp.backward_step = _INSTALLED["backward_step"]
    rdp.solve_horizon = _INSTALLED["solve_horizon"]
    rmpc.solve_horizon = _INSTALLED["mpc_solve"]
    rbench.solve_horizon = _INSTALLED["bench_solve"]
    import ecodrive
    ecodrive.solve_horizon = _INSTALLED["solve_horizon"]
    _INSTALLED.clear()
