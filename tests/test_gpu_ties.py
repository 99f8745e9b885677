"""perturb_ties on the device: the reference's negative control for its
backend-diff harness (test_dp_oracle.py:59-76, test_parallel.py:174-179).
Ties go to the highest flat action index (reverse_ties, _kernels.py:630-632,
738-740); costs must not change while tied policy entries flip."""

import numpy as np
import pytest

from _toys import random_toy
from paper_2104_01284_b200 import GridSpec, PenaltyConfig, backward_step, build_context, solve_horizon, solve_toy

pytestmark = pytest.mark.gpu


def _tied_toy():
    toy = random_toy(4, horizon=2)         # seed 4: a 2x3 action grid
    assert toy.n_actions_eng * toy.n_actions_bsg > 1
    for t in toy.stage1:
        t["c1"][:] = 1.0                   # all actions cost the same
        t["ok"][:] = 1
        t["pbat"][:] = 0.0
        t["dt"][:] = 2.0
    toy.terminal[:] = 0.25
    return toy


@pytest.mark.parametrize("backend", ["b200-fp64", "b200"])
def test_perturbed_ties_change_policies_not_costs(backend):
    toy = _tied_toy()
    Ja, Pa = solve_toy(toy, backend=backend)
    Jb, Pb = solve_toy(toy, backend=backend, perturb_ties=True)
    for a, b in zip(Ja, Jb):
        assert np.array_equal(a, b)
    flips = sum(int(np.count_nonzero(a != b)) for a, b in zip(Pa, Pb))
    assert flips > 0, "tie perturbation produced no policy flips"
    # every flip moves from the lowest to the highest tied index
    for a, b in zip(Pa, Pb):
        assert np.all(b[a >= 0] >= a[a >= 0]) and np.array_equal(a < 0, b < 0)


def test_perturbed_ties_all_equal_pick_last_action():
    toy = _tied_toy()
    U = toy.n_actions_eng * toy.n_actions_bsg
    _, P = solve_toy(toy, backend="b200-fp64", perturb_ties=True)
    _, P0 = solve_toy(toy, backend="b200-fp64")
    # where the plain rule picked action 0 of an all-tied set, the perturbed
    # rule picks a higher index (the last feasible one of the tied set)
    assert np.any(P[0][P0[0] == 0] > 0) and P[0].max() <= U - 1


@pytest.mark.parametrize("backend", ["b200-fp64", "b200"])
def test_perturbed_ties_leave_costs_intact_c1(vehicle, short_route, backend):
    route, spat = short_route
    ctx = build_context(vehicle, route, spat, 45, 50.0, grids=GridSpec(n_v=12, n_soc=8, n_t=40),
                        penalty=PenaltyConfig(), gamma=0.5, horizon=20)
    a = solve_horizon(ctx, backend=backend)
    b = solve_horizon(ctx, backend=backend, perturb_ties=True)
    for x, y in zip(a.tables, b.tables):
        assert np.array_equal(x.values, y.values)
    J, P = backward_step(ctx, 19, ctx.terminal, backend=backend, perturb_ties=True)
    assert np.array_equal(J, a.tables[19].values)
    assert np.all((P == b.policies[19].values))


def test_perturbed_ties_wide_rows(vehicle, urban_route):
    """The wide-row kernel (n_t >= 128) honours the flag as well."""
    route, spat = urban_route
    ctx = build_context(vehicle, route, spat, 150, 40.0, grids=GridSpec(n_v=20, n_soc=10, n_t=160, dt=0.5),
                        penalty=PenaltyConfig(), gamma=0.5, horizon=3)
    a = solve_horizon(ctx, backend="b200-fp64")
    b = solve_horizon(ctx, backend="b200-fp64", perturb_ties=True)
    for x, y in zip(a.tables, b.tables):
        assert np.array_equal(x.values, y.values)
    for x, y in zip(a.policies, b.policies):
        assert np.array_equal(x.values < 0, y.values < 0) and np.all(y.values >= x.values)


def test_concurrent_solves_from_two_threads(vehicle, short_route, urban_route):
    """The stateless solvers share one device workspace: calls from two host
    threads (ctypes releases the GIL) serialise on its mutex and return
    uncorrupted tables (advisor finding, round 1)."""
    import threading
    route, spat = short_route
    uroute, uspat = urban_route
    ctx_a = build_context(vehicle, route, spat, 45, 50.0, grids=GridSpec(n_v=12, n_soc=8, n_t=40),
                          penalty=PenaltyConfig(), gamma=0.5, horizon=20)
    ctx_b = build_context(vehicle, uroute, uspat, 60, 30.0, grids=GridSpec(), penalty=PenaltyConfig(), gamma=0.5,
                          horizon=20)
    ref_a = solve_horizon(ctx_a, backend="b200-fp64")
    ref_b = solve_horizon(ctx_b, backend="b200-fp64")
    errors = []

    def worker(ctx, ref):
        try:
            for _ in range(6):
                res = solve_horizon(ctx, backend="b200-fp64")
                for x, y in zip(res.tables, ref.tables):
                    assert np.array_equal(x.values, y.values)
                for x, y in zip(res.policies, ref.policies):
                    assert np.array_equal(x.values, y.values)
        except Exception as exc:         # pragma: no cover - reported below
            errors.append(exc)

    th = [threading.Thread(target=worker, args=(ctx_a, ref_a)), threading.Thread(target=worker, args=(ctx_b, ref_b))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
