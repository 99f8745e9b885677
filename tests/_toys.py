"""Seeded exact-arithmetic toy instances and a brute-force enumerator.

Test infrastructure restating the reference's tests/enum_oracle.py
(random_toy :137-204, enumerate_costs :58-134).  Toys are built so every
transition lands on grid nodes and every cost is a dyadic rational, so the
enumerated optimum, the reference sweeps, the C oracle and the CUDA kernels
(fp64 and fp32 alike) must agree with tolerance 0.  The generated tables are
checked against the reference-produced tests/golden/toys.npz.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2104_01284_b200.dp import DEFAULT_J_INF, ToyInstance, make_toy_pack

R0, VOC, CNOM, DTG = 0.25, 2.0, 32.0, 2.0
PBAT_CHOICES = (-12.0, 0.0, 4.0)


def random_toy(seed: int, *, horizon=None) -> ToyInstance:
    rng = np.random.default_rng(seed)
    nv = int(rng.integers(2, 6))
    nx = int(rng.integers(2, 5))
    nt = int(rng.integers(3, 7))
    nte = int(rng.integers(1, 4))
    ntb = int(rng.integers(1, 4))
    if horizon is None:
        horizon = int(rng.integers(1, 4))
    t_axis = DTG * np.arange(nt)
    kinds, stage1, green, dep_ok, t_dep, wait = [], [], [], [], [], []
    for _ in range(horizon):
        kind = int(rng.choice([0, 1, 2], p=[0.55, 0.30, 0.15]))
        shape = (nv, nte, ntb)
        stage1.append({
            "ok": (rng.random(shape) < 0.85).astype(np.uint8),
            "v2": rng.integers(0, nv, size=shape).astype(np.float64),
            "dt": rng.choice([2.0, 4.0], size=shape),
            "pbat": rng.choice(np.asarray(PBAT_CHOICES), size=shape),
            "c1": rng.integers(0, 16, size=shape) / 8.0,
        })
        green.append((rng.random(nt) < 0.8).astype(np.uint8))
        if kind == 1:
            dep = (rng.random(nt) < 0.7).astype(np.uint8)
            w = np.zeros(nt)
            td = t_axis.copy()
            for z in range(nt):
                if dep[z] and rng.random() < 0.35:
                    jump = float(rng.choice([2.0, 4.0]))
                    w[z] = jump
                    td[z] = t_axis[z] + jump
        elif kind == 2:
            dep, w, td = np.ones(nt, dtype=np.uint8), np.full(nt, 2.0), t_axis + 2.0
        else:
            dep, w, td = np.ones(nt, dtype=np.uint8), np.zeros(nt), t_axis.copy()
        kinds.append(kind)
        dep_ok.append(dep)
        t_dep.append(td)
        wait.append(w)
    terminal = rng.integers(0, 12, size=(nv, nx, nt)) / 4.0
    blocked = rng.random((nv, nx, nt)) < 0.15
    terminal = np.where(blocked, DEFAULT_J_INF, terminal)
    return ToyInstance(v_axis=np.arange(nv, dtype=np.float64), soc_axis=0.25 * np.arange(nx), t_axis=t_axis,
                       n_actions_eng=nte, n_actions_bsg=ntb, horizon=horizon,
                       pack=make_toy_pack(r0=R0, c_nom=CNOM, voc=VOC), src_kinds=kinds, stage1=stage1,
                       arr_green=green, dep_ok=dep_ok, t_dep=t_dep, wait=wait, terminal=terminal, gamma=0.5,
                       j_inf=DEFAULT_J_INF)


def _current(p):
    if p == 0.0:
        return 0.0, True
    disc = VOC * VOC - 4.0 * R0 * p
    if disc < 0.0:
        return 0.0, False
    return (VOC - math.sqrt(disc)) / (2.0 * R0), True


def _node(x, x0, dx, n):
    f = (x - x0) / dx
    i = math.floor(f)
    w = f - i
    if w > 1.0 - 1e-12:
        i, w = i + 1, 0.0
    assert w < 1e-12, f"toy transition off-node: {x!r}"
    return int(i) if 0 <= i <= n - 1 else None


def enumerate_costs(toy: ToyInstance) -> np.ndarray:
    """Minimum total cost over every action sequence, per start state."""
    nv, nx, nt = toy.v_axis.shape[0], toy.soc_axis.shape[0], toy.t_axis.shape[0]
    v0 = float(toy.v_axis[0])
    dv = (float(toy.v_axis[-1]) - v0) / (nv - 1)
    x0 = float(toy.soc_axis[0])
    dx = (float(toy.soc_axis[-1]) - x0) / (nx - 1)
    t0 = float(toy.t_axis[0])

    def tails(k, iv, jx, z):
        if k == toy.horizon:
            val = float(toy.terminal[iv, jx, z])
            return [] if val >= toy.j_inf else [val]
        v = float(toy.v_axis[iv])
        if int(toy.src_kinds[k]) == 2 and v > 0.0:
            return []
        t = toy.stage1[k]
        out = []
        for a1 in range(toy.n_actions_eng):
            for a2 in range(toy.n_actions_bsg):
                if not t["ok"][iv, a1, a2]:
                    continue
                cur, okb = _current(float(t["pbat"][iv, a1, a2]))
                if not okb:
                    continue
                dt = float(t["dt"][iv, a1, a2])
                jx2 = _node(float(toy.soc_axis[jx]) - dt * cur / CNOM, x0, dx, nx)
                iv2 = _node(float(t["v2"][iv, a1, a2]), v0, dv, nv)
                if jx2 is None or iv2 is None:
                    continue
                if v > 0.0:
                    hold, z2 = 0.0, z + round(dt / DTG)
                    if z2 > nt - 1:
                        continue
                else:
                    if not toy.dep_ok[k][z]:
                        continue
                    hold = float(toy.wait[k][z])
                    if hold > 0.0:
                        z2 = _node(float(toy.t_dep[k][z]) + dt, t0, DTG, nt)
                        if z2 is None:
                            continue
                    else:
                        z2 = z + round(dt / DTG)
                        if z2 > nt - 1:
                            continue
                if float(t["v2"][iv, a1, a2]) > 0.0 and not toy.arr_green[k][z2]:
                    continue
                inc = float(t["c1"][iv, a1, a2]) + (1.0 - toy.gamma) * hold
                out.extend(inc + tv for tv in tails(k + 1, iv2, jx2, z2))
        return out

    J0 = np.full((nv, nx, nt), toy.j_inf)
    for idx in np.ndindex(nv, nx, nt):
        vals = tails(0, *idx)
        if vals:
            J0[idx] = min(vals)
    return J0
