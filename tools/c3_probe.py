"""C3 fine-grid probe: urban route, s=60, t=30, GridSpec(350, 260, 400, dt=0.2).

Times `solve_stacks` on the device (fp32 and optionally fp64) for horizon H and,
with --check H_CHECK, compares the first H_CHECK stages against the C oracle
(OpenMP, all host threads).  Diagnostic tool, not a test."""

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2104_01284_b200 import GridSpec, PenaltyConfig, build_context, load_fixture_route, make_vehicle  # noqa
from paper_2104_01284_b200.dp import solve_stacks  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--horizon", type=int, default=20)
ap.add_argument("--check", type=int, default=0, help="oracle-check a context of this horizon")
ap.add_argument("--fp64", action="store_true")
ap.add_argument("--nv", type=int, default=350)
ap.add_argument("--nsoc", type=int, default=260)
ap.add_argument("--nt", type=int, default=400)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--no-count", action="store_true")
args = ap.parse_args()

veh = make_vehicle()
route, spat = load_fixture_route("urban", seed=0)
grids = GridSpec(n_v=args.nv, n_soc=args.nsoc, n_t=args.nt, dt=0.2)
pen = PenaltyConfig()


def run(H, backend, count=False):
    ctx = build_context(veh, route, spat, 60, 30.0, grids=grids, penalty=pen, gamma=0.5, horizon=H)
    out = None
    for r in range(args.reps):
        t0 = time.perf_counter()
        out = solve_stacks(ctx, backend, count_live=count and r == 0)
        wall = time.perf_counter() - t0
        st = out[2]
        print(f"{backend} H={H} rep={r} wall={wall * 1e3:.1f} ms device={st['device_ms']:.2f} ms "
              f"sweep={st['dominant_ms']:.2f} ms live={st['live_updates']} dense={st['dense_updates']}", flush=True)
    return ctx, out


run(args.horizon, "b200", count=not args.no_count)
if args.fp64:
    run(args.horizon, "b200-fp64")
if args.check:
    from oracle import oracle as O
    H = args.check
    ctx, (J32, P32, _) = run(H, "b200")
    _, (J64, P64, _) = run(H, "b200-fp64")
    t0 = time.perf_counter()
    Jo, Po = O.solve_context(ctx, parallel=True)
    print(f"oracle H={H}: {time.perf_counter() - t0:.1f} s on {O.threads_available()} threads", flush=True)
    for k in range(H):
        eq = np.array_equal(J64[k], Jo[k]) and np.array_equal(P64[k], Po[k])
        f32, f64 = J32[k] < pen.j_inf, Jo[k] < pen.j_inf
        both = f32 & f64
        rel = np.abs(J32[k][both] - Jo[k][both]) / np.maximum(1.0, np.abs(Jo[k][both]))
        pol = float(np.mean(P32[k][both] == Po[k][both]))
        print(f"k={k} fp64 bitwise={eq} fp32 mask={np.mean(f32 == f64):.6f} "
              f"rel_p999={np.quantile(rel, 0.999):.2e} rel_max={rel.max():.2e} argmin={pol:.6f}", flush=True)
