"""The reference package's OWN Table-I harness (ecodrive.bench.run_bench,
bench.py:97-150) on this host, with the device backends registered through
plugin.install(): b200 / b200-fp64 next to the reference's numba parallel
(all host cores) and serial backends on identical contexts (C2 grid, urban
route, bench_schedule seed 0); plus one C3 solve by the reference's parallel
backend (the SURVEY's 145.8 s-on-8-cores measurement, repeated here).

    python tools/reference_table1.py [reps] [out.txt]

Needs the reference importable: /root/reference/pkg/src or baseline/_ref."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
for cand in ("/root/reference/pkg/src", str(ROOT / "baseline" / "_ref")):
    if os.path.isdir(os.path.join(cand, "ecodrive")):
        sys.path.insert(0, cand)
        break
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_eco")
os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count()))

import ecodrive  # noqa: E402
from ecodrive.bench import run_bench  # noqa: E402
from ecodrive.dp import GridSpec, PenaltyConfig, build_context  # noqa: E402
from ecodrive.fixtures import load_fixture_route, make_vehicle  # noqa: E402

from paper_2104_01284_b200 import plugin  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
out = Path(sys.argv[2]) if len(sys.argv) > 2 else None
plugin.install()
solve_horizon = ecodrive.solve_horizon      # the patched name (bound after install)
veh = make_vehicle()
route, spat = load_fixture_route("urban", seed=0)
workers = os.cpu_count()
rep = run_bench(veh, route, spat, grids=GridSpec(), horizon=20, backends=("b200", "b200-fp64", "parallel", "serial"),
                workers=workers, reps=reps, warmup=2)
lines = [f"ecodrive.bench.run_bench, C2 grid, urban, H=20, reps={reps}, parallel workers={workers}", rep.table()]
ctx = build_context(veh, route, spat, 60, 30.0, grids=GridSpec(n_v=350, n_soc=260, n_t=400, dt=0.2),
                    penalty=PenaltyConfig(), gamma=0.5, horizon=20)
solve_horizon(ctx, backend="b200")
t0 = time.perf_counter()
solve_horizon(ctx, backend="b200")
t_gpu = time.perf_counter() - t0
t0 = time.perf_counter()
solve_horizon(ctx, backend="parallel", workers=workers)
t_ref = time.perf_counter() - t0
# the per-stage plug-in point alone (the reference's own Python stage loop
# calling the patched backward_step, dp.py:446-450): every stage ships its
# f64 J_next in and J / P out
import ecodrive.dp as rdp  # noqa: E402
J = ctx.terminal
for k in range(ctx.horizon - 1, ctx.horizon - 3, -1):     # warm-up: the pinned output pool fills
    J, _ = rdp.backward_step(ctx, k, J, backend="b200")
t0 = time.perf_counter()
for k in range(ctx.horizon - 3, ctx.horizon - 7, -1):
    J, _ = rdp.backward_step(ctx, k, J, backend="b200")
t_step = (time.perf_counter() - t0) / 4
lines.append(f"C3 (350x260x400, dt=0.2, urban s=60 t=30, H=20) through ecodrive.solve_horizon: "
             f"backend=b200 {t_gpu * 1e3:.1f} ms (tables on the host), backend=parallel ({workers} workers) "
             f"{t_ref:.1f} s -> {t_ref / t_gpu:.0f}x; one stage through ecodrive.dp.backward_step(backend=b200) "
             f"{t_step * 1e3:.0f} ms (f64 tables in and out per stage)")
text = "\n".join(lines)
print(text)
if out:
    out.write_text(text + "\n")
