"""Per-CTA timeline of one C3 stage (ECO_DEBUG_STAGE=1): where does the time go?
usage: ECO_DEBUG_STAGE=1 python tools/c3_debug.py 2> /tmp/dbg.txt; python tools/c3_debug.py --parse /tmp/dbg.txt"""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
if len(sys.argv) > 2 and sys.argv[1] == "--parse":
    import collections, statistics as S
    blk = open(sys.argv[2]).read().split("stage k=")[-1]
    rows = [l.split() for l in blk.splitlines() if l.strip().startswith("cta")]
    st = [float(r[9]) for r in rows]; sg = [float(r[11]) for r in rows]
    lp = [float(r[13]) for r in rows]; en = [float(r[15]) for r in rows]
    pro = [b - a for a, b in zip(st, sg) if b > 0]; loop = [c - b for b, c in zip(sg, lp) if b > 0]
    mrg = [d - c for c, d in zip(lp, en)]
    if pro:
        print(f"prologue med {S.median(pro):.1f} | loop med {S.median(loop):.1f} max {max(loop):.1f} | merge med {S.median(mrg):.1f}us")
    path = [int(r[5]) for r in rows]; work = [int(r[7]) for r in rows]
    span = max(en) - min(st)
    print(f"ctas={len(rows)} span={span:.1f}us")
    by = collections.defaultdict(list)
    for p, a, b, w in zip(path, st, en, work):
        by[p].append((b - a, w))
    for p, v in sorted(by.items()):
        d = [x for x, _ in v]
        print(f" path {p}: n={len(v)} dur med {S.median(d):.1f} max {max(d):.1f} sum {sum(d):.0f}us work sum {sum(w for _, w in v)}")
    ends = sorted(en)
    for q in (0.5, 0.9, 0.99, 1.0):
        print(f" {q:.0%} of CTAs done by {ends[int(q * (len(ends) - 1))]:.1f}us")
    # busy SM-time vs span
    tot = sum(b - a for a, b in zip(st, en))
    print(f" CTA-time sum {tot:.0f}us = {tot / span:.1f} CTAs resident on average")
    sys.exit()
from paper_2104_01284_b200 import GridSpec, PenaltyConfig, build_context, load_fixture_route, make_vehicle
from paper_2104_01284_b200.dp import solve_stacks
veh = make_vehicle(); route, spat = load_fixture_route("urban", seed=0)
ctx = build_context(veh, route, spat, 60, 30.0, grids=GridSpec(n_v=350, n_soc=260, n_t=400, dt=0.2),
                    penalty=PenaltyConfig(), gamma=0.5, horizon=int(os.environ.get("H", "2")))
solve_stacks(ctx, "b200")
