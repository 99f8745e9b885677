"""Summarise ECO_DEBUG_STAGE per-CTA timelines (stderr of tools/debug_stage.py)."""
import re, statistics as S, sys
txt = open(sys.argv[1]).read().split("stage k=")
for blk in txt[-3:]:
    lines = [l.split() for l in blk.splitlines() if l.strip().startswith("cta")]
    if not lines:
        continue
    st = [float(r[9]) for r in lines]; sg = [float(r[11]) for r in lines]
    lp = [float(r[13]) for r in lines]; en = [float(r[15]) for r in lines]
    span = max(en) - min(st)
    print(f"stage {blk.split()[0]} ctas={len(lines)} span={span:.2f}us late-starts(>2us)={sum(1 for x in st if x > 2)}")
    print(f"  start med {S.median(st):.2f} max {max(st):.2f} | staging med {S.median([b - a for a, b in zip(st, sg) if b > 0]):.2f}"
          f" | loop med {S.median([b - a for a, b in zip(sg, lp) if a > 0]):.2f} max {max(b - a for a, b in zip(sg, lp) if a > 0):.2f}"
          f" | merge med {S.median([b - a for a, b in zip(lp, en)]):.2f} | end max {max(en):.2f}")
