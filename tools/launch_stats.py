"""Per-kernel duration stats from an ncu --csv launch list."""
import collections, csv, sys
lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.reader(lines))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
d = collections.defaultdict(list)
for r in rows[1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]])
    v *= {"nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(r[ix["Metric Unit"]], 1.0)
    d[r[ix["Kernel Name"]].split("(")[0][:60]].append(v)
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} n={len(v):4d} mean={sum(v)/len(v):8.2f}us min={min(v):8.2f} max={max(v):8.2f} share={sum(v)/tot:6.1%}")
