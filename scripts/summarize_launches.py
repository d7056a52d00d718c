"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv
import re
import sys
from collections import defaultdict

src, title = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
rows = []
with open(src) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    name = re.sub(r"\(.*\)$", "", name)            # drop the argument list
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\s+", " ", name)
    unit = r["Metric Unit"]
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    rows.append((name, v * scale))
tot = sum(v for _, v in rows)
agg = defaultdict(lambda: [0.0, 0])
for n, v in rows:
    agg[n][0] += v
    agg[n][1] += 1
print(f"# {title}")
print(f"# {len(rows)} launches, total kernel time {tot:.1f} ms (cold-cache, serialised by ncu)")
for n, (v, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{v:11.3f} ms {100 * v / tot:5.1f}%  x {c:5d}  {n}")
