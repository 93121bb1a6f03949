"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch counts, total device time and share (cold-cache, serialised
timings: compare shares, not absolutes)."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    unit = r["Metric Unit"]
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
             "msecond": 1.0, "s": 1e3, "second": 1e3}[unit]
    rows.append((name, v * scale))
agg = defaultdict(lambda: [0, 0.0])
for n, ms in rows:
    agg[n][0] += 1
    agg[n][1] += ms
tot = sum(v[1] for v in agg.values())
print(f"launches: {len(rows)}, total device time {tot:.1f} ms")
print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for n, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n[:60]:60s} {c:8d} {ms:10.2f} {100 * ms / tot:6.2f}%")
