"""Dev: per-launch durations (ms, launch order) of selected kernels from an
`ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
path, pats = sys.argv[1], sys.argv[2:]
lines = [l for l in open(path) if l.startswith('"')]
series = {p: [] for p in pats}
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[r["Metric Unit"]]
    for p in pats:
        if p in r["Kernel Name"]:
            series[p].append(v)
for p, v in series.items():
    print(p, len(v), "total %.2f" % sum(v))
    print("  " + " ".join("%.2f" % x for x in v))
