"""Dev: per-CUDA-source-line stall samples from `ncu --page source --print-source cuda,sass --csv`."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
cur = None
hdr = None
agg = defaultdict(lambda: [0.0, 0.0, ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 5:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    si = 4  # first metric column after Line No, Source, Address, Source
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    a = agg[(cur, ln)]
    a[0] += v
    wf = r[hdr.get("L1 Wavefronts Shared", 0)] if "L1 Wavefronts Shared" in hdr else "0"
    try:
        a[1] += float(wf or 0)
    except ValueError:
        pass
    a[2] = r[1][:90]
tot = sum(v[0] for v in agg.values())
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for (f, ln), (v, wf, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100 * v / tot:5.1f}% {f}:{ln:<5d} wf={wf:.2e} {src.strip()}")
