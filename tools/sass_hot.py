"""Dev: hottest SASS instructions of an `ncu --page source --print-source sass --csv` dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    data.append(r)
S = ix["Warp Stall Sampling (All Samples)"]
tot = sum(float(r[S]) for r in data)
print("total samples", tot, "instructions", len(data))
wf = sum(float(r[ix["L1 Wavefronts Shared"]] or 0) for r in data)
wfi = sum(float(r[ix["L1 Wavefronts Shared Ideal"]] or 0) for r in data)
print(f"shared wavefronts {wf:.3e} ideal {wfi:.3e}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
order = sorted(range(len(data)), key=lambda i: -float(data[i][S]))
for i in sorted(order[:n]):
    r = data[i]
    print(f"{i:5d} {100 * float(r[S]) / tot:5.1f}% ex={r[ix['Instructions Executed']]:>9s} "
          f"wf={r[ix['L1 Wavefronts Shared']]:>9s}/{r[ix['L1 Wavefronts Shared Ideal']]:>9s} "
          f"{r[ix['Source']].strip()[:70]}")
