# Dev A/B: per-kernel durations of one warm + one refresh iteration of C2 with
# extra nvcc flags (rebuilds the library on the box; never committed results).
mkdir -p gpurun_out
for v in "" "$@"; do
  echo "== flags: $v" >> gpurun_out/ab_dev.log
  GLR_NVCC_EXTRA="$v" python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv python tools/ncu_window.py C2 2>/dev/null > /tmp/ab.csv
  python - >> gpurun_out/ab_dev.log <<'PY'
import csv
rows=[r for r in csv.reader(open('/tmp/ab.csv')) if len(r) > 10]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
for r in rows[1:]:
    t=float(r[ix['Metric Value']].replace(',',''))
    if t > 50000: print(f"  {r[ix['Kernel Name']][:50]:50s} {t/1e6:.3f} ms")
PY
done
cat gpurun_out/ab_dev.log
