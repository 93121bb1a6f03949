# tests + iteration profile + per-kernel durations (one warm + one refresh iteration)
SEL=${1:-tests}
mkdir -p gpurun_out
timeout 1500 python -m pytest $SEL -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 600 python tools/iter_profile.py C2 > gpurun_out/q_iter.log 2>&1; echo "iter rc=$?" >> gpurun_out/q_iter.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --profile-from-start off --csv python tools/ncu_window.py C2 2>/dev/null > /tmp/q.csv
python - > gpurun_out/q_kernels.log <<'PY'
import csv
rows=[r for r in csv.reader(open('/tmp/q.csv')) if len(r) > 10]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
d={}
for r in rows[1:]:
    k=(r[ix['ID']], r[ix['Kernel Name']][:50])
    d.setdefault(k,{})[r[ix['Metric Name']]]=float(r[ix['Metric Value']].replace(',',''))
for (i,n),m in d.items():
    t=m.get('gpu__time_duration.sum',0)
    if t>50000: print(f"{n:50s} {t/1e6:7.3f} ms  read {m.get('dram__bytes_read.sum',0)/1e9:7.3f} GB")
PY
for f in gpurun_out/q_pytest.log gpurun_out/q_iter.log gpurun_out/q_kernels.log; do echo "== $f"; tail -n 30 $f | cut -c1-400; done
