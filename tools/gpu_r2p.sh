mkdir -p gpurun_out
for r in 1 2; do timeout 900 python tools/stage_sweep.py --reps 2 --fused --only 8:16384,8:4096 > gpurun_out/p_sweep_fused_$r.jsonl 2>&1; done
timeout 900 python tools/stage_sweep.py --reps 2 --only 8:16384,8:4096 > gpurun_out/p_sweep_dense.jsonl 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/p_sweep_*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); print(f[-22:], d["P"], d["exemplars"], d["heat"]["ms"], d["topk"]["ms"], d["mode"][:50])
PY
