# fused heat+top-K (sampled floor): parity vs dense on full refreshes + C5 stage sweep both modes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_match.py -q -rf > gpurun_out/i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/i_pytest.log
timeout 900 python tools/stage_sweep.py --reps 2 --fused > gpurun_out/i_sweep_fused.jsonl 2> gpurun_out/i_sweep_fused.err

tail -n 8 gpurun_out/i_pytest.log; tail -3 gpurun_out/i_sweep_fused.err
python - <<'PY'
import json
for f in ("gpurun_out/i_sweep_dense.jsonl", "gpurun_out/i_sweep_fused.jsonl"):
    try:
        for l in open(f):
            d = json.loads(l); print(f[-20:], d["P"], d["exemplars"], d["heat"]["ms"], d["topk"]["ms"], d["wnnm"]["ms"], d.get("mode","")[:80])
    except Exception as e: print(f, e)
PY
