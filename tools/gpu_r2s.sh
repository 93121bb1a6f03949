mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_match.py -q -rf > gpurun_out/s_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s_pytest.log
timeout 900 python tools/stage_sweep.py --reps 2 --fused --only 8:16384,8:4096,12:16384 > gpurun_out/s_sweep_fused.jsonl 2>&1
for c in C2 C4 C1; do GLR_MATCH_MODE=fused timeout 300 python tools/iter_profile.py $c > gpurun_out/s_fused_$c.log 2>&1; done
tail -3 gpurun_out/s_pytest.log
python - <<'PY'
import json
for l in open("gpurun_out/s_sweep_fused.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["P"], d["exemplars"], d["heat"]["ms"], d["topk"]["ms"], d["wnnm"]["ms"], d["mode"][:60])
PY
for c in C2 C4 C1; do echo "== fused $c"; grep "heat per\|^total\|topk" gpurun_out/s_fused_$c.log | cut -c1-200; done
