mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py tests/test_gpu_fused_match.py -q -rf > gpurun_out/o_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/o_pytest.log
timeout 300 python tools/iter_profile.py C2 > gpurun_out/o_iter_C2.log 2>&1
timeout 900 python tools/stage_sweep.py --reps 2 --only 8:16384,12:16384 > gpurun_out/o_sweep_dense.jsonl 2>&1
timeout 900 python tools/stage_sweep.py --reps 2 --fused --only 8:16384,12:16384 > gpurun_out/o_sweep_fused.jsonl 2>&1
tail -4 gpurun_out/o_pytest.log; grep -v "^[a-z_]*:\|iteration ms" gpurun_out/o_iter_C2.log | cut -c1-300
python - <<'PY'
import json
for f in ("gpurun_out/o_sweep_dense.jsonl", "gpurun_out/o_sweep_fused.jsonl"):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); print(f[-18:], d["P"], d["exemplars"], d["heat"]["ms"], d["topk"]["ms"], d["mode"][:60])
PY
