mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/tc_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tc_pytest.log
timeout 600 python tools/iter_profile.py C2 2>&1 | grep -E "topk|total" > gpurun_out/tc_iter.log
timeout 900 python tools/stage_sweep.py --reps 1 2>&1 | cut -c1-330 > gpurun_out/tc_sweep.log
for c in C1 C3 C4; do timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['kernels']['topk'])" >> gpurun_out/tc_cfg.log; done
tail -3 gpurun_out/tc_pytest.log; cat gpurun_out/tc_iter.log gpurun_out/tc_sweep.log gpurun_out/tc_cfg.log
