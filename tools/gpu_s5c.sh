mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py tests/test_gpu_multirank.py tests/test_gpu_dispatch.py -m gpu -x -q > gpurun_out/5c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/5c_pytest.log
tail -3 gpurun_out/5c_pytest.log
for c in C2 C3 C4 C1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', round(d['value'],1), round(d['ms_per_step'],2), {k:round(v['ms_total']/d['steps'],2) for k,v in d['kernels'].items() if k in ('heat_topk','heat_map','topk','wnnm_scatter')})
"
done
