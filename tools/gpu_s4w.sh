mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fused_match.py tests/test_gpu_configs.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/w_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/w_pytest.log
for c in C5 C2; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/w_bench_$c.json 2> gpurun_out/w_bench_$c.err
done
tail -3 gpurun_out/w_pytest.log
for c in C5 C2; do cut -c1-230 gpurun_out/w_bench_$c.json; python -c "
import json
d=json.loads(open('gpurun_out/w_bench_$c.json').read().strip().splitlines()[-1])
print({k:round(v['ms_total']/d['steps'],2) for k,v in d['kernels'].items()})
"; done
