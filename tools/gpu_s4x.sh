mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_full_configs.py -m gpu -x -q -k "corner or c5 or C5 or edges or anchors" > gpurun_out/x_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/x_pytest.log
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/x_bench_C5.json 2> gpurun_out/x_bench_C5.err
tail -3 gpurun_out/x_pytest.log
cut -c1-230 gpurun_out/x_bench_C5.json; python -c "
import json
d=json.loads(open('gpurun_out/x_bench_C5.json').read().strip().splitlines()[-1])
print({k:round(v['ms_total']/d['steps'],2) for k,v in d['kernels'].items()})
"
