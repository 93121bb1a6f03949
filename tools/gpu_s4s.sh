mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/s_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s_pytest.log
for c in C2 C3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s_bench_$c.json 2> gpurun_out/s_bench_$c.err
done
tail -3 gpurun_out/s_pytest.log
for c in C2 C3; do cut -c1-200 gpurun_out/s_bench_$c.json; done
