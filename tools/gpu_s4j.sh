mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fused_match.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j_pytest.log
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/j_bench_C2.json 2> gpurun_out/j_bench_C2.err
timeout 600 python tools/iter_profile.py C2 > gpurun_out/j_iter_C2.txt 2>&1
tail -3 gpurun_out/j_pytest.log
cut -c1-200 gpurun_out/j_bench_C2.json
grep -E "heat per|fallback" gpurun_out/j_iter_C2.txt
