mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_pytest.log
for c in C2 C3 C4 C1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/t_bench_$c.json 2> gpurun_out/t_bench_$c.err
done
GLR_NVCC_EXTRA="-DGLR_EIG_STATS" python -m paper_2301_03047_b200._build -f > gpurun_out/t_build.log 2>&1
timeout 600 python tools/eig_stats.py C2 > gpurun_out/t_eig_C2.log 2>&1
tail -3 gpurun_out/t_pytest.log
for c in C2 C3 C4 C1; do cut -c1-200 gpurun_out/t_bench_$c.json; done
grep pairs gpurun_out/t_eig_C2.log | sed -n '7,10p;17,20p;30,33p;45,48p'
