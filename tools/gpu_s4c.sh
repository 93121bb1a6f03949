# A/B of the eigen-kernel exemption rules: parity subset, sweep histograms (stats build last), benches.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c_pytest.log
for c in C3 C4 C2 C1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c_bench_$c.json 2> gpurun_out/c_bench_$c.err
done
GLR_NVCC_EXTRA="-DGLR_EIG_STATS $EXTRA" python -m paper_2301_03047_b200._build -f > gpurun_out/c_build.log 2>&1
for c in C4 C3; do timeout 600 python tools/eig_stats.py $c > gpurun_out/c_eig_$c.log 2>&1; done
tail -3 gpurun_out/c_pytest.log
for c in C3 C4 C2 C1; do cut -c1-200 gpurun_out/c_bench_$c.json; done
