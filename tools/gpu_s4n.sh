mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py tests/test_gpu_configs.py tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/n_pytest.log
for c in C2 C3 C4 C1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/n_bench_$c.json 2> gpurun_out/n_bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/n_launch_C2.csv python tools/one_solve.py C2 > gpurun_out/n_ncu_C2.log 2>&1
python tools/launch_series.py /tmp/n_launch_C2.csv gram_kernel eig_kernel apply_oz_kernel > gpurun_out/n_series_C2.txt
tail -3 gpurun_out/n_pytest.log
for c in C2 C3 C4 C1; do cut -c1-200 gpurun_out/n_bench_$c.json; done
grep eig_kernel -A1 gpurun_out/n_series_C2.txt
