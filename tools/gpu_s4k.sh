mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_full_configs.py -m gpu -x -q > gpurun_out/k_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k_pytest.log
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/k_bench_C4.json 2> gpurun_out/k_bench_C4.err
timeout 300 python tools/trace_x.py C4 > gpurun_out/k_trace_C4.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/k_launch_C4.csv python tools/one_solve.py C4 > gpurun_out/k_ncu_C4.log 2>&1
python tools/launch_series.py /tmp/k_launch_C4.csv gram_kernel eig_kernel apply_oz_kernel > gpurun_out/k_series_C4.txt
tail -5 gpurun_out/k_pytest.log
cut -c1-200 gpurun_out/k_bench_C4.json
cat gpurun_out/k_series_C4.txt; tail -3 gpurun_out/k_trace_C4.txt
