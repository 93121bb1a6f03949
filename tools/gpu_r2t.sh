mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/t_bench_C2.json 2> gpurun_out/t_bench_C2.err
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/t_bench_C5.json 2> gpurun_out/t_bench_C5.err
tail -4 gpurun_out/t_pytest.log; cut -c1-600 gpurun_out/t_bench_C2.json; tail -3 gpurun_out/t_bench_C2.err; cut -c1-400 gpurun_out/t_bench_C5.json; tail -3 gpurun_out/t_bench_C5.err
