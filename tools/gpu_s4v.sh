mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v_pytest.log
for c in C2 C3 C4 C1 C5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v_bench_$c.json 2> gpurun_out/v_bench_$c.err
done
tail -3 gpurun_out/v_pytest.log
for c in C2 C3 C4 C1 C5; do cut -c1-200 gpurun_out/v_bench_$c.json; tail -2 gpurun_out/v_bench_$c.err; done
