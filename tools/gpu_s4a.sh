# Session baseline at HEAD: GPU suite + bench lines for every solver config.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
for c in C2 C3 C4 C1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/a_bench_$c.json 2> gpurun_out/a_bench_$c.err
done
tail -4 gpurun_out/a_pytest.log
for c in C2 C3 C4 C1; do cut -c1-300 gpurun_out/a_bench_$c.json; tail -2 gpurun_out/a_bench_$c.err; done
