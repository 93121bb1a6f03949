# Round 2 GPU pass C: GPU suite (no -x), per-iteration profiles, C2 / C3 bench lines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c_pytest.log
timeout 300 python tools/iter_profile.py C2 > gpurun_out/c_iter_C2.log 2>&1
timeout 300 python tools/iter_profile.py C3 > gpurun_out/c_iter_C3.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c_bench_C2.json 2> gpurun_out/c_bench_C2.err
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c_bench_C3.json 2> gpurun_out/c_bench_C3.err
tail -n 12 gpurun_out/c_pytest.log; cat gpurun_out/c_iter_C2.log gpurun_out/c_iter_C3.log | cut -c1-400
