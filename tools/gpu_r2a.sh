# Round 2 GPU pass A: full GPU suite, C2 + C3 bench lines, Jacobi sweep stats (C3, C2).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/a_bench_C2.json 2> gpurun_out/a_bench_C2.err; echo "bench rc=$?" >> gpurun_out/a_bench_C2.err
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/a_bench_C3.json 2> gpurun_out/a_bench_C3.err
mkdir -p /tmp/glrb && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2301_03047_b200/csrc -I include tools/micro/tc_peak.cu -o /tmp/glrb/tc_peak && /tmp/glrb/tc_peak > gpurun_out/a_tc_peak.json 2>&1
GLR_NVCC_EXTRA=-DGLR_EIG_STATS timeout 300 python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > gpurun_out/a_statbuild.log 2>&1
timeout 300 python tools/eig_stats.py C3 > gpurun_out/a_eig_C3.log 2>&1
timeout 300 python tools/eig_stats.py C2 > gpurun_out/a_eig_C2.log 2>&1
for f in gpurun_out/a_pytest.log gpurun_out/a_bench_C2.err gpurun_out/a_eig_C3.log; do echo "== $f"; tail -n 25 "$f"; done
