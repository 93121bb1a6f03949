# Quick GPU iteration: selected tests, one profiled solve, per-kernel times of
# one warm + one refresh iteration (ncu duration only).
SEL=${1:-tests/test_gpu_parity.py}
mkdir -p gpurun_out
timeout 1200 python -m pytest $SEL -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 600 python tools/iter_profile.py C2 > gpurun_out/q_iter.log 2>&1; echo "iter rc=$?" >> gpurun_out/q_iter.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv python tools/ncu_window.py C2 > gpurun_out/q_ncu.csv 2> gpurun_out/q_ncu.err; echo "ncu rc=$?" >> gpurun_out/q_ncu.err
for f in gpurun_out/q_*.log gpurun_out/q_ncu.err; do echo "== $f"; tail -n 12 "$f"; done
