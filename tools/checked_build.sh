# Checked build (device bounds / invariant asserts, -DGLR_CHECKS) run over the
# small end-to-end workload, the smoke solve and the device parity tests; the
# stand-in for compute-sanitizer, which this GPU pool does not allow.
mkdir -p gpurun_out
GLR_NVCC_EXTRA=-DGLR_CHECKS timeout 600 python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > gpurun_out/chk_build.log 2>&1 || exit 1
nm -D paper_2301_03047_b200/libglr_b200.so > /dev/null
strings paper_2301_03047_b200/libglr_b200.so | grep -c "GLR_DCHECK failed" > gpurun_out/chk_count.txt
timeout 600 python tools/sanitize_small.py 6 > gpurun_out/chk_small.log 2>&1; echo "small rc=$?" >> gpurun_out/chk_small.log
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/chk_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chk_pytest.log
tail -2 gpurun_out/chk_small.log; tail -3 gpurun_out/chk_pytest.log
