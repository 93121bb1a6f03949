# Quick check of a WNNM change: the image-group test, the solve parity tests,
# then per-kernel times of one warm + one refresh C2 iteration.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wnnm_scatter_image" > gpurun_out/oz_t1.log 2>&1; echo "t1 rc=$?" >> gpurun_out/oz_t1.log
tail -3 gpurun_out/oz_t1.log
grep -q "t1 rc=0" gpurun_out/oz_t1.log || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/oz_t2.log 2>&1; echo "t2 rc=$?" >> gpurun_out/oz_t2.log
tail -3 gpurun_out/oz_t2.log
timeout 600 python tools/iter_profile.py C2 > gpurun_out/oz_iter.log 2>&1; echo "iter rc=$?" >> gpurun_out/oz_iter.log
tail -30 gpurun_out/oz_iter.log
