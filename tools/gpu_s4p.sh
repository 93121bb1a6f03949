# A/B of the first-order finish tolerance (kFinishTol)
mkdir -p gpurun_out; rm -f gpurun_out/p_fin.log
for tol in 3e-5 1e-4; do
  echo "== finish tol $tol" >> gpurun_out/p_fin.log
  GLR_NVCC_EXTRA="-DGLR_EIG_FINISHTOL=$tol" python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_full_configs.py tests/test_gpu_bm.py tests/test_gpu_multirank.py -m gpu -q 2>&1 | tail -4 >> gpurun_out/p_fin.log
  for c in C2 C3 C4; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-190 >> gpurun_out/p_fin.log
  done
done
cat gpurun_out/p_fin.log
