mkdir -p gpurun_out
for tol in 1e-12 1e-10 1e-9; do
  echo "== tol $tol" >> gpurun_out/ab_rottol.log
  GLR_NVCC_EXTRA="-DGLR_EIG_ROTTOL=$tol" python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_bm.py -m gpu -q 2>&1 | tail -2 >> gpurun_out/ab_rottol.log
  timeout 600 python tools/iter_profile.py C2 2>&1 | grep -E "wnnm per|^total" >> gpurun_out/ab_rottol.log
done
cat gpurun_out/ab_rottol.log
