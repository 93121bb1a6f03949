mkdir -p gpurun_out; rm -f gpurun_out/u.log
for q in 0.5 0.1; do
  echo "== quad tol $q" >> gpurun_out/u.log
  GLR_NVCC_EXTRA="-DGLR_EIG_QUADTOL=$q" python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -m gpu -q 2>&1 | tail -2 >> gpurun_out/u.log
  for c in C2 C3 C4; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-190 >> gpurun_out/u.log
  done
done
cat gpurun_out/u.log
