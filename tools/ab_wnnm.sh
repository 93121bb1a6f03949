mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_pytest.log
for v in "GLR_GRAM_IMPL=3 GLR_APPLY_IMPL=s" "GLR_GRAM_IMPL=4 GLR_APPLY_IMPL=s" "GLR_GRAM_IMPL=3 GLR_APPLY_IMPL=r" "GLR_GRAM_IMPL=4 GLR_APPLY_IMPL=r"; do
  echo "== $v" >> gpurun_out/ab_iter.log
  env $v timeout 600 python tools/iter_profile.py C2 2>&1 | head -3 >> gpurun_out/ab_iter.log
  env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv python tools/ncu_window.py C2 2>/dev/null | grep -E "gram|apply|eig" | cut -c1-200 >> gpurun_out/ab_iter.log
done
tail -n 3 gpurun_out/ab_pytest.log; cat gpurun_out/ab_iter.log
