mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wnnm or gap_solve or admm or vcache" > gpurun_out/ab_eig_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_eig_pytest.log
for v in quad oct; do
  echo "== $v" >> gpurun_out/ab_eig.log
  GLR_EIG_IMPL=$v timeout 600 python tools/iter_profile.py C2 2>&1 | grep -E "wnnm per|total" >> gpurun_out/ab_eig.log
done
tail -5 gpurun_out/ab_eig_pytest.log; cat gpurun_out/ab_eig.log
