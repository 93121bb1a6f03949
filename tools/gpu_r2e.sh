# Round 2 GPU pass D: parity suite + per-iteration profiles + sweep stats (eigen finish experiment).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/e_pytest.log
timeout 300 python tools/iter_profile.py C2 > gpurun_out/e_iter_C2.log 2>&1
timeout 300 python tools/iter_profile.py C3 > gpurun_out/e_iter_C3.log 2>&1
timeout 300 python tools/iter_profile.py C1 > gpurun_out/e_iter_C1.log 2>&1
GLR_NVCC_EXTRA=-DGLR_EIG_STATS timeout 300 python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > gpurun_out/e_statbuild.log 2>&1
timeout 300 python tools/eig_stats.py C2 > gpurun_out/e_eig_C2.log 2>&1
timeout 300 python tools/eig_stats.py C1 > gpurun_out/e_eig_C1.log 2>&1
tail -n 12 gpurun_out/e_pytest.log; cat gpurun_out/e_iter_C2.log gpurun_out/e_iter_C3.log gpurun_out/e_iter_C1.log | grep -v "^[a-z_]*:" | cut -c1-400
