# Round 2 GPU pass B: full GPU suite, per-iteration WNNM (C2, C3), per-kernel
# launch times of a warm + a refresh iteration (C2, C3), Jacobi sweep stats.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -x --deselect tests/test_gpu_bm.py > gpurun_out/b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/b_pytest.log
timeout 300 python tools/iter_profile.py C2 > gpurun_out/b_iter_C2.log 2>&1
timeout 300 python tools/iter_profile.py C3 > gpurun_out/b_iter_C3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv python tools/ncu_window.py C2 > gpurun_out/b_win_C2.csv 2> gpurun_out/b_win_C2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv python tools/ncu_window.py C3 > gpurun_out/b_win_C3.csv 2> gpurun_out/b_win_C3.err
GLR_NVCC_EXTRA=-DGLR_EIG_STATS timeout 300 python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > gpurun_out/b_statbuild.log 2>&1
timeout 300 python tools/eig_stats.py C3 > gpurun_out/b_eig_C3.log 2>&1
timeout 300 python tools/eig_stats.py C1 > gpurun_out/b_eig_C1.log 2>&1
tail -n 8 gpurun_out/b_pytest.log; cat gpurun_out/b_iter_C2.log gpurun_out/b_iter_C3.log | cut -c1-600
