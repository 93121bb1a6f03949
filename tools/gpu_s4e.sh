mkdir -p gpurun_out
GLR_NVCC_EXTRA="-DGLR_EIG_STATS" python -m paper_2301_03047_b200._build -f > gpurun_out/e_build.log 2>&1
for c in C2 C4; do timeout 600 python tools/eig_stats.py $c > gpurun_out/e_eig_$c.log 2>&1; done
grep pairs gpurun_out/e_eig_C2.log | head -60
