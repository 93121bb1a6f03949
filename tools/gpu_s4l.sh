mkdir -p gpurun_out
GLR_NVCC_EXTRA="-DGLR_EIG_STATS" python -m paper_2301_03047_b200._build -f > gpurun_out/l_build.log 2>&1
for c in C4; do timeout 600 python tools/eig_stats.py $c > gpurun_out/l_eig_$c.log 2>&1; done
cut -c1-330 gpurun_out/l_eig_C4.log
