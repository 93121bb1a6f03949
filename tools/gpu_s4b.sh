# Jacobi sweep histograms per iteration on C4 and C3 (stats build made on the box).
mkdir -p gpurun_out
GLR_NVCC_EXTRA=-DGLR_EIG_STATS python -m paper_2301_03047_b200._build -f > gpurun_out/b_build.log 2>&1
for c in C4 C3; do timeout 600 python tools/eig_stats.py $c > gpurun_out/b_eig_$c.log 2>&1; done
head -42 gpurun_out/b_eig_C4.log | cut -c1-400
