mkdir -p gpurun_out
GLR_NVCC_EXTRA="-DGLR_EIG_STATS" python -m paper_2301_03047_b200._build -f > gpurun_out/5b_build.log 2>&1
for c in C4 C3; do timeout 600 python tools/eig_stats.py $c > gpurun_out/5b_eig_$c.log 2>&1; done
cut -c1-200 gpurun_out/5b_eig_C4.log | sed -n '3,8p;21,24p;41,44p;55,60p'
echo; cut -c1-200 gpurun_out/5b_eig_C3.log | sed -n '3,8p;21,24p;41,44p;75,80p'
