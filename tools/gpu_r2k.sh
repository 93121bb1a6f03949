mkdir -p gpurun_out
GLR_NVCC_EXTRA=-DGLR_TOPK_STATS timeout 300 python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > gpurun_out/k_build.log 2>&1
for c in C1 C3 C4 C2 C5-8 C5-12; do timeout 300 python tools/cand_stats.py $c 2>&1 | tail -1; done
