# dev: top-K floor divisor A/B on C2 (solve) and C5 (stage sweep), with stats
mkdir -p gpurun_out
for f in 2 1; do
  echo "== floor shift $f" >> gpurun_out/ab_topk.log
  GLR_NVCC_EXTRA="-DGLR_TOPK_STATS -DGLR_TOPK_FLOOR_SHIFT=$f" python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  timeout 600 python tools/topk_stats.py C2 >> gpurun_out/ab_topk.log 2>&1
  GLR_NVCC_EXTRA="-DGLR_TOPK_FLOOR_SHIFT=$f" python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  timeout 600 python tools/iter_profile.py C2 2>&1 | grep -E "topk|total" >> gpurun_out/ab_topk.log
  timeout 900 python tools/stage_sweep.py --reps 1 2>&1 | cut -c1-330 >> gpurun_out/ab_topk.log
done
cat gpurun_out/ab_topk.log
