mkdir -p gpurun_out
for c in C4 C3 C1; do
  for m in dense fused; do
    GLR_MATCH_MODE=$m timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/o_bench_${c}_$m.json 2> gpurun_out/o_bench_${c}_$m.err
    python - <<PY
import json
d=json.loads(open("gpurun_out/o_bench_${c}_$m.json").read().strip().splitlines()[-1])
print("$c $m", round(d["value"],1), round(d["ms_per_step"],2), {k:(round(v["ms_total"]/d["steps"],2), round(v.get("frac",0) or 0,3)) for k,v in d["kernels"].items() if k in ("heat_map","topk","heat_topk")})
PY
  done
done
