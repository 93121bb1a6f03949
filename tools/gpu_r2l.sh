# dense vs fused match per configuration: per-iteration profiles
mkdir -p gpurun_out
for m in dense fused; do for c in C2 C4 C1; do GLR_MATCH_MODE=$m timeout 300 python tools/iter_profile.py $c > gpurun_out/l_${m}_$c.log 2>&1; done; done
for m in dense fused; do for c in C2 C4 C1; do echo "== $m $c"; grep -v "^[a-z_]*:\|wnnm per\|iteration ms" gpurun_out/l_${m}_$c.log | cut -c1-200; done; done
