mkdir -p gpurun_out; rm -f gpurun_out/z.log
for g in 5 7; do
  echo "== epi groups $g" >> gpurun_out/z.log
  GLR_NVCC_EXTRA="-DGLR_HEAT_EPI_GROUPS=$g" python -c "from paper_2301_03047_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  grep -A2 heat_gemm_kernel build/ptxas.log | grep -E "registers|spill" >> gpurun_out/z.log
  timeout 900 python -m pytest tests/test_gpu_fused_match.py tests/test_gpu_parity.py -m gpu -q -k "heat or fused or topk" 2>&1 | tail -2 >> gpurun_out/z.log
  for c in C5 C2 C4; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', round(d['value'],1), round(d['ms_per_step'],2), {k:round(v['ms_total']/d['steps'],2) for k,v in d['kernels'].items() if k in ('heat_topk','heat_map','topk')})
" >> gpurun_out/z.log
  done
done
cat gpurun_out/z.log
