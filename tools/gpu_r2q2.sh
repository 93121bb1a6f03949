mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:"heat_gemm_kernel|topk_cand|sample_thr" -c 4 -o gpurun_out/q_ncu_c5_16k python tools/c5_window.py 8 16384 fused > gpurun_out/q_ncu.log 2>&1
tail -2 gpurun_out/q_ncu.log
