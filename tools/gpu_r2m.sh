mkdir -p gpurun_out
for m in dense fused; do
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:"heat_gemm_kernel" -c 2 -o gpurun_out/m_ncu_c5_$m python tools/c5_window.py 8 4096 $m > gpurun_out/m_ncu_$m.log 2>&1
tail -2 gpurun_out/m_ncu_$m.log
done
