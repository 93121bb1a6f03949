# ncu --set full on the top kernels of a C2 warm iteration + compute-sanitizer runs.
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:"apply_oz_kernel|eig_kernel|topk_kernel|gram_kernel" -c 6 \
  -o gpurun_out/h_ncu_C2 python tools/ncu_window.py C2 > gpurun_out/h_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/h_ncu.log
bash tools/gpu_sanitize.sh
tail -3 gpurun_out/h_ncu.log
