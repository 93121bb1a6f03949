mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"topk_kernel|apply_kernel|gram_kernel" -o /tmp/tk -f python tools/ncu_window.py C2 > gpurun_out/ncu_tk.log 2>&1
ncu -i /tmp/tk.ncu-rep --page raw --csv > gpurun_out/tk_raw.csv 2>>gpurun_out/ncu_tk.log
ncu -i /tmp/tk.ncu-rep --page source --csv -k topk_kernel > gpurun_out/tk_source.csv 2>>gpurun_out/ncu_tk.log
for f in gpurun_out/pytest_gpu.log gpurun_out/bench.log gpurun_out/ncu_tk.log; do echo "== $f"; tail -n 4 $f | cut -c1-600; done
du -sh gpurun_out
