mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:topk_kernel -c 1 -o /tmp/tk -f python tools/ncu_window.py C2 > gpurun_out/tk.log 2>&1
ncu -i /tmp/tk.ncu-rep --page source --csv --print-source cuda > gpurun_out/tk_cuda.csv 2>>gpurun_out/tk.log
ncu -i /tmp/tk.ncu-rep --page raw --csv > gpurun_out/tk_raw2.csv 2>>gpurun_out/tk.log
ls -la gpurun_out; tail -3 gpurun_out/tk.log
