mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:heat_gemm -o /tmp/c5h -f python tools/c5_window.py 8 16384 fused > gpurun_out/y_ncu.log 2>&1
ncu -i /tmp/c5h.ncu-rep --page details > gpurun_out/y_details.txt 2>&1
ncu -i /tmp/c5h.ncu-rep --page source --csv --print-source cuda,sass > /tmp/c5h_src.csv 2>&1
python tools/src_hot.py /tmp/c5h_src.csv 40 > gpurun_out/y_hot.txt 2>&1
tail -3 gpurun_out/y_ncu.log
grep -E "Duration|Issue Slots Busy|Executed Ipc|No Eligible|Stall|L2 Cache Throughput|DRAM Throughput|Mem Busy|Max Bandwidth|Tensor" gpurun_out/y_details.txt | head -40
tail -45 gpurun_out/y_hot.txt
