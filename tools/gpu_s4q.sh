mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:topk_kernel -c 1 -o /tmp/tk -f python tools/ncu_window.py C4 > gpurun_out/q_ncu.log 2>&1
ncu -i /tmp/tk.ncu-rep --page source --csv --print-source cuda,sass > /tmp/tk_src.csv 2>&1
python tools/src_hot.py /tmp/tk_src.csv 45 > gpurun_out/q_tk_hot.txt 2>&1
ncu -i /tmp/tk.ncu-rep --page details > gpurun_out/q_tk_details.txt 2>&1
head -50 gpurun_out/q_tk_hot.txt
grep -E "Duration|Registers|Achieved Occupancy|Theoretical Occ|Block Limit|DRAM Throughput|Shared Memory Config|Dynamic Shared" gpurun_out/q_tk_details.txt | head -20
