mkdir -p gpurun_out
timeout 300 python tools/trace_x.py C4 > gpurun_out/i_trace_new.txt 2>&1
cd _old_r01
python -m paper_2301_03047_b200._build -f > /dev/null 2>&1
timeout 300 python tools/trace_x.py C4 > ../gpurun_out/i_trace_old.txt 2>&1
cd ..
paste -d'\n' gpurun_out/i_trace_new.txt gpurun_out/i_trace_old.txt | head -64
