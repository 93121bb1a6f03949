# ncu --set full of the eigen kernel (C2 warm iteration 6), per-source-line samples and shared wavefronts
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:eig_kernel -c 1 -o /tmp/eig -f python tools/ncu_window.py C2 > gpurun_out/m_ncu.log 2>&1
ncu -i /tmp/eig.ncu-rep --page source --csv --print-source cuda,sass > /tmp/eig_src.csv 2>&1
python tools/src_hot.py /tmp/eig_src.csv 60 > gpurun_out/m_eig_hot.txt 2>&1
ncu -i /tmp/eig.ncu-rep --page details > gpurun_out/m_eig_details.txt 2>&1
head -70 gpurun_out/m_eig_hot.txt
