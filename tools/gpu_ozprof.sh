# ncu --set full of the split-integer apply kernel + per-kernel times (dev)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wnnm_scatter_image or gap_solve_vs" > gpurun_out/oz_t1.log 2>&1; echo "t1 rc=$?" >> gpurun_out/oz_t1.log
tail -2 gpurun_out/oz_t1.log
grep -q "t1 rc=0" gpurun_out/oz_t1.log || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:apply_oz -c 1 -o /tmp/oz -f python tools/ncu_window.py C2 > gpurun_out/oz_ncu.log 2>&1
ncu -i /tmp/oz.ncu-rep --page raw --csv > gpurun_out/oz_raw.csv
ncu -i /tmp/oz.ncu-rep --page source --csv --print-source sass > gpurun_out/oz_src.csv 2>&1
ncu -i /tmp/oz.ncu-rep --page details > gpurun_out/oz_details.txt
rm -f gpurun_out/ab_dev.log; bash tools/ab_dev.sh 2>&1 | grep -E "gram|eig|apply"
