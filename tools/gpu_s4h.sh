mkdir -p gpurun_out
cd _old_r01
python -m paper_2301_03047_b200._build -f > ../gpurun_out/h_build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/h_launch_C4.csv python tools/one_solve.py C4 > ../gpurun_out/h_ncu_C4.log 2>&1
python tools/launch_series.py /tmp/h_launch_C4.csv gram_kernel eig_kernel apply > ../gpurun_out/h_series_C4.txt
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > ../gpurun_out/h_bench_C4.json 2> ../gpurun_out/h_bench_C4.err
cat ../gpurun_out/h_series_C4.txt; cut -c1-200 ../gpurun_out/h_bench_C4.json
