mkdir -p gpurun_out
for c in C4 C2 C3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/d_launch_$c.csv python tools/one_solve.py $c > gpurun_out/d_ncu_$c.log 2>&1
  python tools/launch_series.py /tmp/d_launch_$c.csv gram_kernel eig_kernel apply_oz_kernel > gpurun_out/d_series_$c.txt
done
for c in C3 C4 C2 C1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/d_bench_$c.json 2> gpurun_out/d_bench_$c.err
  cut -c1-200 gpurun_out/d_bench_$c.json
done
cat gpurun_out/d_series_C4.txt
