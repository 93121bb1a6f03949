# Round-2 profiles of the headline command: the ncu launch list of bench.py (C2) and an
# ncu --set full capture of a refresh + a warm iteration (tools/ncu_window.py C2).
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches_C2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof_launch_bench.log 2>&1; echo "launches rc=$?"
timeout 1800 ncu --set full --clock-control none --profile-from-start off -o gpurun_out/prof_full_C2 \
  python tools/ncu_window.py C2 > gpurun_out/prof_full.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/prof_full_C2.ncu-rep --page raw --csv > gpurun_out/prof_full_C2_raw.csv 2>/dev/null
ls -la gpurun_out/prof_*
