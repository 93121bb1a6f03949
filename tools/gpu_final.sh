# Round-end consolidation: full GPU suite, smoke, bench lines (both arms, every config),
# ncu launch list + --set full window of the headline command.
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fin_smi.txt
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/fin_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin_smoke.log
timeout 900 python bench.py > gpurun_out/fin_bench_C2.json 2> gpurun_out/fin_bench_C2.err; echo "bench rc=$?" >> gpurun_out/fin_bench_C2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_bench_ref_C2.json 2> gpurun_out/fin_bench_ref_C2.err
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/fin_bench_$c.json 2> gpurun_out/fin_bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_C2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/fin_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -o /tmp/fin_window -f python tools/ncu_window.py C2 > gpurun_out/fin_ncu_full.log 2>&1; echo "ncufull rc=$?" >> gpurun_out/fin_ncu_full.log
ncu -i /tmp/fin_window.ncu-rep --page raw --csv > gpurun_out/fin_window_raw.csv 2>> gpurun_out/fin_ncu_full.log
tail -4 gpurun_out/fin_pytest.log; tail -2 gpurun_out/fin_smoke.log
for c in C2 C1 C3 C4 C5; do cut -c1-260 gpurun_out/fin_bench_$c.json; done
cut -c1-300 gpurun_out/fin_bench_ref_C2.json
du -sh gpurun_out
