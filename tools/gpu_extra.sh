# stage sweep (C5) + bench lines of the other configurations (C1, C3, C4)
mkdir -p gpurun_out
timeout 1200 python tools/stage_sweep.py --reps 2 --out gpurun_out/stage_sweep_C5.jsonl > gpurun_out/stage_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/stage_sweep.log
for c in C1 C3 C4; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?" >> gpurun_out/bench_$c.log
done
tail -n 8 gpurun_out/stage_sweep.log | cut -c1-300
for c in C1 C3 C4; do tail -n 2 gpurun_out/bench_$c.log | cut -c1-300; done
