# One GPU round trip: tests, smoke, bench (both arms), ncu launch list and a
# --set full capture exported to CSV on the box (the .ncu-rep stays in /tmp:
# gpurun copies back at most 64 MiB of gpurun_out/).
# usage: bash tools/gpu_round.sh "<pytest selection>"
SEL=${1:-tests}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest $SEL -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -o /tmp/window -f python tools/ncu_window.py C2 > gpurun_out/ncu_full.log 2>&1; echo "ncufull rc=$?" >> gpurun_out/ncu_full.log
ncu -i /tmp/window.ncu-rep --page raw --csv > gpurun_out/window_raw.csv 2>> gpurun_out/ncu_full.log
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 "$f"; done
du -sh gpurun_out
