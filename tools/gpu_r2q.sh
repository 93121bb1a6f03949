# Round 2 quick GPU pass: GPU suite + per-iteration profiles of C2 / C3 / C1.
# usage: bash tools/gpu_r2q.sh TAG
T=${1:-q}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for c in C2 C3 C1; do timeout 300 python tools/iter_profile.py $c > gpurun_out/${T}_iter_$c.log 2>&1; done
tail -n 6 gpurun_out/${T}_pytest.log; cat gpurun_out/${T}_iter_C2.log gpurun_out/${T}_iter_C3.log gpurun_out/${T}_iter_C1.log | grep -v "^[a-z_]*:" | cut -c1-400
