"""Key metrics per kernel launch from an `ncu --set full` report (.ncu-rep)."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"]
idx = {k: hdr.index(k) for k in want if k in hdr}
res = []
for r in data:
    d = {k: r[i] for k, i in idx.items()}
    d["units"] = {k: units[i] for k, i in idx.items()}
    res.append(d)
for d in res:
    print(d["Kernel Name"][:70])
    for k in want[1:]:
        if k in d:
            print(f"    {k:80s} {d[k]} {d['units'].get(k, '')}")
if len(sys.argv) > 2:
    json.dump(res, open(sys.argv[2], "w"), indent=1)
