"""Write the round's ncu summaries under profiles/ from gpurun_out captures.

  python tools/profiles_update.py <raw.csv from ncu --set full> <launches.csv> <tag>

raw.csv: `ncu -i <rep> --page raw --csv` of tools/ncu_window.py (one warm GLR
iteration + one refresh iteration of C2). launches.csv: the
`--metrics gpu__time_duration.sum` launch list of `bench.py --steps 2 --warmup 3`.
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
raw, launches, tag = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread"]
ix = {h: i for i, h in enumerate(hdr)}
out, lines = [], []
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
for r in rows[2:]:
    d = {"kernel": r[ix["Kernel Name"]]}
    for k in want:
        if k in ix:
            v, u = r[ix[k]], units[ix[k]]
            try:
                fv = float(v.replace(",", ""))
            except ValueError:
                continue
            if k.startswith("dram__bytes"):
                fv *= scale.get(u, 1)
                u = "byte"
            d[k] = fv
            d[k + ".unit"] = u
    out.append(d)
    lines.append(d["kernel"][:90])
    for k in want:
        if k in d:
            lines.append(f"    {k:78s} {d[k]:.6g} {d[k + '.unit']}")
prof = ROOT / "profiles"
(prof / f"{tag}_ncu_full_C2.json").write_text(json.dumps(out, indent=1))
(prof / f"{tag}_ncu_full_C2.txt").write_text(
    f"# ncu --set full --clock-control none, tools/ncu_window.py C2 (warm iteration 6 + refresh"
    f" iteration 10), round tag {tag}\n" + "\n".join(lines) + "\n")


def per_launch(names, warm_only=True):
    """dram bytes of the FIRST capture of each kernel (the warm iteration)."""
    tot, seen = 0.0, set()
    for d in out:
        for n in names:
            if n in d["kernel"] and n not in seen:
                seen.add(n)
                tot += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    return tot


src = f"profiles/{tag}_ncu_full_C2.txt (ncu --set full, tools/ncu_window.py C2)"
def per_call(names):
    """dram bytes of the first `names[n]` captures of each named kernel (one
    fused-match call launches the heat GEMM twice and the others once)."""
    tot, used = 0.0, {}
    for d in out:
        for n, lim in names.items():
            if n in d["kernel"] and used.get(n, 0) < lim:
                used[n] = used.get(n, 0) + 1
                tot += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    return tot


traffic = {
    "wnnm_scatter": {"bytes": per_launch(["gram_kernel", "eig_kernel", "apply_oz_kernel"]),
                     "unit": "bytes per launch (gram + eig + apply)", "source": src},
    "heat_map": {"bytes": per_launch(["heat_gemm_kernel"]), "unit": "bytes per launch",
                 "source": src},
    "topk": {"bytes": per_launch(["topk_kernel"]), "unit": "bytes per launch", "source": src},
    "heat_topk": {"bytes": per_call({"exemplar_pack_kernel": 1, "heat_gemm_kernel": 2,
                                     "exemplar_thr_kernel": 1, "sample_thr_kernel": 1,
                                     "topk_cand_kernel": 1}),
                  "unit": "bytes per call (pack + sampled pre-pass + candidate GEMM + list top-K)",
                  "source": src},
}
(prof / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
summ = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), launches],
                      capture_output=True, text=True).stdout
(prof / f"{tag}_launches_C2.md").write_text(
    f"# Launch list, {tag} -- `python bench.py --steps 2 --warmup 3 --no-cpu-baseline` (C2)\n\n"
    "Command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "
    "launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline` on one B200 "
    "(gpurun). Covers warm-up + timed + e2e solves. Cold-cache serialised per-launch times: "
    "compare shares, not absolutes.\n\n```\n" + summ + "```\n")
print(json.dumps(traffic, indent=1))
