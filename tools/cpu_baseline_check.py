"""Validate the CPU baseline (bench.py cpu_sample) against the UNMODIFIED
reference on the same host (build container only: needs /root/reference).

For C1 (256x256x8, 30 GAP-GLR iterations) it times
  1. the reference's own gap_solve (glr.gap_solve, as shipped, ref=None),
  2. the oracle port's full gap_solve (oracle/glr_oracle.py),
  3. bench.cpu_sample's extrapolation (the port on a bounded sample),
and writes profiles/r02_cpu_baseline_check.json with the three iters/s
figures and their ratios (the extrapolation must land within +-25 % of the
reference's measured rate to be reported as its stand-in).

    PYTHONPATH=/root/reference/pkg/src python tools/cpu_baseline_check.py [C1]
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, os.environ.get("GLR_REFERENCE_SRC", "/root/reference/pkg/src"))

import glr  # noqa: E402  (the reference)
import glr_oracle as O  # noqa: E402
import bench  # noqa: E402
from paper_2301_03047_b200 import workloads  # noqa: E402


def main(name="C1"):
    wl = workloads.make(name)
    mc = wl.match
    out = {"config": name, "host": platform.processor() or platform.machine(),
           "cores": os.cpu_count(), "numpy": np.__version__}
    # 1. the reference, unmodified
    op = glr.cacti_operator(wl.masks) if wl.kind == "cacti" else glr.msfa_operator(wl.masks)
    cfg = glr.SolverConfig(regularizer="glr", max_iters=wl.max_iters, init=wl.init,
                           match=glr.MatchConfig(patch_size=mc.patch_size,
                                                 group_size=mc.group_size,
                                                 max_corners=mc.max_corners,
                                                 exemplar_stride=mc.exemplar_stride))
    t0 = time.perf_counter()
    glr.gap_solve(op, wl.y, cfg)
    t_ref = time.perf_counter() - t0
    out["reference_s"] = t_ref
    out["reference_iters_per_s"] = wl.max_iters / t_ref
    # 2. the oracle port, full solve
    t0 = time.perf_counter()
    O.gap_solve(O.Operator(wl.kind, masks=wl.masks), wl.y, wl.max_iters,
                patch_size=mc.patch_size, group_size=mc.group_size,
                max_corners=mc.max_corners, exemplar_stride=mc.exemplar_stride, init=wl.init)
    t_port = time.perf_counter() - t0
    out["port_full_s"] = t_port
    out["port_full_iters_per_s"] = wl.max_iters / t_port
    # 3. bench.py's bounded-sample extrapolation
    cs = bench.cpu_sample(wl)
    out["extrapolated_iters_per_s"] = cs["value"]
    out["extrapolated_sample"] = cs["sample"]
    out["ratio_port_full_vs_reference"] = out["port_full_iters_per_s"] / out["reference_iters_per_s"]
    out["ratio_extrapolated_vs_reference"] = cs["value"] / out["reference_iters_per_s"]
    print(json.dumps(out, indent=1))
    (ROOT / "profiles" / f"r02_cpu_baseline_check_{name}.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
