"""One rank of a sharded gap_solve (tests/test_gpu_multirank.py).

Launched once per rank with RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT in
the environment; every rank uses cuda:0 and the ``gloo`` process group (its
all-reduce stages CUDA tensors through host memory, so ranks sharing one GPU
never wait on each other's kernels). Writes x, the residuals and every
refresh's (anchors, positions) to ``<out>.rank<r>.npz``.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def main():
    out, config, iters = sys.argv[1], sys.argv[2], int(sys.argv[3])
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    import paper_2301_03047_b200 as G
    from paper_2301_03047_b200 import workloads
    wl = workloads.make(config)
    cfg = G.SolverConfig(max_iters=iters, match=wl.match)
    trace = []
    x, rep = G.gap_solve(workloads.operator_for(wl), wl.y, cfg, process_group=dist.group.WORLD,
                         trace=trace)
    rank = dist.get_rank()
    arrs = {"x": x, "resid": np.array([r["residual"] for r in rep.rows]),
            "nref": np.array(len(trace))}
    for j, (a, p) in enumerate(trace):
        arrs[f"anchors_{j}"] = np.asarray(a, dtype=np.int32)
        arrs[f"positions_{j}"] = np.asarray(p, dtype=np.int32)
    np.savez(f"{out}.rank{rank}.npz", **arrs)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
