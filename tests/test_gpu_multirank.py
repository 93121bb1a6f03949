"""Sharded gap_solve on the product path (GPU): ranks of a ``gloo`` process
group (all on cuda:0) each run the heat map / top-K / WNNM of their exemplar
block and all-reduce the int64 numerator and int32 counter
(engine.GlrEngine._all_reduce). The result must be BITWISE equal
to the single-rank solve: integer sums are order-independent.

C1 (256x256x8, 10 iterations): refreshes at iterations 0 and 5 have 706 and
705 anchors, so the shards are uneven and change across the refresh (the
vcache re-index then crosses shard boundaries, glr_vcache_remap)."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2301_03047_b200")
from paper_2301_03047_b200 import workloads  # noqa: E402

WORKER = Path(__file__).resolve().parent / "helpers" / "multirank_worker.py"


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_ranks(world, out, config, iters):
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(WORKER), str(out), config, str(iters)],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(o.decode(errors="replace"))
        assert p.returncode == 0, "\n".join(logs)
    return [np.load(f"{out}.rank{r}.npz") for r in range(world)]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_solve_bitwise_equals_single_rank(world, tmp_path):
    wl = workloads.make("C1")
    iters = 10
    cfg = G.SolverConfig(max_iters=iters, match=wl.match)
    trace = []
    x1, rep1 = G.gap_solve(workloads.operator_for(wl), wl.y, cfg, trace=trace)
    res1 = np.array([r["residual"] for r in rep1.rows])
    assert len(trace) == 2
    n0, n1 = len(trace[0][0]), len(trace[1][0])
    ranks = _run_ranks(world, tmp_path / "solve", "C1", iters)
    for r, d in enumerate(ranks):
        assert int(d["nref"]) == 2
        for j, (a, p) in enumerate(trace):
            assert np.array_equal(d[f"anchors_{j}"], np.asarray(a)), (r, j)
            # positions_host assembles every rank's shard (integer all-reduce)
            # and restores the reference anchor order (sticky shards permute it)
            assert np.array_equal(d[f"positions_{j}"], np.asarray(p)), (r, j)
        bad = np.nonzero(d["resid"] != res1)[0]
        assert bad.size == 0, f"rank {r}: residuals differ from iteration {bad[:1].tolist()}"
        assert np.array_equal(d["x"], x1), f"rank {r}: x differs from the single-rank solve"
    # uneven shards that change across the refresh
    bounds = [[(n * q) // world for q in range(world + 1)] for n in (n0, n1)]
    sizes = [np.diff(b) for b in bounds]
    assert any(len(set(s.tolist())) > 1 for s in sizes) or bounds[0] != bounds[1]
