"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): one GAP-GLR solve that runs every hot kernel once per stage --
Sobel, corner response, batched greedy NMS (nms_batch_kernel), anchors, the
edge stack, the tcgen05 heat GEMM (CTA pair, TMA multicast), top-K, the
Gram / Jacobi eigen / split-integer apply (tcgen05 kind::i8) WNNM trio, the
fixed-point scatter and the GAP update -- at a shape small enough for the
instrumented run (64 x 64 x 8, P = 8, K = 64), then checks the result
against the oracle so a silently corrupted run also fails.

    compute-sanitizer --tool racecheck python tools/sanitize_small.py
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import glr_oracle as O  # noqa: E402  (checker only)
import paper_2301_03047_b200 as G  # noqa: E402
from paper_2301_03047_b200 import workloads  # noqa: E402

h, w, t = 64, 64, 8
scene = workloads.cacti_scene(h, w, t, seed=5)
masks = G.bernoulli_masks(h, w, t, seed=6)
y = O.masksum_forward(scene, masks)
mc = G.MatchConfig(patch_size=8, group_size=64, max_corners=24, exemplar_stride=6)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 6
x, _ = G.gap_solve(G.cacti_operator(masks), y, G.SolverConfig(max_iters=iters, match=mc))
xo, _, _ = O.gap_solve(O.Operator("cacti", masks=masks), y, iters, patch_size=8, group_size=64,
                       max_corners=24, exemplar_stride=6)
err = float(np.abs(x - xo).max())
print(f"sanitize workload: {h}x{w}x{t}, {iters} iterations, max|x - oracle| = {err:.2e}")
assert err <= 1e-6
