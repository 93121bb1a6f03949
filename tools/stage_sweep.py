"""Isolated-stage sweep (BASELINE.json configs[4]): global
matching (heat-map GEMM + exact top-K) and batched WNNM + aggregation on a
seeded 2048 x 2048 blob + texture image, patch 8 and 12, 1k / 4k / 16k
exemplars, K = 64, no solver loop. One JSON line per (P, N) with device
times (CUDA events on the launching stream, best of `--reps` after one
warm-up) and the roofline numbers of each stage:

  heat   2 M (4 C P^2) N flops (tcgen05 kind::mxf4; peak: measured mxf4 rate)
  top-K  2 M N bytes (one read of the u16 heat rows; peak measured HBM)
  WNNM   m K (K + 1) + 2 m K^2 flops per group (fp64 DMMA peak 37.1 TF/s)

Exemplars are the device Shi-Tomasi corners (max_corners = N) plus one grid
anchor (the engine's `glr` exemplar rule with a stride beyond the image).

    python tools/stage_sweep.py [--reps 3] [--out profiles/r01_stage_sweep_C5.json]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2301_03047_b200 as G  # noqa: E402
from paper_2301_03047_b200 import _device as D, workloads  # noqa: E402
from paper_2301_03047_b200.engine import GlrEngine  # noqa: E402

FP64_PEAK = 37.1


def peaks():
    import bench
    d, _ = bench._peaks()
    return d["hbm_gbs"], bench._fp4_peak(d)["tflops"]


def stage_times(eng, x_d, sigma):
    eng.timing = []
    eng.refresh(x_d)
    eng.regularize(x_d, sigma)
    torch.cuda.synchronize()
    out = {}
    for (name, nb), a, b in eng.timing:
        d = out.setdefault(name, [0.0, 0])
        d[0] += a.elapsed_time(b)
        d[1] += nb
    eng.timing = None
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--fused", action="store_true",
                    help="heat map + top-K fused (glr_heat_topk, sampled candidate floor)")
    ap.add_argument("--only", default=None, help="P:N pairs, e.g. 8:16384,12:4096")
    args = ap.parse_args()
    hbm, fp4 = peaks()
    wl = workloads.make("C5")
    h, w, c = wl.shape
    x_d = D.f64(wl.scene)
    lines = []
    combos = [(p, n) for p in (8, 12) for n in (1024, 4096, 16384)]
    if args.only:
        combos = [tuple(int(v) for v in c.split(":")) for c in args.only.split(",")]
    for p, n in combos:
        if True:
            mc = G.MatchConfig(patch_size=p, group_size=64, max_corners=n, exemplar_stride=4096)
            eng = GlrEngine((h, w, c), mc, low_memory_match=args.fused)
            best = None
            for r in range(args.reps + 1):  # first run = warm-up
                t = stage_times(eng, x_d, 0.05)
                if r and (best is None or sum(v[0] for v in t.values()) <
                          sum(v[0] for v in best.values())):
                    best = t
            N = eng.n
            M = (h - p + 1) * (w - p + 1)
            m = p * p * c
            k = mc.group_size
            if args.fused:
                heat_ms = best["heat_topk"][0]
                topk_ms = sum(best[k][0] for k in ("heat_map", "topk") if k in best)
            else:
                heat_ms = best["heat_map"][0]
                topk_ms = best["topk"][0]
            wn_ms = best["wnnm_scatter"][0]
            heat_tf = 2.0 * M * 4 * c * p * p * N / (heat_ms / 1e3) / 1e12
            topk_gbs = 2.0 * M * N / (topk_ms / 1e3) / 1e9 if topk_ms > 0 else 0.0
            wn_tf = (m * k * (k + 1) + 2.0 * m * k * k) * N / (wn_ms / 1e3) / 1e12
            line = {
                "workload": f"C5 stage sweep: 2048x2048x1, P={p}, K={k}", "P": p,
                "exemplars": N, "positions": M,
                "heat": {"ms": round(heat_ms, 3), "tflops": round(heat_tf, 1),
                         "frac": round(heat_tf / fp4, 3),
                         "matches_per_s": N * M / (heat_ms / 1e3)},
                "topk": {"ms": round(topk_ms, 3), "gbs": round(topk_gbs, 1),
                         "frac": round(topk_gbs / hbm, 3)},
                "groups_per_s": N / ((heat_ms + topk_ms) / 1e3),
                "wnnm": {"ms": round(wn_ms, 3), "tflops": round(wn_tf, 2),
                         "frac": round(wn_tf / FP64_PEAK, 3), "m": m},
                "peaks": {"fp4_tflops": fp4, "hbm_gbs": hbm, "fp64_tflops": FP64_PEAK},
                "heat_chunks": -(-N // eng.heat_chunk),
                "mode": ("fused heat+top-K (heat = fused kernel pair, topk = dense fallback "
                         f"for {eng.n_fallback} exemplars)") if args.fused else "dense map + top-K",
            }
            print(json.dumps(line), flush=True)
            lines.append(line)
            del eng
            torch.cuda.empty_cache()
    if args.out:
        Path(args.out).write_text("\n".join(json.dumps(x) for x in lines) + "\n")


if __name__ == "__main__":
    main()
