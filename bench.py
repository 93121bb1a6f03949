"""GLR hot-path benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config C2] [--no-cpu-baseline]

A step is one full GAP-GLR reconstruction of the workload (BASELINE.json
configs[1] = C2 by default: 1024x1024x24 CACTI, 50 iterations, 8x8 patches,
4096 exemplars, K = 64 — refreshes every 5 iterations included). The metric
is GLR iterations per second of the whole job:

  value  device-resident: measurement and masks already in HBM, CUDA events,
         barrier + synchronize on both sides, max over ranks;
  e2e    the public API gap_solve(op, y, cfg) with host (pinned) numpy inputs,
         H2D of y/masks/gram and D2H of the result inside the timed region.

N > 1 (torchrun): exemplars shard over the ranks of one solve with an int64
NCCL all-reduce of the aggregation numerator per iteration (strong scaling).
``--impl reference`` times the CPU oracle port (oracle/glr_oracle.py — the
reference's algorithm restated; the reference is pure Python and cannot
travel to the box) on a bounded sample of the same workload, extrapolated to
the full solve; only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GLR iters/s (C2 1024x1024x24 CACTI GAP-GLR, 50 it, 4096 exemplars, K=64)"


def metric_for(wl) -> str:
    """The headline metric string (C2) or its analogue for another config."""
    if wl.name == "C2":
        return METRIC
    h, w, c = wl.shape
    return (f"GLR iters/s ({wl.name} {h}x{w}x{c} {wl.kind.upper()} GAP-GLR, {wl.max_iters} it, "
            f"{wl.match.max_corners} max corners, K={wl.match.group_size})")
UNIT = "iters/s"
FP64_DMMA_PEAK = 37.1  # TFLOP/s, measured on B200 (tools/micro/dmma.cu, profiles/r01_fp64_peak.md)


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def _tc_peaks() -> dict:
    """Measured dense tcgen05 rates per kind (tools/micro/tc_peak.cu on a
    B200 of this pool, profiles/r02_tc_peak.json): {kind: TFLOP/s}."""
    p = ROOT / "profiles" / "r02_tc_peak.json"
    out = {}
    if p.exists():
        for line in p.read_text().splitlines():
            line = line.strip()
            if line.startswith("{"):
                d = json.loads(line)
                out[d["kind"].split()[0]] = float(d["tflops"])
    return out


def _fp4_peak(peaks) -> dict:
    """Peak for the heat map's kind::mxf4 MMAs: the measured microbenchmark
    rate when recorded, else 4 x the driver's measured bf16 rate (the dense
    fp4 : bf16 ratio, 9 : 2.25 PFLOP/s nominal)."""
    tc = _tc_peaks()
    if "e2m1" in tc:
        return {"tflops": tc["e2m1"], "kind": "measured tcgen05 kind::mxf4 dense rate "
                                              "(tools/micro/tc_peak.cu, profiles/r02_tc_peak.json)"}
    return {"tflops": 4.0 * peaks["bf16_tflops"], "kind": "fp4 (kind::mxf4) = 4 x measured bf16"}


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md clocks line)

class Clocks:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.path = Path(os.environ.get("TMPDIR", "/tmp")) / f"glr_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self, device_index: int = 0):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or f[0] != str(device_index):
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port on a bounded sample, extrapolated

CPU_CHECK = ("profiles/r02_cpu_baseline_check_C1.json: at C1 this extrapolation landed "
             "within +6.6 % of the unmodified reference gap_solve timed on the same host")


def cpu_full(wl) -> dict:
    """The oracle port's FULL solve (no extrapolation), for configurations
    whose whole CPU solve takes minutes (C1)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import glr_oracle as O
    mc = wl.match
    op = O.Operator(wl.kind, masks=wl.masks) if wl.kind != "fourier" else \
        O.Operator("fourier", mask=wl.masks, channels=wl.scene.shape[2])
    t0 = time.perf_counter()
    O.gap_solve(op, wl.y, wl.max_iters, patch_size=mc.patch_size, group_size=mc.group_size,
                max_corners=mc.max_corners, exemplar_stride=mc.exemplar_stride,
                clip=wl.kind != "fourier", init=wl.init)
    t = time.perf_counter() - t0
    return {"value": wl.max_iters / t, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "extrapolated": False,
            "sample": (f"oracle/glr_oracle.py: the full {wl.max_iters}-iteration {wl.name} solve "
                       f"({t:.1f} s, all host BLAS threads), not extrapolated")}


def cpu_sample(wl, n_heat=8, n_groups=64) -> dict:
    """Times the oracle on one slice of every stage of the solve and
    extrapolates to the full reconstruction (iters/s)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import glr_oracle as O
    mc = wl.match
    p, k = mc.patch_size, mc.group_size
    sep = mc.sep
    if wl.kind == "fourier":
        op = O.Operator("fourier", mask=wl.masks, channels=wl.scene.shape[2])
    else:
        op = O.Operator(wl.kind, masks=wl.masks)
    t0 = time.perf_counter()
    x = O.init_x(op, wl.y, wl.init)
    t_init = time.perf_counter() - t0
    t0 = time.perf_counter()
    anchors = O.build_exemplars(x, p, mc.max_corners, mc.nms, mc.corner_quality,
                                mc.exemplar_stride)
    t_exemplars = time.perf_counter() - t0
    n = len(anchors)
    t0 = time.perf_counter()
    gh, gv = O.sobel_gradients(x)
    maps = O.binarize_gradients(gh, gv, mc.edge_threshold)
    t_edges = time.perf_counter() - t0
    sub = anchors[:n_heat]
    t0 = time.perf_counter()
    heat = O.similarity_heatmap(maps, sub, p)
    t_heat = (time.perf_counter() - t0) / len(sub)
    t0 = time.perf_counter()
    positions, _ = O.match_positions(heat, sub, k, sep)
    t_topk = (time.perf_counter() - t0) / len(sub)
    groups = [positions[i % len(positions)] for i in range(n_groups)]
    sigma = O.sigma_at(0, wl.max_iters)
    t0 = time.perf_counter()
    acc = np.zeros_like(x)
    cnt = np.zeros_like(x)
    for pos in groups:
        den = O.wnnm_prox(O.gather_group(x, pos, p), sigma)
        O.scatter_group(acc, cnt, den, pos, p)
    t_group = (time.perf_counter() - t0) / n_groups
    t0 = time.perf_counter()
    z = x + op.adjoint(O.safe_div(wl.y - op.forward(x), op.gram))
    np.linalg.norm((wl.y - op.forward(np.clip(z, -0.5, 1.5))).ravel())
    t_proj = time.perf_counter() - t0
    iters = wl.max_iters
    n_refresh = -(-iters // 5)
    total = (t_init + n_refresh * (t_exemplars + t_edges + n * (t_heat + t_topk))
             + iters * (n * t_group + t_proj))
    sampled = t_init + t_exemplars + t_edges + len(sub) * (t_heat + t_topk) \
        + n_groups * t_group + t_proj
    return {
        "value": iters / total, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
        "extrapolated": True,
        "sample": (f"EXTRAPOLATED: oracle/glr_oracle.py on {wl.name}: full exemplar detection + "
                   f"edges, heat map + top-K for {len(sub)} of {n} exemplars, "
                   f"gather+WNNM+scatter for {n_groups} groups, one projection ({sampled:.1f} s "
                   f"sampled); extrapolated to {n_refresh} refreshes + {iters} iterations = "
                   f"{total:.0f} s per solve ({CPU_CHECK})"),
        "stage_s": {"exemplars": t_exemplars, "edges": t_edges, "heat_per_exemplar": t_heat,
                    "topk_per_exemplar": t_topk, "group": t_group, "projection": t_proj},
        "n_exemplars": n,
    }


# ---------------------------------------------------------------------------

def run_reference(args, rank):
    if rank != 0:
        return
    from paper_2301_03047_b200 import workloads
    wl = workloads.make(args.config)
    vals, details = [], None
    for _ in range(args.warmup):
        cpu_sample(wl, n_heat=2, n_groups=8)
    t_start = time.perf_counter()
    for _ in range(args.steps):
        details = cpu_sample(wl)
        vals.append(details["value"])
    wall = time.perf_counter() - t_start
    v = float(statistics.mean(vals))
    line = {
        "metric": metric_for(wl), "value": v, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(args, wl, details["n_exemplars"]),
        "cpu_baseline": {k: details[k] for k in ("value", "unit", "cores", "kind", "extrapolated",
                                                  "sample")},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config(args, wl, n_exemplars):
    h, w, c = wl.shape
    return {"workload": f"{wl.name}: {wl.kind.upper()} {h}x{w}x{c}, GAP-GLR {wl.max_iters} it, "
                        f"P={wl.match.patch_size}, K={wl.match.group_size}, "
                        f"max_corners={wl.match.max_corners}, "
                        f"exemplar_stride={wl.match.exemplar_stride}, init={wl.init}",
            "exemplars": n_exemplars, "iters_per_step": wl.max_iters,
            "parallelism": f"exemplar-shard x{args.gpus}",
            "l2": _l2_note(wl, n_exemplars, _fused_auto(wl)),
            "seed": 0}


L2_BYTES = 126 * 2 ** 20


def _working_set(wl, n_exemplars):
    """(x bytes, heat-map bytes per refresh) of a workload"""
    h, w, c = wl.shape
    p = wl.match.patch_size
    return h * w * c * 8, n_exemplars * (h - p + 1) * (w - p + 1) * 2


def _needs_flush(wl, n_exemplars):
    xb, hb = _working_set(wl, n_exemplars)
    return hb + 4 * xb < 2 * L2_BYTES


def _fused_auto(wl) -> bool:
    """GlrEngine's automatic choice of the fused heat map + top-K (engine.py:
    the dense u16 map would exceed 4 GB)."""
    mc = wl.match
    h, w, _ = wl.shape
    p, g = mc.patch_size, 3 * mc.exemplar_stride
    n_est = mc.max_corners + ((h - p) // g + 1) * ((w - p) // g + 1)
    return n_est * (h - p + 1) * (w - p + 1) * 2 > (4 << 30)


def _l2_note(wl, n_exemplars, fused=False):
    xb, hb = _working_set(wl, n_exemplars)
    if fused:  # no dense heat map: candidate lists (glr_heat_topk)
        return (f"inputs > L2 (x {xb / 1e6:.0f} MB per array; fused matching: candidate lists "
                f"instead of a {hb / 1e9:.2f} GB dense heat map per refresh)")
    if _needs_flush(wl, n_exemplars):
        return (f"L2 flushed between timed steps (256 MB write outside the per-step events); "
                f"x {xb / 1e6:.0f} MB, heat map {hb / 1e6:.0f} MB per refresh")
    return f"inputs > L2 (x {xb / 1e6:.0f} MB, heat map {hb / 1e9:.2f} GB per refresh)"


def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        pg = dist.group.WORLD
    import paper_2301_03047_b200 as G
    from paper_2301_03047_b200 import _device as D, _native as N, workloads
    from paper_2301_03047_b200.solvers import GapRunner
    wl = workloads.make(args.config)
    h, w, c = wl.shape
    cfg = wl.solver_config()
    op = workloads.operator_for(wl)
    runner = GapRunner(op, cfg, process_group=pg)
    y_d = runner.dop.upload_y(wl.y)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        runner.run(y_d)
    torch.cuda.synchronize()
    n_ex = runner.eng.n
    # ---- timed region: device-resident solves ----
    clocks = Clocks() if rank == 0 else None
    runner.eng.timing = []
    barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    launches0 = N.launch_count
    N.call("glr_eig_work", None, 1)  # clear the eigen step's work counters
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda") \
        if _needs_flush(wl, n_ex) else None
    ev = []
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1)  # evict the previous step's working set from L2
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        runner.run(y_d)
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    barrier()
    launches = N.launch_count - launches0  # fill_ is a torch kernel, not counted
    import ctypes as _C
    _ew = (_C.c_uint64 * 3)()
    N.call("glr_eig_work", _C.addressof(_ew), 0)
    eig_work = [int(v) for v in _ew]  # this rank's groups, super-rounds, first-order finishes
    ck = clocks.stop(local_rank) if clocks else None
    ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    timing = runner.eng.timing
    runner.eng.timing = None
    kern = {}
    for (name, nb), a, b in timing:
        d = kern.setdefault(name, {"launches": 0, "ms": 0.0, "units": 0})
        d["launches"] += 1
        d["ms"] += a.elapsed_time(b)
        d["units"] += nb
    iters_total = args.steps * wl.max_iters
    value = iters_total / (ms / 1e3)

    # ---- e2e: public API with host inputs ----
    import torch as _t
    pin = lambda a: _t.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    y_host = pin(wl.y)
    op_host = workloads.operator_for(wl)
    if wl.kind != "fourier":
        op_host.meta["masks"] = pin(op_host.meta["masks"])
        op_host.gram_diag = pin(op_host.gram_diag)
        if "masks_u8" in op_host.meta:
            # binary masks travel as their 1-byte copy (operators._binary_u8);
            # CACTI's gram is then formed on device
            op_host.meta["masks_u8"] = pin(op_host.meta["masks_u8"])
            op_host.meta["masks_u8_of"] = id(op_host.meta["masks"])
            h2d = y_host.nbytes + op_host.meta["masks_u8"].nbytes + \
                (0 if wl.kind == "cacti" else op_host.gram_diag.nbytes)
        else:
            h2d = y_host.nbytes + op_host.meta["masks"].nbytes + op_host.gram_diag.nbytes
    else:
        op_host.meta["mask"] = pin(op_host.meta["mask"])
        h2d = 2 * y_host.nbytes + op_host.meta["mask"].nbytes
    d2h = h * w * c * 8 + wl.max_iters * 8
    e2e_steps = max(1, min(args.steps, 3))
    G.gap_solve(op_host, y_host, cfg, process_group=pg)  # allocator warm
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        G.gap_solve(op_host, y_host, cfg, process_group=pg)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = e2e_steps * wl.max_iters / e2e_s

    if rank == 0:
        peaks, peak_src = _peaks()
        mp = wl.match.patch_size
        oh, ow = h - mp + 1, w - mp + 1
        roof = {}
        for hk in ("heat_topk", "heat_map"):
            if hk not in kern:
                continue
            d = kern[hk]
            # heat_topk = the fused heat GEMM + candidate top-K; its roofline is
            # the GEMM's algorithmic work over the fused time
            flops = 2.0 * oh * ow * 4 * c * mp * mp * d["units"] / d["launches"]
            avg_s = d["ms"] / d["launches"] / 1e3
            ach = flops / avg_s / 1e12
            fp4 = _fp4_peak(peaks)
            pk = fp4["tflops"]
            roof[hk] = {"bound": "tensor", "achieved": ach, "peak": pk,
                        "unit": "TFLOP/s", "frac": ach / pk,
                        "peak_kind": fp4["kind"],
                        "avg_ms": d["ms"] / d["launches"]}
        if "wnnm_scatter" in kern:
            d = kern["wnnm_scatter"]
            m = mp * mp * c
            k = wl.match.group_size
            # algorithmic fp64 work per group: symmetric Gram m*K*(K+1) + apply
            # 2*m*K^2 flops (the O(K^3) eigen step is not counted); the Gram runs
            # on the fp64 tensor cores (DMMA), the apply's fp64 product exactly
            # emulated on the int8 tensor cores (split-integer / Ozaki, six digit
            # slices); peak = measured DMMA rate (profiles/r01_fp64_peak.md), so
            # frac is fp64-equivalent work over the fp64 tensor peak
            flops = (m * k * (k + 1) + 2.0 * m * k * k) * d["units"] / d["launches"]
            avg_s = d["ms"] / d["launches"] / 1e3
            ach = flops / avg_s / 1e12
            byts = 2.0 * m * k * 8 * d["units"] / d["launches"]
            # The eigen step's work is data dependent and counted by the library
            # (glr_eig_work): per group the warm-start products G' = Vp^T G Vp
            # (2 x 2*64^3) and Wm = V diag V^T (one product, two with the
            # first-order finish); per 4x4 block super-round the G update
            # (256 blocks x 2 x 4^3 FMA) and the V update (16 quads x 64 rows x
            # 16 FMA) = 98.3 kflop, nominal (blocks of unrotated quads are skipped).
            eg = max(eig_work[0], 1)
            sr_per_group = eig_work[1] / eg
            fin_frac = eig_work[2] / eg
            eig_flops_group = (3.0 + fin_frac) * 2.0 * 64 ** 3 + sr_per_group * 98304.0
            eig_flops = eig_flops_group * d["units"] / d["launches"]
            ach_all = (flops + eig_flops) / avg_s / 1e12
            roof["wnnm_scatter"] = {"bound": "tensor", "achieved": ach_all,
                                    "peak": FP64_DMMA_PEAK,
                                    "unit": "TFLOP/s", "frac": ach_all / FP64_DMMA_PEAK,
                                    "peak_kind": "fp64-equivalent work (Gram + eigen step + apply) vs "
                                                 "the measured fp64 DMMA peak (Gram and the eigen "
                                                 "step's products on DMMA, rotations on the fp64 "
                                                 "pipe, apply on int8 tcgen05 as an exact "
                                                 "split-integer product)",
                                    "avg_ms": d["ms"] / d["launches"],
                                    "achieved_gram_apply_only": ach,
                                    "frac_gram_apply_only": ach / FP64_DMMA_PEAK,
                                    "eig": {"super_rounds_per_group": sr_per_group,
                                            "sweeps_per_group": sr_per_group / 21.0,
                                            "first_order_finish_frac": fin_frac,
                                            "gflop_per_launch": eig_flops / 1e9,
                                            "gram_apply_gflop_per_launch": flops / 1e9},
                                    "hbm_gbs": byts / avg_s / 1e9}
        if "topk" in kern:
            d = kern["topk"]
            byts = 2.0 * oh * ow * d["units"] / d["launches"]  # the u16 heat rows, read once
            avg_s = d["ms"] / d["launches"] / 1e3
            ach = byts / avg_s / 1e9
            roof["topk"] = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"],
                            "unit": "GB/s", "frac": ach / peaks["hbm_gbs"],
                            "avg_ms": d["ms"] / d["launches"]}
        dominant = max(kern, key=lambda n: kern[n]["ms"]) if kern else None
        roofline = dict(roof.get(dominant, {})) if dominant else {}
        traffic = None
        prof = ROOT / "profiles" / "ncu_traffic.json"
        if prof.exists() and dominant and args.config == "C2":  # the capture is C2's
            traffic = json.loads(prof.read_text()).get(dominant)
        roofline["traffic"] = traffic
        roofline["kernel"] = dominant
        roofline["peak_source"] = f"{peak_src} (MEASURED_PEAKS.json)" if peak_src == "measured" \
            else "fallback (B200_PROFILING.md)"
        line = {
            "metric": metric_for(wl), "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64+e2m1+s8",
            "data": "synthetic (seeded generator, workloads.py)",
            "config": _config(args, wl, n_ex),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": e2e_steps},
            "gpu_launches": int(launches),
            "roofline": roofline,
            "kernels": {n: {"launches": d["launches"], "ms_total": round(d["ms"], 3),
                            "share_of_step": round(d["ms"] / ms, 4),
                            **({k2: v for k2, v in roof[n].items()} if n in roof else {})}
                        for n, d in kern.items()},
            "clocks": ck,
        }
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_full(wl) if wl.name == "C1" else cpu_sample(wl)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind",
                                                       "extrapolated", "sample")}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_b200_c5(args, rank, world, local_rank):
    """C5, the isolated-stage sweep (BASELINE.json configs[4]): no solver
    loop. A step = one pass of the stages over the seeded 2048x2048x1 image:
    exemplar detection, edge stack, heat map + exact top-K for every exemplar
    of this rank's shard, then one batched WNNM + fixed-point aggregation
    (+ all-reduce) and the normalisation. metric = matches/s = N x M
    exemplar-position scores per second of the whole step (N exemplars over
    all ranks, M = (H-P+1)(W-P+1) positions); exemplars shard over the ranks
    (strong scaling, the image is replicated)."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        pg = dist.group.WORLD
    import paper_2301_03047_b200 as G
    from paper_2301_03047_b200 import _device as D, _native as N, workloads
    from paper_2301_03047_b200.engine import GlrEngine
    wl = workloads.make("C5")
    h, w, c = wl.shape
    p, n_req = args.c5_patch, args.c5_exemplars
    mc = G.MatchConfig(patch_size=p, group_size=64, max_corners=n_req, exemplar_stride=4096)
    eng = GlrEngine((h, w, c), mc, process_group=pg)
    x_host = torch.from_numpy(np.ascontiguousarray(wl.scene)).pin_memory()
    x_d = x_host.to("cuda")
    z_d = torch.empty_like(x_d)
    sigma = 0.05

    def step(x):
        eng.refresh(x)
        eng.regularize(x, sigma)
        N.call("glr_normalize", eng.acc.data_ptr(), eng.cnt.data_ptr(), x.data_ptr(), h, w, c,
               eng.frac, z_d.data_ptr(), D.stream())
        eng.consumed()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step(x_d)
    torch.cuda.synchronize()
    clocks = Clocks() if rank == 0 else None
    eng.timing = []
    barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    launches0 = N.launch_count
    ev = []
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        step(x_d)
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    barrier()
    launches = N.launch_count - launches0
    ck = clocks.stop(local_rank) if clocks else None
    ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    kern = {}
    for (name, nb), a, b in eng.timing:
        d = kern.setdefault(name, {"launches": 0, "ms": 0.0, "units": 0})
        d["launches"] += 1
        d["ms"] += a.elapsed_time(b)
        d["units"] += nb
    eng.timing = None
    n_ex = eng.n
    M = (h - p + 1) * (w - p + 1)
    value = args.steps * n_ex * M / (ms / 1e3)
    # e2e: host image in (pinned H2D) and the match positions out (D2H) per step
    pos_host = torch.empty((n_ex, mc.group_size, 2), dtype=torch.int32, pin_memory=True)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 3))
    for _ in range(e2e_steps):
        xd = x_host.to("cuda", non_blocking=True)
        step(xd)
        pos_host.copy_(eng.positions[:n_ex], non_blocking=True)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    if rank == 0:
        peaks, peak_src = _peaks()
        fp4 = _fp4_peak(peaks)
        roof = {}
        for hk in ("heat_map", "heat_topk"):
            # heat_topk: the fused heat GEMM + candidate top-K (one-channel
            # images); its roofline is the GEMM's algorithmic work over the
            # fused time
            if hk not in kern:
                continue
            d = kern[hk]
            flops = 2.0 * M * 4 * c * p * p * d["units"] / d["launches"]
            ach = flops / (d["ms"] / d["launches"] / 1e3) / 1e12
            roof[hk] = {"bound": "tensor", "achieved": ach, "peak": fp4["tflops"],
                        "unit": "TFLOP/s", "frac": ach / fp4["tflops"],
                        "peak_kind": fp4["kind"], "avg_ms": d["ms"] / d["launches"]}
        if "topk" in kern:
            d = kern["topk"]
            ach = 2.0 * M * d["units"] / d["launches"] / (d["ms"] / d["launches"] / 1e3) / 1e9
            roof["topk"] = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"],
                            "unit": "GB/s", "frac": ach / peaks["hbm_gbs"],
                            "avg_ms": d["ms"] / d["launches"]}
        dominant = max(kern, key=lambda k: kern[k]["ms"]) if kern else None
        roofline = dict(roof.get(dominant, {})) if dominant else {}
        roofline.update({"kernel": dominant, "traffic": None,
                         "peak_source": f"{peak_src} (MEASURED_PEAKS.json)"})
        line = {
            "metric": f"C5 matches/s (2048x2048x1 stage pass: exemplars, heat map + top-K, WNNM "
                      f"+ aggregation; P={p}, K=64)",
            "value": value, "unit": "matches/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64+e2m1+s8",
            "data": "synthetic (seeded generator, workloads.py)",
            "config": {"workload": f"C5: 2048x2048x1 blob+texture, P={p}, K=64, "
                                   f"max_corners={n_req} (+1 grid anchor)",
                       "exemplars": n_ex, "positions": M,
                       "parallelism": f"exemplar-shard x{world}",
                       "l2": "inputs > L2 (heat map "
                             f"{n_ex * M * 2 / 1e9:.1f} GB per step)", "seed": 0},
            "e2e": {"value": e2e_steps * n_ex * M / e2e_s, "unit": "matches/s",
                    "h2d_bytes_per_step": int(x_host.numel() * 8),
                    "d2h_bytes_per_step": int(pos_host.numel() * 4), "steps": e2e_steps},
            "groups_per_s": args.steps * n_ex / (ms / 1e3),
            "gpu_launches": int(launches),
            "roofline": roofline,
            "kernels": {k: {"launches": d["launches"], "ms_total": round(d["ms"], 3),
                            "share_of_step": round(d["ms"] / ms, 4), **roof.get(k, {})}
                        for k, d in kern.items()},
            "clocks": ck,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--c5-patch", type=int, default=8, choices=[8, 12],
                    help="C5 stage sweep: patch size")
    ap.add_argument("--c5-exemplars", type=int, default=16384,
                    help="C5 stage sweep: exemplar count (1024 / 4096 / 16384)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank "
                         f"per GPU (torchrun --nproc-per-node {args.gpus}) or drop WORLD_SIZE")
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if args.config == "C5":
        run_b200_c5(args, rank, world, local_rank)
        return
    run_b200(args, rank, world, local_rank)


def _spawn_ranks(args) -> int:
    """--gpus N without a launcher: re-exec this script under torchrun, one
    rank per GPU (127.0.0.1 rendezvous). Fails loudly when the box has fewer
    than N GPUs instead of running (and labelling) a smaller job."""
    import socket
    if args.impl != "reference":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, this box has "
                  f"{have}", file=sys.stderr, flush=True)
            return 3
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


if __name__ == "__main__":
    main()
