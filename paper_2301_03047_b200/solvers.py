"""GAP reconstruction loop with the global low-rank regularizer, on device
(reference: glr/solvers.py:35-354).

``gap_solve(op, y, cfg, ref=None)`` keeps the reference signature and
returns (x, ReconReport) as numpy float64. The iterate never leaves the GPU
inside the loop (engine.GlrEngine); the report's residuals, PSNRs and phase
times are gathered once at the end. ``process_group`` (extra keyword) shards
exemplars over the ranks of a torch.distributed group (one GPU per rank).
"""

from __future__ import annotations

import csv
import io
import json
import time
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _native as N
from .engine import DeviceOperator, GlrEngine
from .lowrank import WnnmParams
from .matching import MatchConfig
from .metrics import PSNR_CAP_DB, ssim

REGULARIZERS = ("glr", "nlr-bm", "nlr-corner-bm", "nlr-corner-uniform-bm", "tv")
ALGORITHMS = ("gap", "admm")


class SolverDivergenceError(RuntimeError):
    pass


@dataclass
class SolverConfig:
    """solvers.py:35-69."""

    algorithm: str = "gap"
    regularizer: str = "glr"
    max_iters: int = 200
    match_refresh_interval: int = 5
    sigma0: float = 0.10
    sigma_min: float = 0.003
    admm_rho: float = 0.01
    tv_weight: float = 0.05
    tv_iters: int = 20
    peak: float = 1.0
    init: str = "adjoint"
    seed: int = 0
    match: MatchConfig = field(default_factory=MatchConfig)
    wnnm: WnnmParams = field(default_factory=WnnmParams)

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if self.regularizer not in REGULARIZERS:
            raise ValueError(f"unknown regularizer {self.regularizer!r}")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.match_refresh_interval < 1:
            raise ValueError("match_refresh_interval must be >= 1")
        if not (self.sigma0 >= self.sigma_min > 0):
            raise ValueError("need sigma0 >= sigma_min > 0")
        if self.init not in ("adjoint", "zero", "interp"):
            raise ValueError(f"unknown init {self.init!r}")

    def sigma_at(self, k: int) -> float:
        """Geometric noise-level schedule, in absolute units (solvers.py:66-69)."""
        frac = self.sigma0 * (self.sigma_min / self.sigma0) ** (k / self.max_iters)
        return frac * self.peak


REPORT_COLUMNS = ["iteration", "residual", "psnr_db", "ssim",
                  "match_ms", "lowrank_ms", "projection_ms"]


@dataclass
class ReconReport:
    """solvers.py:76-98."""

    rows: list[dict] = field(default_factory=list)
    total_ms: float = 0.0
    diverged: bool = False

    def add(self, **kw) -> None:
        self.rows.append(kw)

    def to_csv(self) -> str:
        buf = io.StringIO()
        w = csv.DictWriter(buf, fieldnames=REPORT_COLUMNS)
        w.writeheader()
        for row in self.rows:
            w.writerow({k: row.get(k, "") for k in REPORT_COLUMNS})
        return buf.getvalue()

    def to_jsonl(self) -> str:
        return "\n".join(json.dumps(r) for r in self.rows) + "\n"

    @property
    def final_psnr(self) -> float | None:
        return self.rows[-1].get("psnr_db") if self.rows else None


@dataclass
class MatchState:
    """Group anchor positions reused between matching refreshes
    (solvers.py:145-151); ``engine`` holds the device state."""

    positions: list[list[tuple[int, int]]] | None = None
    last_refresh: int = -1
    last_match_ms: float = 0.0
    engine: object = None
    synced: object = None   # the positions list the engine's device copy holds


def _expected_y_shape(op) -> tuple:
    h, w = op.x_shape[:2]
    return (h, w) if op.kind == "fourier" else (h, w, 1)


def _check_measurement(op, y: np.ndarray) -> None:
    """solvers.py:350-354."""
    expect = _expected_y_shape(op)
    if y.shape != expect:
        raise ValueError(f"measurement shape {y.shape} does not match operator output {expect}")


def _check_divergence(residuals: list[float], y_norm: float) -> None:
    """solvers.py:272-281 — residual 10x above its minimum for 20 iterations."""
    if len(residuals) < 21:
        return
    best = max(min(residuals), 1e-6 * y_norm)
    tail = residuals[-20:]
    if all(r > 10.0 * best for r in tail):
        raise SolverDivergenceError(
            f"data residual grew 10x over its minimum ({best:.3e}) for 20 "
            f"consecutive iterations, last {tail[-1]:.3e}")


class _DivergenceGuard:
    """solvers.py:272-281 checked while the solve runs, as the reference does
    after every iteration (solvers.py:306-307), without a per-iteration host
    sync: each iteration's squared residual is copied to pinned host memory
    behind an event, and the check runs on every iteration whose copy has
    landed. A diverging solve stops a few iterations after the failing one at
    most and raises the reference's error for that iteration."""

    def __init__(self, resid_sq_d, iters: int, y_norm: float):
        t = D.torch()
        self.src = resid_sq_d
        self.host = t.empty((iters,), dtype=t.float64, pin_memory=True)
        self.events: list = []
        self.checked = 0
        self.y_norm = y_norm

    def push(self, it: int) -> None:
        t = D.torch()
        self.host[it:it + 1].copy_(self.src[it:it + 1], non_blocking=True)
        e = t.cuda.Event()
        e.record()
        self.events.append(e)
        self.poll()

    def poll(self, block: bool = False) -> None:
        while self.checked < len(self.events):
            e = self.events[self.checked]
            if block:
                e.synchronize()
            elif not e.query():
                return
            self.checked += 1
            if self.checked >= 21:
                res = np.sqrt(self.host[:self.checked].numpy()).tolist()
                _check_divergence(res, self.y_norm)


def _init_device(dop: DeviceOperator, y_d, cfg: SolverConfig):
    t = D.torch()
    x = D.zeros(dop.shape, t.float64)
    dop.init_x(y_d, x, cfg.init)
    return x


def regularize_dispatch(x: np.ndarray, cfg: SolverConfig, state: MatchState,
                        iteration: int = 0, sigma: float | None = None) -> np.ndarray:
    """solvers.py:170-210 — nonlocal regularizer with cached match positions
    ("glr" global matching, "nlr-*" block matching) or the TV prox."""
    x = np.asarray(x, dtype=np.float64)
    if cfg.regularizer == "tv":
        state.last_match_ms = 0.0
        return tv_denoise(x, cfg.tv_weight, cfg.tv_iters)
    sigma = cfg.sigma_at(iteration) if sigma is None else sigma
    WnnmParams(c_weight=cfg.wnnm.c_weight, eps=cfg.wnnm.eps, noise_sigma=sigma)
    eng = state.engine
    if eng is None or eng.shape != x.shape or eng.regularizer != cfg.regularizer:
        eng = GlrEngine(x.shape, cfg.match, cfg.peak, cfg.wnnm.c_weight, cfg.wnnm.eps,
                        regularizer=cfg.regularizer)
        state.engine = eng
    x_d = D.f64(x)
    refresh = (state.positions is None
               or iteration - state.last_refresh >= cfg.match_refresh_interval)
    if refresh:
        t0 = time.perf_counter()
        n = eng.refresh(x_d)
        if n:
            _, pos, _ = eng.positions_host()
            state.positions = [[tuple(q) for q in g] for g in pos.tolist()]
        else:
            state.positions = []
        state.synced = state.positions
        state.last_refresh = iteration
        D.torch().cuda.synchronize()
        state.last_match_ms = (time.perf_counter() - t0) * 1e3
    else:
        state.last_match_ms = 0.0
        if state.positions and (state.synced is not state.positions
                                or eng.n != len(state.positions)):
            # re-gather at the caller's cached positions (solvers.py:204-207):
            # a state built or edited outside this engine is uploaded first
            pos = np.asarray(state.positions, dtype=np.int32).reshape(-1, eng.k, 2)
            if pos.shape[0] > eng.max_anchors:
                raise ValueError(f"{pos.shape[0]} cached groups exceed the engine's "
                                 f"{eng.max_anchors} anchors")
            eng.set_positions(pos[:, 0, :], pos)
            state.synced = state.positions
    if not state.positions:
        return x.copy()
    eng.regularize(x_d, sigma)
    z = D.empty(x.shape, D.torch().float64)
    h, w, c = x.shape
    N.call("glr_normalize", eng.acc.data_ptr(), eng.cnt.data_ptr(), x_d.data_ptr(), h, w, c,
           eng.frac, z.data_ptr(), D.stream())
    eng.consumed()
    return D.host(z)


class GapRunner:
    """A prepared device operator + GLR engine for repeated GAP solves: the
    solver state is allocated once and a solve is `run(y_d)` on a device
    measurement (bench.py times this; gap_solve wraps it)."""

    def __init__(self, op, cfg: SolverConfig, process_group=None):
        t = D.torch()
        self.cfg = cfg
        self.dop = DeviceOperator(op)
        h, w, c = self.dop.shape
        self.tv = None
        if cfg.regularizer == "tv":
            # TV prox on device (solvers.py:121-139); no matching, no engine
            self.eng = _TvState(h, w)
            self.tv = TvProx(self.dop.shape, cfg.tv_weight, cfg.tv_iters)
        else:
            self.eng = GlrEngine(op.x_shape, cfg.match, cfg.peak, cfg.wnnm.c_weight,
                                 cfg.wnnm.eps, process_group=process_group,
                                 regularizer=cfg.regularizer)
        self.xa = D.empty(self.dop.shape, t.float64)
        self.xb = D.empty(self.dop.shape, t.float64)
        self.resid_sq = D.zeros((cfg.max_iters,), t.float64)
        self.sq = D.zeros((cfg.max_iters,), t.float64)
        self.sq_ws = D.empty((N.query("glr_gap_workspace", 1, 1),), t.uint8)
        self.events = None

    def sq_err(self, x, ref_d, it):
        n_el = int(np.prod(self.dop.shape))
        N.call("glr_sq_err", x.data_ptr(), ref_d.data_ptr(), n_el, float(self.cfg.peak),
               self.sq[it:it + 1].data_ptr(), self.sq_ws.data_ptr(), D.stream())

    def record_metrics(self, x, ref_d, it):
        """PSNR numerator and SSIM of clip(x, 0, peak) vs ref on device (f3:
        _record solvers.py:257-269 without a per-iteration host copy)."""
        t = D.torch()
        self.sq_err(x, ref_d, it)
        h, w, c = self.dop.shape
        if h < 11 or w < 11:
            return
        if getattr(self, "ssim_sum", None) is None:
            self.ssim_sum = D.zeros((self.cfg.max_iters,), t.float64)
            self.ssim_ws = D.empty((N.query("glr_ssim_workspace", h, w, c),), t.uint8)
            ax = np.arange(11) - 5.0
            g = np.exp(-(ax ** 2) / (2.0 * 1.5 ** 2))
            self._ssim_taps = np.ascontiguousarray(g / g.sum())
        taps = self._ssim_taps.ctypes.data_as(N.C.POINTER(N.C.c_double))
        N.call("glr_ssim", x.data_ptr(), ref_d.data_ptr(), h, w, c, float(self.cfg.peak), 1,
               taps, 11, self.ssim_sum[it:it + 1].data_ptr(), self.ssim_ws.data_ptr(), D.stream())

    def ssim_host(self):
        """Per-iteration SSIM values (one D2H at the end of the solve)."""
        h, w, c = self.dop.shape
        if getattr(self, "ssim_sum", None) is None:
            return None
        return D.host(self.ssim_sum) / float(c * (h - 10) * (w - 10))

    def run(self, y_d, positions_override=None, trace=None, on_iter=None, events=False,
            guard: _DivergenceGuard | None = None):
        """One full GAP-GLR solve (solvers.py:284-308) on device; returns the
        final iterate (device tensor, before the final [0, peak] clip).
        ``guard`` runs the divergence check as iterations complete."""
        t = D.torch()
        cfg, dop, eng = self.cfg, self.dop, self.eng
        iters = cfg.max_iters
        x, x_next = self.xa, self.xb
        dop.init_x(y_d, x, cfg.init)
        # a fresh solve: no match state and no eigenvector warm start carried
        # over from a previous run() (gap_solve always starts cold)
        eng.has_positions = False
        eng.vcache_valid = False
        eng.warm = 0
        lo, hi = -0.5 * cfg.peak, 1.5 * cfg.peak
        self.events = ([[t.cuda.Event(enable_timing=True) for _ in range(4)]
                        for _ in range(iters)] if events else None)
        last = -1
        refresh_no = 0
        for it in range(iters):
            ev = self.events[it] if events else None
            if ev:
                ev[0].record()
            sigma = cfg.sigma_at(it)
            if self.tv is None and ((not eng.has_positions)
                                    or it - last >= cfg.match_refresh_interval):
                if positions_override is not None:
                    anc, pos = positions_override[refresh_no]
                    eng.set_positions(np.asarray(anc), np.asarray(pos))
                else:
                    eng.refresh(x)
                if trace is not None:
                    a, pz, _ = eng.positions_host()
                    trace.append((a.tolist(), pz.tolist()))
                last = it
                refresh_no += 1
            if ev:
                ev[1].record()
            if self.tv is not None:
                z = self.tv(x)
                if ev:
                    ev[2].record()
                dop.gap_update(None, None, 0, z, y_d, lo, hi, x_next, self.resid_sq[it:it + 1],
                               eng.gap_ws)
            else:
                has = eng.regularize(x, sigma)
                if ev:
                    ev[2].record()
                dop.gap_update(eng.acc if has else None, eng.cnt if has else None, eng.frac, x,
                               y_d, lo, hi, x_next, self.resid_sq[it:it + 1], eng.gap_ws)
                if has:
                    eng.consumed()
            if ev:
                ev[3].record()
            x, x_next = x_next, x
            if on_iter is not None:
                on_iter(it, x)
            if guard is not None:
                guard.push(it)
        if guard is not None:
            guard.poll(block=True)
        return x


def _ssim_values(runner, ref):
    """Device SSIM per iteration; the host formula only for images below the
    11x11 window (where the reference raises, metrics.py:71-72)."""
    v = runner.ssim_host()
    if v is None:  # image smaller than the window: the reference's error path
        ssim(ref, ref, 1.0)
    return v


def _final_host(runner, x) -> np.ndarray:
    """The solver's return value: clip(x, 0, peak) (solvers.py:307) computed on
    device into the runner's spare iterate buffer, then one pinned D2H copy."""
    if not runner.dop.clip:
        return D.host_pinned(x)
    spare = runner.xb if x.data_ptr() == runner.xa.data_ptr() else runner.xa
    N.call("glr_lincomb", x.data_ptr(), 1.0, None, 0.0, None, 0.0, int(x.numel()), 1, 0.0,
           float(runner.cfg.peak), spare.data_ptr(), D.stream())
    return D.host_pinned(spare)


def gap_solve(op, y: np.ndarray, cfg: SolverConfig, ref: np.ndarray | None = None,
              process_group=None, positions_override=None, trace=None):
    """solvers.py:284-308 — regularize, then project onto the measurement-
    consistent set; everything device-resident.

    Extra keywords (not in the reference): ``process_group`` shards exemplars
    across ranks; ``positions_override`` (list of (anchors, positions) per
    refresh) locks matching for positions-locked parity; ``trace`` (a list)
    receives (anchors, positions) of every refresh."""
    y = np.asarray(y)
    _check_measurement(op, y)
    t = D.torch()
    t_start = time.perf_counter()
    report = ReconReport()
    runner = GapRunner(op, cfg, process_group=process_group)
    dop = runner.dop
    y_d = dop.upload_y(y)
    iters = cfg.max_iters
    ref_d = D.f64(ref) if ref is not None else None

    def on_iter(it, x):
        if ref_d is not None:
            runner.record_metrics(x, ref_d, it)

    guard = _DivergenceGuard(runner.resid_sq, iters, float(np.linalg.norm(y.ravel())))
    x = runner.run(y_d, positions_override=positions_override, trace=trace,
                   on_iter=on_iter, events=True, guard=guard)
    t.cuda.synchronize()
    res = np.sqrt(D.host(runner.resid_sq)).tolist()
    sqh = D.host(runner.sq) if ref_d is not None else None
    ssims = _ssim_values(runner, ref) if ref_d is not None else None
    ev = runner.events
    for it in range(iters):
        e0, e1, e2, e3 = ev[it]
        row = {"iteration": it, "residual": float(res[it]),
               "match_ms": round(e0.elapsed_time(e1), 3),
               "lowrank_ms": round(e1.elapsed_time(e2), 3),
               "projection_ms": round(e2.elapsed_time(e3), 3)}
        if sqh is not None:
            mse = sqh[it] / float(np.prod(dop.shape))
            row["psnr_db"] = PSNR_CAP_DB if mse == 0.0 else \
                min(10.0 * np.log10(cfg.peak ** 2 / mse), PSNR_CAP_DB)
            row["ssim"] = float(ssims[it])
        report.add(**row)
    report.total_ms = (time.perf_counter() - t_start) * 1e3
    return _final_host(runner, x), report


class AdmmRunner(GapRunner):
    """Scaled-form ADMM (solvers.py:311-341) on the same device operator and
    GLR engine; the x-update is the fused projection kernel with the divisor
    rho + gram, the bookkeeping is glr_lincomb in numpy's evaluation order."""

    def __init__(self, op, cfg: SolverConfig, process_group=None):
        super().__init__(op, cfg, process_group)
        t = D.torch()
        self.z = D.empty(self.dop.shape, t.float64)
        self.u = D.empty(self.dop.shape, t.float64)
        self.v = D.empty(self.dop.shape, t.float64)

    def _lincomb(self, out, x, a, y=None, b=0.0, z=None, c=0.0, clip=False):
        lo, hi = -0.5 * self.cfg.peak, 1.5 * self.cfg.peak
        N.call("glr_lincomb", x.data_ptr(), float(a), y.data_ptr() if y is not None else None,
               float(b), z.data_ptr() if z is not None else None, float(c), int(x.numel()),
               1 if clip else 0, lo, hi, out.data_ptr(), D.stream())

    def run(self, y_d, positions_override=None, trace=None, on_iter=None, events=False,
            guard: _DivergenceGuard | None = None):
        t = D.torch()
        cfg, dop, eng = self.cfg, self.dop, self.eng
        iters = cfg.max_iters
        h, w, c = dop.shape
        z, u, x, m, v = self.z, self.u, self.xa, self.xb, self.v
        dop.init_x(y_d, z, cfg.init)
        u.zero_()
        eng.has_positions = False
        eng.vcache_valid = False
        eng.warm = 0
        lo, hi = -0.5 * cfg.peak, 1.5 * cfg.peak
        clip = dop.clip
        self.events = ([[t.cuda.Event(enable_timing=True) for _ in range(4)]
                        for _ in range(iters)] if events else None)
        last, refresh_no = -1, 0
        for it in range(iters):
            ev = self.events[it] if events else None
            if ev:
                ev[0].record()
            self._lincomb(m, z, 1.0, u, -1.0)                                  # m = z - u
            dop.gap_update(None, None, eng.frac, m, y_d, lo, hi, x, self.resid_sq[it:it + 1],
                           eng.gap_ws, rho=cfg.admm_rho)                         # x-update + clip
            if ev:
                ev[1].record()
            self._lincomb(v, x, 1.0, u, 1.0)                                   # v = x + u
            if self.tv is None and ((not eng.has_positions)
                                    or it - last >= cfg.match_refresh_interval):
                if positions_override is not None:
                    anc, pos = positions_override[refresh_no]
                    eng.set_positions(np.asarray(anc), np.asarray(pos))
                else:
                    eng.refresh(v)
                if trace is not None:
                    a, pz, _ = eng.positions_host()
                    trace.append((a.tolist(), pz.tolist()))
                last = it
                refresh_no += 1
            if ev:
                ev[2].record()
            if self.tv is not None:
                self._lincomb(z, self.tv(v), 1.0, clip=clip)                   # z = clip(tv(v))
            elif eng.regularize(v, cfg.sigma_at(it)):
                N.call("glr_normalize", eng.acc.data_ptr(), eng.cnt.data_ptr(), v.data_ptr(),
                       h, w, c, eng.frac, z.data_ptr(), D.stream())
                eng.consumed()
                self._lincomb(z, z, 1.0, clip=clip)                            # z = clip(z)
            else:
                self._lincomb(z, v, 1.0, clip=clip)
            self._lincomb(u, u, 1.0, x, 1.0, z, -1.0)                          # u = (u + x) - z
            if ev:
                ev[3].record()
            if on_iter is not None:
                on_iter(it, x)
            if guard is not None:
                guard.push(it)
        if guard is not None:
            guard.poll(block=True)
        return x


def admm_solve(op, y: np.ndarray, cfg: SolverConfig, ref: np.ndarray | None = None,
               process_group=None, trace=None):
    """solvers.py:311-341 — scaled-form ADMM; the x-update uses the Woodbury
    identity through the measurement-domain diagonal (divisor rho + gram)."""
    y = np.asarray(y)
    _check_measurement(op, y)
    t = D.torch()
    t_start = time.perf_counter()
    report = ReconReport()
    runner = AdmmRunner(op, cfg, process_group=process_group)
    y_d = runner.dop.upload_y(y)
    ref_d = D.f64(ref) if ref is not None else None

    def on_iter(it, x):
        if ref_d is not None:
            runner.record_metrics(x, ref_d, it)

    guard = _DivergenceGuard(runner.resid_sq, cfg.max_iters, float(np.linalg.norm(y.ravel())))
    x = runner.run(y_d, trace=trace, on_iter=on_iter, events=True, guard=guard)
    t.cuda.synchronize()
    res = np.sqrt(D.host(runner.resid_sq)).tolist()
    sqh = D.host(runner.sq) if ref_d is not None else None
    ssims = _ssim_values(runner, ref) if ref_d is not None else None
    n_el = float(np.prod(runner.dop.shape))
    for it, (e0, e1, e2, e3) in enumerate(runner.events):
        row = {"iteration": it, "residual": float(res[it]),
               "match_ms": round(e1.elapsed_time(e2), 3),
               "lowrank_ms": round(e2.elapsed_time(e3), 3),
               "projection_ms": round(e0.elapsed_time(e1), 3)}
        if sqh is not None:
            mse = sqh[it] / n_el
            row["psnr_db"] = PSNR_CAP_DB if mse == 0.0 else \
                min(10.0 * np.log10(cfg.peak ** 2 / mse), PSNR_CAP_DB)
            row["ssim"] = float(ssims[it])
        report.add(**row)
    report.total_ms = (time.perf_counter() - t_start) * 1e3
    return _final_host(runner, x), report


def solve(op, y: np.ndarray, cfg: SolverConfig, ref: np.ndarray | None = None):
    """solvers.py:344-347."""
    fn = gap_solve if cfg.algorithm == "gap" else admm_solve
    return fn(op, y, cfg, ref)


class _TvState:
    """Stand-in for the match engine under the TV regularizer: no positions,
    just the projection workspace."""

    def __init__(self, h, w):
        self.gap_ws = D.empty((N.query("glr_gap_workspace", h, w),), D.torch().uint8)
        self.has_positions = False
        self.frac = 0


class TvProx:
    """Device TV prox (glr_tv_denoise) with its output and dual workspaces."""

    def __init__(self, shape, weight: float, iters: int):
        t = D.torch()
        h, w, c = shape
        self.shape, self.weight, self.iters = (h, w, c), float(weight), int(iters)
        self.out = D.empty((h, w, c), t.float64)
        self.ws = D.empty((N.query("glr_tv_workspace", h, w, c),), t.uint8)

    def __call__(self, x_d):
        h, w, c = self.shape
        N.call("glr_tv_denoise", x_d.data_ptr(), h, w, c, self.weight, self.iters,
               self.out.data_ptr(), self.ws.data_ptr(), self.ws.numel(), D.stream())
        return self.out


def tv_denoise(x: np.ndarray, weight: float, iters: int = 20) -> np.ndarray:
    """solvers.py:121-139 — proximal operator of anisotropic TV per channel,
    dual projected gradient (tau = 1/8); bit-identical to the reference."""
    x = np.asarray(x, dtype=np.float64)
    if weight <= 0:
        return x.copy()
    if x.ndim != 3:
        raise ValueError(f"image must be (H, W, C), got shape {x.shape}")
    return D.host(TvProx(x.shape, weight, iters)(D.f64(x)))
