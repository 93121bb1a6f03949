"""Weighted nuclear norm minimisation on patch groups and the image-space
low-rank pass (reference: glr/lowrank.py:1-87), on the batched fp64
Gram + Jacobi kernel of csrc/wnnm.cu."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from .patches import PatchGroup, _positions_array

KMAX = 64


@dataclass
class WnnmParams:
    """lowrank.py:18-31."""

    c_weight: float = 2.0 * np.sqrt(2.0)
    eps: float = 1e-16
    noise_sigma: float = 0.0
    uniform_weight: float | None = None  # test hook: plain SVT at this level

    def __post_init__(self):
        if self.c_weight <= 0:
            raise ValueError("c_weight must be positive")
        if self.eps <= 0:
            raise ValueError("eps must be positive")
        if self.noise_sigma < 0:
            raise ValueError("noise_sigma must be nonnegative")


def frac_bits_for(peak: float) -> int:
    """Fixed-point scale of the aggregation numerator: 2^40 for peak <= 1,
    reduced by the peak's binary magnitude to keep >20 bits of headroom."""
    return 40 - max(0, int(math.ceil(math.log2(max(float(peak), 1.0)))))


def wnnm_batch(mats: np.ndarray, params: WnnmParams) -> np.ndarray:
    """Batched WNNM of (G, m, K) group matrices; returns (G, m, K)."""
    mats = np.asarray(mats, dtype=np.float64)
    g, m, k = mats.shape
    if not np.isfinite(mats).all():
        raise ValueError("non-finite entries in group matrix")
    src = D.f64(np.ascontiguousarray(mats.transpose(0, 2, 1)))  # (G, K, m) column-major
    out = D.empty((g, k, m), D.torch().float64)
    uw = -1.0 if params.uniform_weight is None else float(params.uniform_weight)
    ws = D.workspace().get("wnnm", N.query("glr_wnnm_workspace", g, k))
    N.call("glr_wnnm", src.data_ptr(), g, m, k, float(params.noise_sigma),
           float(params.c_weight), float(params.eps), uw, out.data_ptr(), None, ws.data_ptr(),
           ws.numel(), D.stream())
    return D.host(out).transpose(0, 2, 1).copy()


def wnnm_prox(m: np.ndarray, params: WnnmParams) -> np.ndarray:
    """lowrank.py:46-65 — weighted singular value thresholding of one group."""
    m = np.asarray(m, dtype=np.float64)
    if not np.isfinite(m).all():
        raise ValueError("non-finite entries in group matrix")
    if m.ndim != 2:
        raise ValueError("group matrix must be 2-D")
    return wnnm_batch(m[None], params)[0]


def glr_regularize(x: np.ndarray, groups: list[PatchGroup], params: WnnmParams) -> np.ndarray:
    """lowrank.py:68-87 — shrink every group, scatter back, count-normalise;
    uncovered pixels pass through. Aggregation is int64 fixed point
    (deterministic; within 2^-40 per term of the reference's fp64 sum)."""
    x = np.asarray(x, dtype=np.float64)
    if not groups:
        return x.copy()
    h, w, c = x.shape
    t = D.torch()
    frac = frac_bits_for(max(1.0, float(np.abs(x).max()) if x.size else 1.0))
    acc = D.zeros((h, w, c), t.int64)
    cnt = D.zeros((h, w), t.int32)
    batches: dict[tuple[int, int], list] = {}
    for g in groups:
        pos = _positions_array(g.positions, h, w, g.patch_size)
        if len(pos):
            batches.setdefault((g.patch_size, len(pos)), []).append((pos, g.matrix))
    for (p, k), items in batches.items():
        pos = np.stack([it[0] for it in items])                       # (G, K, 2)
        mats = np.stack([np.asarray(it[1], dtype=np.float64) for it in items])  # (G, m, K)
        den = wnnm_batch(mats, params)
        src = D.f64(np.ascontiguousarray(den.transpose(0, 2, 1)))     # (G, K, m)
        pos_d = D.i32(pos)
        N.call("glr_scatter_fixed", src.data_ptr(), pos_d.data_ptr(), len(items), k, p, h, w, c,
               frac, acc.data_ptr(), D.stream())
        N.call("glr_scatter_count", pos_d.data_ptr(), len(items), None, k, p, h, w,
               cnt.data_ptr(), D.stream())
    x_d = D.f64(x)
    z = D.empty((h, w, c), t.float64)
    N.call("glr_normalize", acc.data_ptr(), cnt.data_ptr(), x_d.data_ptr(), h, w, c, frac,
           z.data_ptr(), D.stream())
    return D.host(z)
