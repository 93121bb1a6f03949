"""Global matching: edge-overlap heat map on tcgen05 tensor cores and exact
tie-ordered top-K (reference: glr/matching.py:1-253).

MatchConfig keeps the reference's fields and validation; `backend` is
accepted for config compatibility but every backend runs the same B200
kernel (the reference's backends agree exactly, tests/test_acceptance.py
criterion 1).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from .edges import EdgeMaps, ExemplarSet
from .patches import PatchGroup, _check_anchor

MODES = ("bm-uniform", "bm-corner", "bm-corner-uniform", "gm")
BACKENDS = ("direct", "im2col", "fft")
TOPK_MAX_SCORE = 12287


@dataclass
class MatchConfig:
    """matching.py:25-63."""

    patch_size: int = 8
    group_size: int = 64
    bm_window: int = 20
    bm_stride: int = 1
    exemplar_stride: int = 6
    mode: str = "gm"
    min_separation: int | None = None
    backend: str = "im2col"
    edge_threshold: float = 0.2
    max_corners: int = 512
    corner_quality: float = 0.01
    nms_radius: int | None = None
    rerank_pixel: bool = False

    def __post_init__(self):
        if self.group_size < 1:
            raise ValueError("group_size must be >= 1")
        if self.patch_size < 2:
            raise ValueError("patch_size must be >= 2")
        if self.mode not in MODES:
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.backend not in BACKENDS:
            raise ValueError(f"unknown backend {self.backend!r}")
        if self.mode.startswith("bm") and self.bm_window < self.patch_size:
            raise ValueError("bm_window must be >= patch_size for bm modes")

    @property
    def sep(self) -> int:
        if self.min_separation is not None:
            return self.min_separation
        return -(-self.patch_size // 4)

    @property
    def nms(self) -> int:
        if self.nms_radius is not None:
            return self.nms_radius
        return -(-self.patch_size // 2)


@dataclass
class SimilarityHeatMap:
    """(H-P+1, W-P+1, N) overlap-count scores, one slice per exemplar."""

    values: np.ndarray
    anchors: list[tuple[int, int]]
    patch_size: int


def _maps_array(edge: EdgeMaps) -> np.ndarray:
    maps = np.stack([np.asarray(m) for m in edge.as_tuple()])
    if maps.ndim != 4:
        raise ValueError(f"edge maps must be (H, W, C), got {maps.shape[1:]}")
    if not np.all((maps == 0) | (maps == 1)):
        raise ValueError("edge maps must be binary (0/1)")
    return maps.astype(np.uint8)


def heat_device(maps_d, h, w, c, p, anchors_d, n):
    """Device heat map from binary maps (4,H,W,C) u8: returns u16 (n, stride)."""
    t = D.torch()
    e = N.query("glr_heat_expand_factor", c, p)
    stack = D.empty((h * w * 2 * c * e,), t.uint8)  # packed fp4 (two elements per byte)
    N.call("glr_stack_from_maps", maps_d.data_ptr(), h, w, c, e, stack.data_ptr(), D.stream())
    stride = N.query("glr_heat_stride", h, w, p)
    heat = D.empty((n, stride), t.int16)
    wsb = N.query("glr_heat_workspace", c, p, n)
    ws = D.workspace().get("heat", wsb)
    N.call("glr_heat_map", stack.data_ptr(), h, w, c, p, e, anchors_d.data_ptr(), n, None,
           heat.data_ptr(), ws.data_ptr(), ws.numel(), D.stream())
    return heat


def similarity_heatmap(edge: EdgeMaps, exemplars: ExemplarSet,
                       backend: str = "im2col") -> SimilarityHeatMap:
    """matching.py:140-167 — sum of the four per-map correlations of each
    exemplar's edge patches against the full edge maps (exact integers)."""
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}")
    maps = _maps_array(edge)
    _, h, w, c = maps.shape
    p = exemplars.patch_size
    if p > h or p > w:
        raise ValueError(f"kernel {p}x{p} larger than input {h}x{w}")
    anchors = [tuple(map(int, a)) for a in exemplars.anchors]
    for i, a in enumerate(anchors):
        _check_anchor(h, w, p, a, i)
    oh, ow = h - p + 1, w - p + 1
    n = len(anchors)
    if n == 0:
        return SimilarityHeatMap(values=np.zeros((oh, ow, 0)), anchors=[], patch_size=p)
    heat = heat_device(D.to_dev(maps), h, w, c, p, D.i32(np.array(anchors)), n)
    vals = D.host(heat)[:, :oh * ow].view(np.uint16).astype(np.float64)
    vals = vals.reshape(n, oh, ow).transpose(1, 2, 0).copy()
    return SimilarityHeatMap(values=vals, anchors=anchors, patch_size=p)


def topk_device(heat_d, n, oh, ow, max_score, anchors_d, k, sep):
    t = D.torch()
    pos = D.empty((n, k, 2), t.int32)
    pad = D.empty((n,), t.int32)
    N.call("glr_topk", heat_d.data_ptr(), n, None, oh, ow, int(max_score), anchors_d.data_ptr(),
           int(k), int(sep), pos.data_ptr(), pad.data_ptr(), None, 0, D.stream())
    return pos, pad


def top_k_positions(slice2d: np.ndarray, anchor: tuple[int, int], k: int,
                    min_separation: int) -> tuple[list[tuple[int, int]], int]:
    """matching.py:170-231 — the exemplar's anchor in slot 0, then the highest
    scores (ties row-major) at Chebyshev separation > min_separation, relaxed
    to 0, then anchor padding.

    The B200 kernel ranks integer overlap counts (what the heat map holds);
    slices must be integer-valued in [0, 12287]."""
    s = np.asarray(slice2d, dtype=np.float64)
    if s.ndim != 2 or s.size == 0:
        raise ValueError("slice must be a non-empty 2-D array")
    if k < 1:
        raise ValueError("group_size must be >= 1")
    if min_separation < 0:
        raise ValueError("min_separation must be >= 0")
    if not (np.all(np.isfinite(s)) and np.all(s == np.rint(s)) and s.min() >= 0
            and s.max() <= TOPK_MAX_SCORE):
        raise ValueError("top_k_positions ranks integer overlap counts in "
                         f"[0, {TOPK_MAX_SCORE}] on the B200 path")
    oh, ow = s.shape
    stride = -(-(oh * ow) // 8) * 8
    row = np.zeros((1, stride), dtype=np.uint16)
    row[0, :oh * ow] = s.ravel().astype(np.uint16)
    heat_d = D.to_dev(row.view(np.int16))
    anchor = (int(anchor[0]), int(anchor[1]))
    pos, pad = topk_device(heat_d, 1, oh, ow, int(s.max()), D.i32(np.array([anchor])), k,
                           min_separation)
    positions = [tuple(q) for q in D.host(pos[0]).tolist()]
    return positions, int(pad.item())


def global_match(x: np.ndarray, exemplars: ExemplarSet, cfg: MatchConfig,
                 edge: EdgeMaps) -> list[PatchGroup]:
    """matching.py:234-253 — per exemplar, the top-K structurally similar
    patches by edge overlap; patches gathered from ``x``."""
    x = np.asarray(x, dtype=np.float64)
    maps = _maps_array(edge)
    _, h, w, c = maps.shape
    p = exemplars.patch_size
    anchors = [tuple(map(int, a)) for a in exemplars.anchors]
    for i, a in enumerate(anchors):
        _check_anchor(h, w, p, a, i)
    n = len(anchors)
    if n == 0:
        return []
    k = cfg.group_size
    anchors_d = D.i32(np.array(anchors))
    heat = heat_device(D.to_dev(maps), h, w, c, p, anchors_d, n)
    oh, ow = h - p + 1, w - p + 1
    pos, pad = topk_device(heat, n, oh, ow, 4 * c * p * p, anchors_d, k, cfg.sep)
    x_d = D.f64(x)
    if cfg.rerank_pixel:
        xh, xw, xc = x.shape
        N.call("glr_rerank_pixel", x_d.data_ptr(), xh, xw, xc, p, pos.data_ptr(), n, k,
               D.stream())
    return _gather_groups(x_d, x.shape, p, pos, pad)


def _gather_groups(x_d, shape, p, pos, pad) -> list[PatchGroup]:
    """Device gather of every group's (m, K) matrix (patches.py:43-54)."""
    xh, xw, xc = shape
    n, k = pos.shape[0], pos.shape[1]
    m = p * p * xc
    groups_d = D.empty((n, k, m), D.torch().float64)
    N.call("glr_gather", x_d.data_ptr(), xh, xw, xc, p, pos.data_ptr(), n, k,
           groups_d.data_ptr(), D.stream())
    pos_h = D.host(pos)
    pad_h = D.host(pad)
    mats = D.host(groups_d)
    out = []
    for i in range(n):
        g = PatchGroup(patch_size=p, positions=[tuple(q) for q in pos_h[i].tolist()],
                       matrix=np.ascontiguousarray(mats[i].T))
        g.padded = int(pad_h[i])
        out.append(g)
    return out


def xcorr2_valid_batch(x: np.ndarray, kernels, backend: str = "im2col") -> np.ndarray:
    """matching.py:116-137 — valid 2-D cross-correlation of x (H, W, C) with N
    (P, P, C) kernels, channels summed: (H-P+1, W-P+1, N). One device kernel
    serves every backend name; it accumulates in the (dr, dc, ch) order of
    the reference tests' loop oracle (bit-identical to it)."""
    x = np.asarray(x, dtype=np.float64)
    kernels = np.asarray(kernels, dtype=np.float64)
    if kernels.ndim == 3:
        kernels = kernels[None]
    n, p, q, c = kernels.shape
    if p != q:
        raise ValueError("kernels must be square")
    h, w, xc = x.shape
    if c != xc:
        raise ValueError(f"channel mismatch: input {xc}, kernels {c}")
    if p > h or p > w:
        raise ValueError(f"kernel {p}x{p} larger than input {h}x{w}")
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}")
    # keep the device copies referenced until the launch (a temporary's block
    # could be handed to the next upload before the kernel reads it)
    x_d, k_d = D.f64(x), D.f64(kernels)
    out = D.empty((h - p + 1, w - p + 1, n), D.torch().float64)
    N.call("glr_xcorr_valid", x_d.data_ptr(), h, w, c, k_d.data_ptr(), n, p, out.data_ptr(),
           D.stream())
    return D.host(out)


def block_match_device(x_d, shape, p, anchors_d, n, cfg: MatchConfig, positions_d=None,
                       padded_d=None):
    """glr_block_match over n device anchors: (positions (n, K, 2), padded (n,))."""
    t = D.torch()
    h, w, c = shape
    k = cfg.group_size
    pos = positions_d if positions_d is not None else D.empty((n, k, 2), t.int32)
    pad = padded_d if padded_d is not None else D.empty((n,), t.int32)
    N.call("glr_block_match", x_d.data_ptr(), h, w, c, p, anchors_d.data_ptr(), n,
           int(cfg.bm_window), int(cfg.bm_stride), k, pos.data_ptr(), pad.data_ptr(), D.stream())
    return pos, pad


def block_match(x: np.ndarray, exemplars: ExemplarSet, cfg: MatchConfig) -> list[PatchGroup]:
    """matching.py:256-283 — classic local KNN block matching by squared pixel
    distance: the anchor, then the group_size-1 nearest window positions
    (ties row-major), anchor padding; one CTA per exemplar on device."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 3:
        raise ValueError(f"image must be (H, W, C), got shape {x.shape}")
    h, w, c = x.shape
    p = cfg.patch_size
    if p > h or p > w:
        raise ValueError(f"patch size {p} exceeds image {h}x{w}")
    anchors = [tuple(map(int, a)) for a in exemplars.anchors]
    for i, a in enumerate(anchors):
        _check_anchor(h, w, p, a, i)
    n = len(anchors)
    if n == 0:
        return []
    x_d = D.f64(x)
    pos, pad = block_match_device(x_d, x.shape, p, D.i32(np.array(anchors)), n, cfg)
    return _gather_groups(x_d, x.shape, p, pos, pad)
