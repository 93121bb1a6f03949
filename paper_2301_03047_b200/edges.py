"""Sobel gradients, sign-split binary edge maps and corner-seeded exemplars
(reference: glr/edges.py:1-162), computed by the fp64 kernels of
csrc/edges.cu, which reproduce the reference's floating-point evaluation
order bit for bit."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N

SOBEL_H = np.array([[-1.0, 0.0, 1.0],
                    [-2.0, 0.0, 2.0],
                    [-1.0, 0.0, 1.0]])
SOBEL_V = SOBEL_H.T.copy()


@dataclass
class EdgeMaps:
    """Four binary (H, W, C) maps: gradient sign x direction (edges.py:24-38)."""

    h_pos: np.ndarray
    h_neg: np.ndarray
    v_pos: np.ndarray
    v_neg: np.ndarray

    def as_tuple(self):
        return (self.h_pos, self.h_neg, self.v_pos, self.v_neg)

    @property
    def shape(self):
        return self.h_pos.shape


@dataclass
class ExemplarSet:
    """Patch anchors (top-left) with their provenance tag (edges.py:41-50)."""

    anchors: list[tuple[int, int]]
    tags: list[str]
    patch_size: int

    def __len__(self) -> int:
        return len(self.anchors)


def _image(img) -> np.ndarray:
    img = np.asarray(img, dtype=np.float64)
    if img.ndim == 2:
        img = img[:, :, None]
    return img


def sobel_gradients(img: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """edges.py:53-64 — per-channel Sobel with edge-replicate borders."""
    img = _image(img)
    h, w, c = img.shape
    if h < 3 or w < 3:
        raise ValueError(f"image {h}x{w} too small for 3x3 Sobel")
    x_d = D.f64(img)
    gh = D.empty(img.shape, D.torch().float64)
    gv = D.empty(img.shape, D.torch().float64)
    N.call("glr_sobel", x_d.data_ptr(), h, w, c, gh.data_ptr(), gv.data_ptr(), D.stream())
    return D.host(gh), D.host(gv)


def binarize_gradients(gh: np.ndarray, gv: np.ndarray, th: float = 0.2,
                       relative: bool = True) -> EdgeMaps:
    """edges.py:67-85 — threshold rectified gradients into four binary maps
    (float64 0/1, like the reference)."""
    if th < 0:
        raise ValueError(f"threshold must be nonnegative, got {th}")
    gh = np.asarray(gh, dtype=np.float64)
    gv = np.asarray(gv, dtype=np.float64)
    if gh.shape != gv.shape:
        raise ValueError(f"gradient shapes differ: {gh.shape} vs {gv.shape}")
    shape = gh.shape
    # elementwise + one global max: any shape maps onto a 1 x 1 x size image
    h, w, c = 1, 1, int(gh.size)
    if c == 0:
        z = np.zeros(shape)
        return EdgeMaps(h_pos=z, h_neg=z.copy(), v_pos=z.copy(), v_neg=z.copy())
    gh_d = D.f64(gh)
    gv_d = D.f64(gv)
    maps = D.empty((4,) + tuple(shape), D.torch().uint8)
    ws = D.workspace().get("edge_max", 64)
    N.call("glr_edge_stack", gh_d.data_ptr(), gv_d.data_ptr(), h, w, c, float(th),
           1 if relative else 0, 1, maps.data_ptr(), None, ws.data_ptr(), D.stream())
    m = D.host(maps).astype(np.float64)
    return EdgeMaps(h_pos=m[0], h_neg=m[1], v_pos=m[2], v_neg=m[3])


def detect_corners(img: np.ndarray, max_n: int = 512, nms_radius: int = 4,
                   quality: float = 0.01) -> list[tuple[int, int]]:
    """edges.py:100-128 — Shi-Tomasi corners of the channel-averaged gradient
    magnitude, strongest first, greedy Chebyshev NMS, ties row-major."""
    if max_n < 1:
        raise ValueError("max_n must be >= 1")
    img = _image(img)
    h, w, c = img.shape
    if h < 3 or w < 3:
        raise ValueError(f"image {h}x{w} too small for 3x3 Sobel")
    t = D.torch()
    x_d = D.f64(img)
    resp = D.empty((h, w), t.float64)
    ws = D.workspace()
    cw = ws.get("corner", N.query("glr_corner_workspace", h, w, c))
    N.call("glr_corner_response", x_d.data_ptr(), h, w, c, resp.data_ptr(), cw.data_ptr(),
           D.stream())
    nb = N.query("glr_nms_workspace", h, w)
    nw = ws.get("nms", nb)
    out = D.empty((max_n, 2), t.int32)
    n_d = D.zeros((1,), t.int32)
    N.call("glr_corners", resp.data_ptr(), h, w, int(max_n), int(nms_radius), float(quality),
           out.data_ptr(), n_d.data_ptr(), nw.data_ptr(), nw.numel(), D.stream())
    n = int(n_d.item())
    return [tuple(rc) for rc in D.host(out[:n]).tolist()]


def select_exemplars(corners, shape: tuple[int, int], patch_size: int,
                     uniform_interval: int | None = None) -> ExemplarSet:
    """edges.py:131-162 — clamped, deduplicated corner anchors plus an
    optional row-major uniform grid (tagged "uniform")."""
    h, w = shape
    p = patch_size
    if p > min(h, w):
        raise ValueError(f"patch size {p} exceeds image {h}x{w}")
    if uniform_interval is not None and uniform_interval < 1:
        raise ValueError("uniform_interval must be >= 1")
    corners = np.asarray([tuple(map(int, q)) for q in corners], dtype=np.int32).reshape(-1, 2)
    nc = len(corners)
    grid = 0
    if uniform_interval is not None:
        grid = ((h - p) // uniform_interval + 1) * ((w - p) // uniform_interval + 1)
    max_anchors = nc + grid
    if max_anchors == 0:
        return ExemplarSet(anchors=[], tags=[], patch_size=p)
    t = D.torch()
    c_d = D.i32(corners) if nc else D.zeros((1, 2), t.int32)
    nc_d = D.i32(np.array([nc]))
    anchors = D.empty((max_anchors, 2), t.int32)
    tags = D.empty((max_anchors,), t.uint8)
    n_d = D.zeros((1,), t.int32)
    ws = D.workspace().get("anchors", N.query("glr_anchor_workspace", h, w))
    N.call("glr_select_anchors", c_d.data_ptr(), nc_d.data_ptr(), max(nc, 1), h, w, p,
           int(uniform_interval or 0), max_anchors, anchors.data_ptr(), tags.data_ptr(),
           n_d.data_ptr(), ws.data_ptr(), D.stream())
    n = int(n_d.item())
    a = [tuple(q) for q in D.host(anchors[:n]).tolist()]
    tg = ["uniform" if v else "corner" for v in D.host(tags[:n]).tolist()]
    return ExemplarSet(anchors=a, tags=tg, patch_size=p)
