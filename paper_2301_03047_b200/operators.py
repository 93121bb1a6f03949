"""Sensing operators: CACTI temporal compression, masked-Fourier sampling
(real and complex (re, im) images) and MSFA mosaicking
(reference: glr/operators.py:1-218).

Each SensingOperator bundles forward, adjoint and the measurement-domain
diagonal of Phi Phi^T like the reference. The callables run on the GPU
(csrc/ops.cu, csrc/fft.cu); gap_solve never calls them — it rebuilds the
device operator from ``kind`` and ``meta`` (the reference's plug point).
Mask *generators* are host-side setup code.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _device as D
from . import _native as N


@dataclass
class SensingOperator:
    """operators.py:15-22."""

    kind: str
    forward: Callable[[np.ndarray], np.ndarray]
    adjoint: Callable[[np.ndarray], np.ndarray]
    gram_diag: np.ndarray
    x_shape: tuple[int, int, int]
    meta: dict = field(default_factory=dict)


# ---------------------------------------------------------------------------
# mask-sum family (CACTI, MSFA)

def bernoulli_masks(h: int, w: int, t: int, seed: int = 0, density: float = 0.5) -> np.ndarray:
    """operators.py:28-32 — seeded i.i.d. Bernoulli masks, shape (H, W, T)."""
    rng = np.random.default_rng(seed)
    return (rng.random((h, w, t)) < density).astype(np.float64)


def _masksum_forward(x: np.ndarray, masks: np.ndarray) -> np.ndarray:
    h, w, t = masks.shape
    x_d = D.f64(x)
    m_d = D.f64(masks)
    y = D.empty((h, w, 1), D.torch().float64)
    N.call("glr_masksum_forward", x_d.data_ptr(), m_d.data_ptr(), h, w, t, y.data_ptr(),
           D.stream())
    return D.host(y)


def _masksum_adjoint(y: np.ndarray, masks: np.ndarray) -> np.ndarray:
    y = np.asarray(y, dtype=np.float64)
    if y.ndim == 3:
        y = y[:, :, 0]
    h, w, t = masks.shape
    if y.shape != (h, w):
        raise ValueError(f"measurement shape {y.shape} != mask shape {(h, w)}")
    y_d = D.f64(y)
    m_d = D.f64(masks)
    x = D.empty((h, w, t), D.torch().float64)
    N.call("glr_masksum_adjoint", y_d.data_ptr(), m_d.data_ptr(), h, w, t, x.data_ptr(),
           D.stream())
    return D.host(x)


def cacti_forward(x: np.ndarray, masks: np.ndarray) -> np.ndarray:
    """operators.py:35-39 — y = sum_t M_t x_t (keepdims)."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != masks.shape:
        raise ValueError(f"frame shape {x.shape} != mask shape {masks.shape}")
    return _masksum_forward(x, masks)


def cacti_adjoint(y: np.ndarray, masks: np.ndarray) -> np.ndarray:
    """operators.py:42-46 — A^T y = M_t y."""
    return _masksum_adjoint(y, masks)


def _binary_u8(masks: np.ndarray) -> dict:
    """Compact copy of binary {0, 1} masks (checked once when the operator is
    built): the device path uploads these 8x smaller bytes and widens them
    on the GPU (and, for CACTI, forms gram = sum_t M_t there: exact integer
    counts), instead of the float64 masks and gram."""
    u8 = masks.astype(np.uint8)
    if not np.array_equal(u8, masks):
        return {}
    # tied to this masks object: replacing meta["masks"] disables the copy
    return {"masks_u8": u8, "masks_u8_of": id(masks)}


def cacti_operator(masks: np.ndarray) -> SensingOperator:
    """operators.py:49-59."""
    masks = np.asarray(masks, dtype=np.float64)
    h, w, t = masks.shape
    return SensingOperator(
        kind="cacti",
        forward=lambda x: cacti_forward(x, masks),
        adjoint=lambda y: cacti_adjoint(y, masks),
        gram_diag=(masks ** 2).sum(axis=2, keepdims=True),
        x_shape=(h, w, t),
        meta={"masks": masks, **_binary_u8(masks)},
    )


def _check_partition(masks: np.ndarray) -> None:
    """operators.py:150-157."""
    c = masks.shape[2]
    for i in range(c):
        for j in range(i + 1, c):
            if np.any(masks[:, :, i] * masks[:, :, j] != 0):
                raise ValueError(f"MSFA masks {i} and {j} are not orthogonal")
    if not np.array_equal(masks.sum(axis=2), np.ones(masks.shape[:2])):
        raise ValueError("MSFA masks do not partition the sensor (sum != 1)")


def msfa_forward(x: np.ndarray, masks: np.ndarray) -> np.ndarray:
    """operators.py:160-164."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != masks.shape:
        raise ValueError(f"scene shape {x.shape} != mask shape {masks.shape}")
    return _masksum_forward(x, masks)


def msfa_adjoint(y: np.ndarray, masks: np.ndarray) -> np.ndarray:
    """operators.py:167-171."""
    return _masksum_adjoint(y, masks)


def msfa_operator(masks: np.ndarray) -> SensingOperator:
    """operators.py:174-185."""
    masks = np.asarray(masks, dtype=np.float64)
    _check_partition(masks)
    h, w, c = masks.shape
    return SensingOperator(
        kind="msfa",
        forward=lambda x: msfa_forward(x, masks),
        adjoint=lambda y: msfa_adjoint(y, masks),
        gram_diag=np.ones((h, w, 1)),
        x_shape=(h, w, c),
        meta={"masks": masks, **_binary_u8(masks)},
    )


MSFA_KINDS = ("bayer-like-2x2", "periodic-3x3", "periodic-4x4", "custom-tile")


def msfa_pattern(kind: str, channels: int, h: int, w: int,
                 tile: np.ndarray | None = None) -> np.ndarray:
    """operators.py:191-218 — periodic MSFA partition masks (H, W, C)."""
    if kind not in MSFA_KINDS:
        raise ValueError(f"unknown MSFA kind {kind!r}")
    if kind == "custom-tile":
        if tile is None:
            raise ValueError("custom-tile requires a tile grid")
        tile = np.asarray(tile, dtype=np.int64)
        if tile.min() < 0 or tile.max() >= channels:
            raise ValueError("tile indices out of range")
    else:
        k = {"bayer-like-2x2": 2, "periodic-3x3": 3, "periodic-4x4": 4}[kind]
        if channels != k * k:
            raise ValueError(f"{kind} requires C = {k * k}, got {channels}")
        tile = np.arange(k * k, dtype=np.int64).reshape(k, k)
    th, tw = tile.shape
    grid = np.tile(tile, (-(-h // th), -(-w // tw)))[:h, :w]
    return (grid[:, :, None] == np.arange(channels)[None, None, :]).astype(np.float64)


# ---------------------------------------------------------------------------
# masked Fourier

def _fourier_image(x: np.ndarray, channels: int) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 2:
        x = x[:, :, None]
    if channels == 1 and x.shape[2] != 1:
        x = x[:, :, :1]
    return x


def fourier_forward(x: np.ndarray, mask: np.ndarray, channels: int = 1) -> np.ndarray:
    """operators.py:65-71 — y = M * fft2(x, norm="ortho"); channels=2 reads
    (re, im) image channels (SURVEY §8c complex variant)."""
    x = _fourier_image(x, channels)
    mask = np.asarray(mask, dtype=np.float64)
    if x.shape[:2] != mask.shape:
        raise ValueError(f"image shape {x.shape[:2]} != mask shape {mask.shape}")
    h, w = mask.shape
    x_d = D.f64(np.ascontiguousarray(x[:, :, :channels]))
    m_d = D.f64(mask)
    y = D.empty((h, w, 2), D.torch().float64)
    N.call("glr_fourier_forward", x_d.data_ptr(), m_d.data_ptr(), h, w, channels, y.data_ptr(),
           None, D.stream())
    yh = D.host(y)
    return yh[:, :, 0] + 1j * yh[:, :, 1]


def fourier_adjoint(y: np.ndarray, mask: np.ndarray, channels: int = 1) -> np.ndarray:
    """operators.py:74-76 — Re(ifft2(M * y, ortho)) (or (re, im) for C=2)."""
    y = np.asarray(y)
    mask = np.asarray(mask, dtype=np.float64)
    if y.ndim == 3:
        y = y[:, :, 0]
    h, w = mask.shape
    if y.shape != (h, w):
        raise ValueError(f"measurement shape {y.shape} != mask shape {(h, w)}")
    yc = np.stack([y.real, y.imag], axis=2).astype(np.float64) if np.iscomplexobj(y) else \
        np.stack([y, np.zeros_like(y)], axis=2).astype(np.float64)
    y_d = D.f64(yc)
    m_d = D.f64(mask)
    x = D.empty((h, w, channels), D.torch().float64)
    ws = D.workspace().get("fft", N.query("glr_fft_workspace", h, w))
    N.call("glr_fourier_adjoint", y_d.data_ptr(), m_d.data_ptr(), h, w, channels, x.data_ptr(),
           ws.data_ptr(), D.stream())
    return D.host(x)


def fourier_operator(mask: np.ndarray, channels: int = 1) -> SensingOperator:
    """operators.py:79-89; ``channels=2`` is the complex (re, im) variant used
    by the MRI configuration (x_shape (H, W, 2))."""
    if channels not in (1, 2):
        raise ValueError("channels must be 1 (real image) or 2 (re, im)")
    mask = np.asarray(mask, dtype=np.float64)
    h, w = mask.shape
    return SensingOperator(
        kind="fourier",
        forward=lambda x: fourier_forward(x, mask, channels),
        adjoint=lambda y: fourier_adjoint(y, mask, channels),
        gram_diag=mask.copy(),
        x_shape=(h, w, channels),
        meta={"mask": mask, "sampling_ratio": float(mask.mean())},
    )


def _line_points(y1: int, x1: int):
    """Integer raster of the segment (0,0) -> (y1, x1), inclusive, stepping
    the error term like Bresenham's algorithm (operators.py:127-144)."""
    dy, dx = abs(y1), abs(x1)
    sy = 1 if y1 >= 0 else -1
    sx = 1 if x1 >= 0 else -1
    err = dx - dy
    y = x = 0
    pts = [(0, 0)]
    while (y, x) != (y1, x1):
        e2 = 2 * err
        if e2 > -dy:
            err -= dy
            x += sx
        if e2 < dx:
            err += dx
            y += sy
        pts.append((y, x))
    return pts


def radial_mask(h: int, w: int, num_lines: int) -> np.ndarray:
    """operators.py:92-124 — radial spokes through DC, symmetrised, in
    unshifted FFT order (host-side mask generator)."""
    if num_lines < 1:
        raise ValueError("num_lines must be >= 1")
    cen = np.zeros((h, w), dtype=bool)
    cy, cx = h // 2, w // 2
    reach = int(np.ceil(np.hypot(h, w)))
    for k in range(num_lines):
        ang = k * np.pi / num_lines
        for py, px in _line_points(int(round(reach * np.sin(ang))),
                                   int(round(reach * np.cos(ang)))):
            for r, c in ((cy + py, cx + px), (cy - py, cx - px)):
                if 0 <= r < h and 0 <= c < w:
                    cen[r, c] = True
    ys, xs = np.nonzero(cen)
    r2, c2 = 2 * cy - ys, 2 * cx - xs
    ok = (r2 >= 0) & (r2 < h) & (c2 >= 0) & (c2 < w)
    flip = np.zeros_like(cen)
    flip[r2[ok], c2[ok]] = True
    cen |= flip
    cen[cy, cx] = True
    return np.fft.ifftshift(cen).astype(np.float64)
