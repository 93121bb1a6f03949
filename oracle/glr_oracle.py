"""CPU oracle for the GLR hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference package `glr` (arXiv 2301.03047,
/root/reference/pkg/src/glr) for exactly the functions on the north-star
path. Every function cites the reference
file:line it restates.

Pinning: this module is checked against golden vectors produced by running
the *reference itself* in the build container (tests/golden/make_golden.py ->
tests/golden/*.npz; tests/test_oracle_golden.py). The decision stages (edges,
corners, heat map, top-K) are pinned bit-for-bit; fp stages to 1e-12.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker or the timed CPU
baseline. The product package (paper_2301_03047_b200) never imports it.
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# A1/A2 — edges.py:53-85

# edges.py:18-21: horizontal-gradient Sobel taps; the vertical kernel is the
# transpose. Kept as explicit (row, col, weight) lists in row-major order so
# the accumulation order is visible.
_SOBEL_H_TAPS = [(0, 0, -1.0), (0, 2, 1.0), (1, 0, -2.0), (1, 2, 2.0), (2, 0, -1.0), (2, 2, 1.0)]
_SOBEL_V_TAPS = [(0, 0, -1.0), (0, 1, -2.0), (0, 2, -1.0), (2, 0, 1.0), (2, 1, 2.0), (2, 2, 1.0)]


def _correlate3(img2d: np.ndarray, taps) -> np.ndarray:
    """scipy.ndimage.correlate(img, K, mode="nearest") for a 3x3 K, restated:
    acc = 0; acc += w * x over non-zero taps in row-major order, with
    edge-replicate borders (scipy ni_filters.c correlation loop)."""
    h, w = img2d.shape
    pad = np.pad(img2d, 1, mode="edge")
    acc = np.zeros((h, w))
    for dr, dc, wt in taps:
        acc = acc + wt * pad[dr:dr + h, dc:dc + w]
    return acc


def sobel_gradients(img: np.ndarray):
    """edges.py:53-64 — per-channel Sobel, edge-replicate borders."""
    img = np.asarray(img, dtype=np.float64)
    h, w, c = img.shape
    if h < 3 or w < 3:
        raise ValueError(f"image {h}x{w} too small for 3x3 Sobel")
    gh = np.empty_like(img)
    gv = np.empty_like(img)
    for ch in range(c):
        gh[:, :, ch] = _correlate3(img[:, :, ch], _SOBEL_H_TAPS)
        gv[:, :, ch] = _correlate3(img[:, :, ch], _SOBEL_V_TAPS)
    return gh, gv


def binarize_gradients(gh, gv, th: float = 0.2, relative: bool = True):
    """edges.py:67-85 — four {0,1} maps (h_pos, h_neg, v_pos, v_neg) as uint8."""
    if th < 0:
        raise ValueError(f"threshold must be nonnegative, got {th}")
    th_h = th * np.abs(gh).max() if relative else th
    th_v = th * np.abs(gv).max() if relative else th
    return (
        (np.maximum(gh, 0.0) > th_h).astype(np.uint8),
        (np.maximum(-gh, 0.0) > th_h).astype(np.uint8),
        (np.maximum(gv, 0.0) > th_v).astype(np.uint8),
        (np.maximum(-gv, 0.0) > th_v).astype(np.uint8),
    )


# ---------------------------------------------------------------------------
# A3/A4 — edges.py:88-162, solvers.py:154-167

def _box3_axis(a: np.ndarray, axis: int) -> np.ndarray:
    """scipy uniform_filter1d(size=3, mode="nearest") restated as its running
    sum: t = (p0+p1)+p2, out0 = t/3, t += p[i+2]-p[i-1], out_i = t/3."""
    a = np.moveaxis(a, axis, 0)
    n = a.shape[0]
    idx = np.clip(np.arange(-1, n + 1), 0, n - 1)
    p = a[idx]
    out = np.empty_like(a)
    t = (p[0] + p[1]) + p[2]
    out[0] = t / 3.0
    for i in range(1, n):
        t = t + (p[i + 2] - p[i - 1])
        out[i] = t / 3.0
    return np.moveaxis(out, 0, axis)


def shi_tomasi_response(mag: np.ndarray) -> np.ndarray:
    """edges.py:88-97 — min-eigenvalue of the 3x3 box-filtered structure
    tensor of the Sobel gradients of ``mag``."""
    gx = _correlate3(mag, _SOBEL_H_TAPS)
    gy = _correlate3(mag, _SOBEL_V_TAPS)
    box = lambda z: _box3_axis(_box3_axis(z, 0), 1)  # noqa: E731 (axis 0 then 1)
    sxx, syy, sxy = box(gx * gx), box(gy * gy), box(gx * gy)
    return 0.5 * ((sxx + syy) - np.sqrt((sxx - syy) * (sxx - syy) + 4.0 * (sxy * sxy)))


def corner_response(img: np.ndarray) -> np.ndarray:
    """edges.py:110-112 — response of the channel-averaged gradient magnitude."""
    gh, gv = sobel_gradients(img)
    mag = np.sqrt(gh * gh + gv * gv).mean(axis=2)  # numpy pairwise mean over C
    return shi_tomasi_response(mag)


def detect_corners(img, max_n: int = 512, nms_radius: int = 4, quality: float = 0.01):
    """edges.py:100-128 — strongest-first corners after greedy Chebyshev NMS."""
    if max_n < 1:
        raise ValueError("max_n must be >= 1")
    resp = corner_response(img)
    rmax = resp.max()
    if rmax <= 0:
        return []
    h, w = resp.shape
    flat = resp.ravel()
    cand = np.nonzero(flat >= quality * rmax)[0]           # ascending flat index
    order = cand[np.argsort(-flat[cand], kind="stable")]   # (score desc, row, col)
    blocked = np.zeros((h, w), dtype=bool)
    picked: list[tuple[int, int]] = []
    r_ = nms_radius
    for idx in order:
        r, c = divmod(int(idx), w)
        if blocked[r, c]:
            continue
        picked.append((r, c))
        blocked[max(0, r - r_):r + r_ + 1, max(0, c - r_):c + r_ + 1] = True
        if len(picked) == max_n:
            break
    return picked


def select_exemplars(corners, shape, patch_size: int, uniform_interval: int | None = None):
    """edges.py:131-162 — (anchors, tags): clamped corner anchors deduplicated
    in order, then the row-major uniform grid."""
    h, w = shape
    p = patch_size
    if p > min(h, w):
        raise ValueError(f"patch size {p} exceeds image {h}x{w}")
    seen: set[tuple[int, int]] = set()
    anchors, tags = [], []
    for r, c in corners:
        a = (min(max(int(r) - p // 2, 0), h - p), min(max(int(c) - p // 2, 0), w - p))
        if a not in seen:
            seen.add(a)
            anchors.append(a)
            tags.append("corner")
    if uniform_interval is not None:
        if uniform_interval < 1:
            raise ValueError("uniform_interval must be >= 1")
        for r in range(0, h - p + 1, uniform_interval):
            for c in range(0, w - p + 1, uniform_interval):
                if (r, c) not in seen:
                    seen.add((r, c))
                    anchors.append((r, c))
                    tags.append("uniform")
    return anchors, tags


def build_exemplars(x, patch_size=8, max_corners=512, nms=None, quality=0.01,
                    exemplar_stride=6):
    """solvers.py:154-167, regularizer "glr": corners unioned with the grid at
    3 * exemplar_stride. ``nms`` defaults to ceil(P/2) (matching.py:59-63)."""
    nms = -(-patch_size // 2) if nms is None else nms
    corners = detect_corners(x, max_n=max_corners, nms_radius=nms, quality=quality)
    anchors, _ = select_exemplars(corners, x.shape[:2], patch_size,
                                  uniform_interval=3 * exemplar_stride)
    return anchors


# ---------------------------------------------------------------------------
# A5 — matching.py:140-167

def similarity_heatmap(maps, anchors, patch_size: int, chunk: int = 256) -> np.ndarray:
    """matching.py:140-167 — (oh, ow, N) edge-overlap counts, int64.

    Computed exactly in float32 (integers < 2^24, like the reference's f32
    GEMM of 0/1 values) without an im2col copy: for each kernel row dr one
    GEMM of the contiguous row block E[dr:dr+oh] against all P column taps of
    every exemplar, then the P column-shifted partials are summed.
    Exemplars go in chunks to bound memory (they are independent)."""
    e = np.concatenate([np.asarray(m, dtype=np.uint8) for m in maps], axis=2)  # (H,W,4C)
    h, w, c4 = e.shape
    p = patch_size
    oh, ow = h - p + 1, w - p + 1
    n = len(anchors)
    out = np.zeros((oh, ow, n), dtype=np.int64)
    ef = e.astype(np.float32)
    for s in range(0, n, chunk):
        block = anchors[s:s + chunk]
        b = len(block)
        ker = np.stack([ef[r:r + p, c:c + p, :] for r, c in block])      # (b,P,P,4C)
        acc = np.zeros((oh, ow, b), dtype=np.float32)
        for dr in range(p):
            rows = ef[dr:dr + oh].reshape(oh * w, c4)                    # contiguous
            kt = ker[:, dr].transpose(2, 1, 0).reshape(c4, p * b)        # (4C, P*b)
            part = (rows @ kt).reshape(oh, w, p, b)
            for dc in range(p):
                acc += part[:, dc:dc + ow, dc, :]
        out[:, :, s:s + b] = acc.astype(np.int64)
    return out


# ---------------------------------------------------------------------------
# A6 — matching.py:170-231

def top_k_positions(slice2d, anchor, k: int, min_separation: int):
    """matching.py:170-231 — slot 0 = anchor; then (score desc, flat idx asc)
    greedy with Chebyshev separation, relaxed to 0, then anchor padding."""
    oh, ow = slice2d.shape
    vals = np.asarray(slice2d).ravel()
    anchor = (int(anchor[0]), int(anchor[1]))
    m = k * (2 * min_separation + 1) ** 2 + 1
    if m < vals.size:
        # pool = top-m plus every tie with the cutoff (fills pass 1, see
        # matching.py:219-225); ordered by a stable descending sort
        part = np.argpartition(-vals, m - 1)[:m]
        cut = vals[part].min()
        cand = np.nonzero(vals >= cut)[0]
        order = cand[np.argsort(-vals[cand], kind="stable")]
        passes = (min_separation,)
    else:
        order = np.argsort(-vals, kind="stable")
        passes = (min_separation, 0)
    chosen = [anchor]
    for sep in passes:
        if len(chosen) >= k:
            break
        blocked = np.zeros((oh, ow), dtype=bool)
        for r, c in chosen:
            blocked[max(0, r - sep):r + sep + 1, max(0, c - sep):c + sep + 1] = True
        for idx in order:
            if len(chosen) >= k:
                break
            r, c = divmod(int(idx), ow)
            if blocked[r, c]:
                continue
            chosen.append((r, c))
            blocked[max(0, r - sep):r + sep + 1, max(0, c - sep):c + sep + 1] = True
    padded = k - len(chosen)
    chosen.extend([anchor] * padded)
    return chosen, padded


def match_positions(heat: np.ndarray, anchors, k: int, sep: int):
    """matching.py:240-245 — per-exemplar top-K over the heat map."""
    out, pads = [], []
    for n, a in enumerate(anchors):
        pos, pad = top_k_positions(heat[:, :, n], a, k, sep)
        out.append(pos)
        pads.append(pad)
    return out, pads


# ---------------------------------------------------------------------------
# f2 — matching.py:243-249 (rerank_pixel), matching.py:256-283 (block_match)

def block_match(x, anchors, patch_size: int, group_size: int, bm_window: int = 20,
                bm_stride: int = 1):
    """matching.py:256-283 — local KNN by squared pixel distance: the anchor,
    then the group_size-1 nearest window positions by (d, row, col), anchor
    padding. d is numpy's 3-axis sum of the squared broadcast difference.
    Returns (positions, pads)."""
    x = np.asarray(x, dtype=np.float64)
    h, w, c = x.shape
    p = patch_size
    # windows[r, c] = x[r:r+p, c:c+p, :] in (p, q, c) memory order
    win = np.lib.stride_tricks.sliding_window_view(x, (p, p), axis=(0, 1))
    out, pads = [], []
    for r0, c0 in anchors:
        r0, c0 = int(r0), int(c0)
        rows = np.arange(max(0, r0 - bm_window), min(h - p, r0 + bm_window) + 1, bm_stride)
        cols = np.arange(max(0, c0 - bm_window), min(w - p, c0 + bm_window) + 1, bm_stride)
        diff = win[np.ix_(rows, cols)] - win[r0, c0]
        dist = (diff * diff).sum(axis=(2, 3, 4)).ravel()
        rr = np.repeat(rows, len(cols))
        cc = np.tile(cols, len(rows))
        keep = ~((rr == r0) & (cc == c0))
        dist, rr, cc = dist[keep], rr[keep], cc[keep]
        pick = np.lexsort((cc, rr, dist))[:group_size - 1]
        pos = [(r0, c0)] + [(int(rr[i]), int(cc[i])) for i in pick]
        pad = group_size - len(pos)
        pos += [(r0, c0)] * pad
        out.append(pos)
        pads.append(max(pad, 0))
    return out, pads


def rerank_pixel(x, positions, patch_size: int):
    """matching.py:243-249 — slot 0 kept, slots 1.. ordered by (pixel L2
    distance to the anchor patch, (row, col)); the distance is numpy's sum
    over axis 0 of the (m, K) squared differences (sequential over rows)."""
    x = np.asarray(x, dtype=np.float64)
    out = []
    for pos in positions:
        pos = [tuple(map(int, q)) for q in pos]
        mat = gather_group(x, pos, patch_size)
        diff = mat - mat[:, :1]
        d = (diff * diff).sum(axis=0)
        order = [0] + sorted(range(1, len(pos)), key=lambda j: (d[j], pos[j]))
        out.append([pos[j] for j in order])
    return out


def tv_denoise(x, weight: float, iters: int = 20):
    """solvers.py:101-139 — anisotropic TV prox per channel by dual projected
    gradient (tau = 1/8): z = x - w div(p); p = clip(p - (tau/w) grad z)."""
    x = np.asarray(x, dtype=np.float64)
    if weight <= 0:
        return x.copy()

    def grad(z):
        gh, gv = np.zeros_like(z), np.zeros_like(z)
        gh[:, :-1] = z[:, 1:] - z[:, :-1]
        gv[:-1, :] = z[1:, :] - z[:-1, :]
        return gh, gv

    def div(ph, pv):
        d = np.empty_like(ph)
        d[:, 0] = ph[:, 0]
        d[:, 1:] = ph[:, 1:] - ph[:, :-1]
        d[0, :] += pv[0, :]
        d[1:, :] += pv[1:, :] - pv[:-1, :]
        return d

    out = np.empty_like(x)
    step = 0.125 / weight
    for ch in range(x.shape[2]):
        xc = x[:, :, ch]
        ph, pv = np.zeros_like(xc), np.zeros_like(xc)
        for _ in range(iters):
            gh, gv = grad(xc - weight * div(ph, pv))
            ph = np.clip(ph - step * gh, -1.0, 1.0)
            pv = np.clip(pv - step * gv, -1.0, 1.0)
        out[:, :, ch] = xc - weight * div(ph, pv)
    return out


# ---------------------------------------------------------------------------
# A7/A9/A10 — patches.py:43-70, lowrank.py:46-87

def gather_group(img, positions, patch_size: int) -> np.ndarray:
    """patches.py:43-54 — (P*P*C, K) matrix, column j = patch at positions[j]."""
    img = np.asarray(img, dtype=np.float64)
    h, w, c = img.shape
    p = patch_size
    for i, (r, col) in enumerate(positions):
        if not (0 <= r <= h - p and 0 <= col <= w - p):
            raise ValueError(f"anchor {i} at {(r, col)} out of bounds for patch size {p} "
                             f"in {h}x{w} image")
    return np.stack([img[r:r + p, col:col + p, :].ravel() for r, col in positions], axis=1)


def wnnm_prox(m, noise_sigma: float, c_weight: float = 2.0 * np.sqrt(2.0), eps: float = 1e-16,
              uniform_weight: float | None = None) -> np.ndarray:
    """lowrank.py:46-65 — one-pass weighted singular value thresholding."""
    m = np.asarray(m, dtype=np.float64)
    if not np.isfinite(m).all():
        raise ValueError("non-finite entries in group matrix")
    u, s, vt = np.linalg.svd(m, full_matrices=False)
    k = m.shape[1]
    if uniform_weight is not None:
        w = np.full_like(s, uniform_weight)
    else:
        sig_hat = np.sqrt(np.maximum(s ** 2 - k * noise_sigma ** 2, 0.0))
        w = c_weight * np.sqrt(k) * noise_sigma ** 2 / (sig_hat + eps)
    return (u * np.maximum(s - w, 0.0)) @ vt


def scatter_group(acc, cnt, matrix, positions, patch_size: int) -> None:
    """patches.py:57-70 — in-place scatter-add with counts."""
    h, w, c = acc.shape
    p = patch_size
    for j, (r, col) in enumerate(positions):
        acc[r:r + p, col:col + p, :] += matrix[:, j].reshape(p, p, c)
        cnt[r:r + p, col:col + p, :] += 1.0


def glr_regularize(x, groups_positions, patch_size: int, noise_sigma: float,
                   c_weight: float = 2.0 * np.sqrt(2.0), eps: float = 1e-16) -> np.ndarray:
    """lowrank.py:68-87 — WNNM per group, scatter, count-normalise."""
    x = np.asarray(x, dtype=np.float64)
    if not groups_positions:
        return x.copy()
    acc = np.zeros_like(x)
    cnt = np.zeros_like(x)
    for pos in groups_positions:
        den = wnnm_prox(gather_group(x, pos, patch_size), noise_sigma, c_weight, eps)
        scatter_group(acc, cnt, den, pos, patch_size)
    out = x.copy()
    cov = cnt > 0
    out[cov] = acc[cov] / cnt[cov]
    return out


# ---------------------------------------------------------------------------
# A11-A13 — operators.py

def bernoulli_masks(h, w, t, seed=0, density=0.5):
    """operators.py:28-32."""
    return (np.random.default_rng(seed).random((h, w, t)) < density).astype(np.float64)


def msfa_pattern_periodic(k: int, h: int, w: int) -> np.ndarray:
    """operators.py:191-218 for the periodic-kxk kinds: channel = row-major
    cell index of a k x k tile, repeated."""
    tile = np.arange(k * k).reshape(k, k)
    grid = np.tile(tile, (-(-h // k), -(-w // k)))[:h, :w]
    return np.stack([(grid == ch).astype(np.float64) for ch in range(k * k)], axis=2)


def masksum_forward(x, masks):
    """operators.py:35-39 / :160-164 — y = sum_t M_t x_t, keepdims."""
    return (masks * np.asarray(x, dtype=np.float64)).sum(axis=2, keepdims=True)


def masksum_adjoint(y, masks):
    """operators.py:42-46 / :167-171."""
    y = np.asarray(y, dtype=np.float64)
    if y.ndim == 3:
        y = y[:, :, 0]
    return masks * y[:, :, None]


def fourier_forward(x, mask):
    """operators.py:65-71 (real x, C=1) and the complex (re, im) variant of
    SURVEY §8c for C=2: y = M * fft2(x, ortho)."""
    x = np.asarray(x, dtype=np.float64)
    z = x[:, :, 0] if x.shape[2] == 1 else x[:, :, 0] + 1j * x[:, :, 1]
    return mask * np.fft.fft2(z, norm="ortho")


def fourier_adjoint(y, mask, channels: int):
    """operators.py:74-76 (real part, C=1) / stacked (re, im) for C=2."""
    out = np.fft.ifft2(mask * y, norm="ortho")
    if channels == 1:
        return out.real[:, :, None]
    return np.stack([out.real, out.imag], axis=2)


class Operator:
    """Minimal stand-in for SensingOperator (operators.py:15-22)."""

    def __init__(self, kind, masks=None, mask=None, channels=1):
        self.kind = kind
        if kind in ("cacti", "msfa"):
            self.masks = np.asarray(masks, dtype=np.float64)
            h, w, t = self.masks.shape
            self.x_shape = (h, w, t)
            self.gram = ((self.masks ** 2).sum(axis=2, keepdims=True) if kind == "cacti"
                         else np.ones((h, w, 1)))
        else:
            self.mask = np.asarray(mask, dtype=np.float64)
            h, w = self.mask.shape
            self.channels = channels
            self.x_shape = (h, w, channels)
            self.gram = self.mask.copy()

    def forward(self, x):
        if self.kind in ("cacti", "msfa"):
            return masksum_forward(x, self.masks)
        return fourier_forward(x, self.mask)

    def adjoint(self, y):
        if self.kind in ("cacti", "msfa"):
            return masksum_adjoint(y, self.masks)
        return fourier_adjoint(y, self.mask, self.channels)


# ---------------------------------------------------------------------------
# A8/A14/A15/A16 — solvers.py:66-69, 170-308; metrics.py:26-37

def sigma_at(k, max_iters, sigma0=0.10, sigma_min=0.003, peak=1.0):
    """solvers.py:66-69 — geometric noise schedule."""
    return sigma0 * (sigma_min / sigma0) ** (k / max_iters) * peak


def safe_div(num, den):
    """solvers.py:220-226."""
    out = np.zeros_like(num)
    nz = den != 0
    np.divide(num, den, out=out, where=nz)
    return out


def gaussian_weights(sigma=1.5, truncate=4.0):
    """The taps scipy.ndimage.gaussian_filter builds (radius int(truncate*sigma+0.5),
    exp(-x^2/(2 sigma^2)) normalised by its numpy sum)."""
    r = int(truncate * float(sigma) + 0.5)
    x = np.arange(-r, r + 1)
    phi = np.exp(-0.5 / (sigma * sigma) * x ** 2)
    return phi / phi.sum(), r


def gaussian_filter_reflect(img, sigma=1.5):
    """scipy.ndimage.gaussian_filter(img, sigma) on a 2-D float64 image, mode
    "reflect", restated in the symmetric-kernel evaluation order scipy's
    correlate1d uses: out = x[i] w[0] + sum_{j=-r..-1} (x[i+j] + x[i-j]) w[j],
    axis 0 then axis 1. Bit-identical (tests/test_oracle_golden.py)."""
    w, r = gaussian_weights(sigma)
    a = np.asarray(img, dtype=np.float64)
    for axis in (0, 1):
        n = a.shape[axis]
        idx = np.arange(n)

        def refl(i):
            i = np.mod(i, 2 * n)
            return np.where(i < n, i, 2 * n - 1 - i)

        take = lambda k: np.take(a, refl(idx + k), axis=axis)
        acc = a * w[r]
        for j in range(-r, 0):
            acc = acc + (take(j) + take(-j)) * w[r + j]
        a = acc
    return a


def interp_init(op: "Operator", y):
    """solvers.py:237-254 (_interp_init): MSFA normalised-convolution
    inpainting, CACTI adjoint / max(gram, 1e-12), plain adjoint otherwise."""
    xt = op.adjoint(y)
    if op.kind == "msfa":
        out = np.zeros_like(xt)
        for c in range(xt.shape[2]):
            num = gaussian_filter_reflect(xt[:, :, c])
            den = gaussian_filter_reflect(op.masks[:, :, c])
            np.divide(num, den, out=out[:, :, c], where=den > 1e-12)
        return out
    if op.kind == "cacti":
        return xt / np.maximum(op.gram, 1e-12)
    return xt


def init_x(op: "Operator", y, init="adjoint"):
    """solvers.py:229-234 (_init_x)."""
    if init == "zero":
        return np.zeros(op.x_shape)
    if init == "interp":
        return interp_init(op, y)
    return op.adjoint(y)


def psnr(a, b, peak=1.0):
    """metrics.py:26-37 (cap 100 dB)."""
    mse = np.mean((np.asarray(a, float) - np.asarray(b, float)) ** 2)
    if mse == 0.0:
        return 100.0
    return min(10.0 * np.log10(peak ** 2 / mse), 100.0)


def gap_solve(op: Operator, y, max_iters, patch_size=8, group_size=64, max_corners=512,
              exemplar_stride=6, edge_threshold=0.2, refresh=5, sigma0=0.10, sigma_min=0.003,
              peak=1.0, c_weight=2.0 * np.sqrt(2.0), eps=1e-16, min_separation=None,
              clip=True, ref=None, trace=None, positions_override=None, init="adjoint",
              regularizer="glr", bm_window=20, bm_stride=1, rerank=False, tv_weight=0.05,
              tv_iters=20):
    """solvers.py:284-308 with the nonlocal regularizers or "tv" (solvers.py:170-210):
    "glr" (optionally with the pixel re-rank) and the block-matching
    baselines (see _glr_match).

    ``clip=False`` is the documented policy for complex (re, im) images
    (DESIGN.md). ``trace`` (a list) receives per-refresh anchors
    and positions; ``positions_override`` (refresh index -> (anchors,
    positions)) locks matching for positions-locked parity.
    Returns (x, residuals, psnrs)."""
    p = patch_size
    sep = -(-p // 4) if min_separation is None else min_separation
    x = init_x(op, y, init)
    lo, hi = -0.5 * peak, 1.5 * peak
    positions, last = None, -1
    residuals, psnrs = [], []
    refresh_no = 0
    for it in range(max_iters):
        sigma = sigma_at(it, max_iters, sigma0, sigma_min, peak)
        if regularizer == "tv":
            positions = []
        elif positions is None or it - last >= refresh:
            if positions_override is not None:
                anchors, positions = positions_override[refresh_no]
            else:
                anchors, positions = _glr_match(x, p, group_size, max_corners, exemplar_stride,
                                                edge_threshold, sep, regularizer, bm_window,
                                                bm_stride, rerank)
            if trace is not None:
                trace.append((list(anchors), [list(q) for q in positions]))
            last = it
            refresh_no += 1
        if regularizer == "tv":
            z = tv_denoise(x, tv_weight, tv_iters)
        else:
            z = glr_regularize(x, positions, p, sigma, c_weight, eps) if positions else x.copy()
        x = z + op.adjoint(safe_div(y - op.forward(z), op.gram))
        if clip:
            x = np.clip(x, lo, hi)
        residuals.append(float(np.linalg.norm((y - op.forward(x)).ravel())))
        if ref is not None:
            psnrs.append(psnr(ref, np.clip(x, 0.0, peak), peak))
    out = np.clip(x, 0.0, peak) if clip else x
    return out, residuals, psnrs


def _glr_match(x, p, group_size, max_corners, exemplar_stride, edge_threshold, sep,
               regularizer="glr", bm_window=20, bm_stride=1, rerank=False):
    """solvers.py:154-167 + 187-203: (anchors, positions) of one refresh for
    the "glr" regularizer (corners + grid at 3*stride, edge-overlap global
    match, optional pixel re-rank) and the block-matching baselines
    ("nlr-bm": grid at stride only, "nlr-corner-bm": corners only,
    "nlr-corner-uniform-bm": corners + grid at 3*stride)."""
    h, w = x.shape[:2]
    if regularizer == "nlr-bm":
        anchors, _ = select_exemplars([], (h, w), p, uniform_interval=exemplar_stride)
    else:
        corners = detect_corners(x, max_n=max_corners, nms_radius=-(-p // 2), quality=0.01)
        interval = None if regularizer == "nlr-corner-bm" else 3 * exemplar_stride
        anchors, _ = select_exemplars(corners, (h, w), p, uniform_interval=interval)
    if not anchors:
        return anchors, []
    if regularizer != "glr":
        positions, _ = block_match(x, anchors, p, group_size, bm_window, bm_stride)
        return anchors, positions
    gh, gv = sobel_gradients(x)
    maps = binarize_gradients(gh, gv, edge_threshold)
    heat = similarity_heatmap(maps, anchors, p)
    positions, _ = match_positions(heat, anchors, group_size, sep)
    if rerank:
        positions = rerank_pixel(x, positions, p)
    return anchors, positions


def admm_solve(op: Operator, y, max_iters, patch_size=8, group_size=64, max_corners=512,
               exemplar_stride=6, edge_threshold=0.2, refresh=5, sigma0=0.10, sigma_min=0.003,
               peak=1.0, rho=0.01, c_weight=2.0 * np.sqrt(2.0), eps=1e-16, min_separation=None,
               clip=True, ref=None, trace=None, init="adjoint", regularizer="glr",
               bm_window=20, bm_stride=1, rerank=False, tv_weight=0.05, tv_iters=20):
    """solvers.py:311-341 — scaled-form ADMM with the "glr" regularizer:
    m = z - u; x = clip(m + A^T((y - A m) / (rho + gram))); z = clip(R(x + u));
    u = u + x - z. Returns (x, residuals, psnrs)."""
    p = patch_size
    sep = -(-p // 4) if min_separation is None else min_separation
    z = init_x(op, y, init)
    u = np.zeros_like(z)
    lo, hi = -0.5 * peak, 1.5 * peak
    positions, last = None, -1
    residuals, psnrs = [], []
    x = z.copy()
    for it in range(max_iters):
        m = z - u
        x = m + op.adjoint((y - op.forward(m)) / (rho + op.gram))
        if clip:
            x = np.clip(x, lo, hi)
        v = x + u
        sigma = sigma_at(it, max_iters, sigma0, sigma_min, peak)
        if regularizer == "tv":
            positions = []
        elif positions is None or it - last >= refresh:
            anchors, positions = _glr_match(v, p, group_size, max_corners, exemplar_stride,
                                            edge_threshold, sep, regularizer, bm_window,
                                            bm_stride, rerank)
            if trace is not None:
                trace.append((list(anchors), [list(q) for q in positions]))
            last = it
        if regularizer == "tv":
            z = tv_denoise(v, tv_weight, tv_iters)
        else:
            z = glr_regularize(v, positions, p, sigma, c_weight, eps) if positions else v.copy()
        if clip:
            z = np.clip(z, lo, hi)
        u = u + x - z
        residuals.append(float(np.linalg.norm((y - op.forward(x)).ravel())))
        if ref is not None:
            psnrs.append(psnr(ref, np.clip(x, 0.0, peak), peak))
    out = np.clip(x, 0.0, peak) if clip else x
    return out, residuals, psnrs


def ssim(a, b, peak=1.0, win_size=11, win_sigma=1.5):
    """metrics.py:40-78 — mean SSIM over all valid 11x11 Gaussian windows,
    averaged over channels (2-D window = outer product of the normalised
    1-D taps; sums evaluated with the separable form)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    h, w, c = a.shape
    if h < win_size or w < win_size:
        raise ValueError(f"image {h}x{w} smaller than {win_size}x{win_size} window")
    ax = np.arange(win_size) - (win_size - 1) / 2.0
    g = np.exp(-(ax ** 2) / (2.0 * win_sigma ** 2))
    g = g / g.sum()
    c1, c2 = (0.01 * peak) ** 2, (0.03 * peak) ** 2

    def filt(z):  # valid separable correlation, rows then columns
        from numpy.lib.stride_tricks import sliding_window_view
        r = (sliding_window_view(z, win_size, axis=1) * g).sum(axis=-1)
        return (sliding_window_view(r, win_size, axis=0) * g).sum(axis=-1)

    vals = []
    for ch in range(c):
        x, y = a[:, :, ch], b[:, :, ch]
        ma, mb = filt(x), filt(y)
        va = filt(x * x) - ma ** 2
        vb = filt(y * y) - mb ** 2
        cov = filt(x * y) - ma * mb
        num = (2 * ma * mb + c1) * (2 * cov + c2)
        den = (ma ** 2 + mb ** 2 + c1) * (va + vb + c2)
        vals.append(float(np.mean(num / den)))
    return float(np.mean(vals))


def heat_flops(h, w, c, p, n):
    """2*M*(4*C*P^2)*N flops per refresh."""
    return 2.0 * (h - p + 1) * (w - p + 1) * 4 * c * p * p * n


__all__ = [name for name in dir() if not name.startswith("_") and name != "math"]
