"""Seeded synthetic inputs for the BASELINE.json configurations.

No public dataset ships with the reference (Kobe/Runner/fastMRI/CAVE are
absent), so these numpy generators stand in for them with the
configs' shapes, sizes and value distributions. Every input is
generated in float64, rounded once to float32 and returned as float64, so the
GPU path and the CPU oracle see identical values.

  C1  CACTI 256x256x8,   GAP 30 it, P=8, K=64, max_corners=512 (+ reference grid)
  C2  CACTI 1024x1024x24, GAP 50 it, P=8, K=64, 4096 exemplars
  C3  MRI 512x512 complex (re, im), Cartesian VD 25 %, GAP 40 it, P=8, K=48, 2048 ex.
      (897 corners + the interval-15 grid = 2048 anchors on the first refresh)
  C4  MSFA 512x512x16, periodic 4x4, GAP 30 it, P=8, K=64, 2048 exemplars, init="interp"
  C5  2048x2048x1 stage sweep (matching / top-K / WNNM / aggregation only)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .matching import MatchConfig
from .operators import bernoulli_masks, msfa_pattern


def _f32(a: np.ndarray) -> np.ndarray:
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def blob_texture_image(h: int, w: int, rng, n_blobs: int = 40, tex: int = 16) -> np.ndarray:
    """Sum of anisotropic Gaussian blobs plus a tiled tex x tex random texture,
    normalised to [0, 1] (C1/C2/C5 base image)."""
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    img = np.zeros((h, w))
    for _ in range(n_blobs):
        cy, cx = rng.uniform(0, h), rng.uniform(0, w)
        sy, sx = rng.uniform(0.02, 0.15) * h, rng.uniform(0.02, 0.15) * w
        th = rng.uniform(0, np.pi)
        c, s = np.cos(th), np.sin(th)
        dy, dx = yy - cy, xx - cx
        u = (c * dx + s * dy) / sx
        v = (-s * dx + c * dy) / sy
        img += rng.uniform(0.3, 1.0) * np.exp(-0.5 * (u * u + v * v))
    t = rng.random((tex, tex))
    img = img / max(img.max(), 1e-12) + 0.35 * np.tile(t, (h // tex + 1, w // tex + 1))[:h, :w]
    img -= img.min()
    return img / max(img.max(), 1e-12)


def cacti_scene(h: int, w: int, t: int, seed: int) -> np.ndarray:
    """Frames of the blob+texture image translated 1-2 px per frame."""
    rng = np.random.default_rng(seed)
    base = blob_texture_image(h + 2 * t + 2, w + 2 * t + 2, rng)
    frames = []
    oy = ox = 0
    for _ in range(t):
        frames.append(base[oy:oy + h, ox:ox + w])
        oy += int(rng.integers(1, 3))
        ox += int(rng.integers(1, 3))
    return _f32(np.stack(frames, axis=2))


def ellipse_phantom(h: int, w: int, rng, n: int = 20) -> np.ndarray:
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    img = np.zeros((h, w))
    for _ in range(n):
        cy, cx = rng.uniform(0.2, 0.8) * h, rng.uniform(0.2, 0.8) * w
        ay, ax = rng.uniform(0.03, 0.3) * h, rng.uniform(0.03, 0.3) * w
        th = rng.uniform(0, np.pi)
        c, s = np.cos(th), np.sin(th)
        dy, dx = yy - cy, xx - cx
        inside = ((c * dx + s * dy) / ax) ** 2 + ((-s * dx + c * dy) / ay) ** 2 <= 1.0
        img[inside] = rng.uniform(0.0, 1.0)
    return img


def smooth_field(h: int, w: int, rng, n: int = 6) -> np.ndarray:
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64) / max(h, w)
    f = np.zeros((h, w))
    for _ in range(n):
        f += rng.normal() * np.cos(2 * np.pi * (rng.uniform(0, 2) * yy + rng.uniform(0, 2) * xx)
                                   + rng.uniform(0, 2 * np.pi))
    return f


def cartesian_vd_mask(h: int, w: int, fraction: float, center_lines: int, seed: int) -> np.ndarray:
    """Cartesian variable-density k-space mask (phase-encode rows), keeping the
    central ``center_lines`` rows and sampling the rest with a density that
    decays with distance from the centre, ``fraction`` of all rows in total.
    Returned in unshifted FFT order (like glr.operators.radial_mask)."""
    rng = np.random.default_rng(seed)
    n_keep = int(round(fraction * h))
    c0 = h // 2 - center_lines // 2
    rows = set(range(c0, c0 + center_lines))
    dist = np.abs(np.arange(h) - h / 2.0) / (h / 2.0)
    prob = (1.0 - dist) ** 2 + 1e-3
    prob[list(rows)] = 0.0
    prob /= prob.sum()
    extra = rng.choice(h, size=max(0, n_keep - len(rows)), replace=False, p=prob)
    rows.update(int(r) for r in extra)
    cen = np.zeros((h, w))
    cen[sorted(rows), :] = 1.0
    return np.fft.ifftshift(cen)


@dataclass
class Workload:
    name: str
    kind: str                 # "cacti" | "msfa" | "fourier"
    scene: np.ndarray         # (H, W, C) float64 (fp32-rounded)
    masks: np.ndarray         # (H, W, T) masks, or (H, W) k-space mask
    y: np.ndarray             # measurement (noisy)
    max_iters: int
    match: MatchConfig
    noise: float
    init: str = "adjoint"     # SolverConfig.init (solvers.py:47)

    @property
    def shape(self):
        return self.scene.shape

    def solver_config(self, **overrides):
        """The configuration's SolverConfig (iterations, matching, init)."""
        from .solvers import SolverConfig
        kw = dict(max_iters=self.max_iters, match=self.match, init=self.init)
        kw.update(overrides)
        return SolverConfig(**kw)


def _masksum(x, masks):
    return (masks * x).sum(axis=2, keepdims=True)


def make(name: str, seed: int = 0) -> Workload:
    """Build one BASELINE.json configuration (see module docstring)."""
    rng = np.random.default_rng(10_000 + seed)
    if name in ("C1", "C2"):
        h, w, t, iters, corners, stride = ((256, 256, 8, 30, 512, 6) if name == "C1"
                                           else (1024, 1024, 24, 50, 4096, 342))
        scene = cacti_scene(h, w, t, seed)
        masks = bernoulli_masks(h, w, t, seed=seed + 1)
        y = _masksum(scene, masks) + rng.normal(0.0, 0.01, (h, w, 1))
        mc = MatchConfig(patch_size=8, group_size=64, max_corners=corners, exemplar_stride=stride)
        return Workload(name, "cacti", scene, masks, y, iters, mc, 0.01)
    if name == "C3":
        h = w = 512
        mag = ellipse_phantom(h, w, rng)
        ph = 0.5 * np.pi * np.tanh(smooth_field(h, w, rng))
        scene = _f32(np.stack([mag * np.cos(ph), mag * np.sin(ph)], axis=2))
        mask = cartesian_vd_mask(h, w, 0.25, 32, seed + 1)
        z = scene[:, :, 0] + 1j * scene[:, :, 1]
        y = mask * (np.fft.fft2(z, norm="ortho")
                    + 0.005 * (rng.normal(size=(h, w)) + 1j * rng.normal(size=(h, w))))
        # the piecewise-constant phantom yields 944 Shi-Tomasi corners (nms 4);
        # the reference's glr mode unions them with a uniform grid
        # (solvers.py:165-167), here at interval 15 (exemplar_stride 5, 34 x 34
        # anchors): the first 897 corners plus the grid deduplicate to exactly
        # the config's 2048 exemplars on the first refresh
        mc = MatchConfig(patch_size=8, group_size=48, max_corners=897, exemplar_stride=5)
        return Workload(name, "fourier", scene, mask, y, 40, mc, 0.005)
    if name == "C4":
        h = w = 512
        bands = 16
        lam = np.linspace(0.0, 1.0, bands)
        spectra = np.stack([np.clip(0.5 + 0.4 * np.sin(2 * np.pi * (rng.uniform(0.3, 1.5) * lam
                                                                      + rng.uniform())), 0, 1)
                            for _ in range(6)])            # (6, bands)
        ab = np.stack([blob_texture_image(h, w, rng, n_blobs=12, tex=8) for _ in range(6)], 2)
        ab /= ab.sum(axis=2, keepdims=True) + 1e-12
        scene = _f32(np.clip(ab @ spectra, 0.0, 1.0))
        masks = msfa_pattern("periodic-4x4", bands, h, w)
        y = _masksum(scene, masks) + rng.normal(0.0, 0.005, (h, w, 1))
        mc = MatchConfig(patch_size=8, group_size=64, max_corners=2048, exemplar_stride=171)
        # init="interp", as the reference's own MSFA runs (scripts/run_msfa_demo.py:38,
        # tests/test_acceptance.py:231): from the adjoint the iterate never moves --
        # every patch of a group shares the anchor's mosaic phase (the edge maps of a
        # mosaic repeat with the 4x4 pattern), so a row of the group matrix is sampled
        # in all of its columns or in none, M Wm keeps the unsampled rows at zero and
        # the projection restores the sampled ones: x is a fixed point, bit for bit
        # (measured: 30 identical iterates). The normalised-convolution start fills
        # every band, and the solve then iterates like the reference's demo.
        return Workload(name, "msfa", scene, masks, y, 30, mc, 0.005, init="interp")
    if name == "C5":
        h = w = 2048
        scene = _f32(blob_texture_image(h, w, rng)[:, :, None])
        mc = MatchConfig(patch_size=8, group_size=64, max_corners=16384, exemplar_stride=683)
        return Workload(name, "cacti", scene, np.ones((h, w, 1)), _masksum(scene, np.ones((h, w, 1))),
                        0, mc, 0.0)
    raise ValueError(f"unknown workload {name!r}")


def operator_for(wl: Workload):
    from .operators import cacti_operator, fourier_operator, msfa_operator
    if wl.kind == "cacti":
        return cacti_operator(wl.masks)
    if wl.kind == "msfa":
        return msfa_operator(wl.masks)
    return fourier_operator(wl.masks, channels=2)
