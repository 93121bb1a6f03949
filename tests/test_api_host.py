"""Host-side logic of the reference-facing API: dataclass validation, mask
generators and argument checks that raise before any launch (CPU tests)."""

import numpy as np
import pytest

import paper_2301_03047_b200 as G
from conftest import load_golden


def test_match_config_validation_and_defaults():
    with pytest.raises(ValueError, match="group_size"):
        G.MatchConfig(group_size=0)
    with pytest.raises(ValueError, match="patch_size"):
        G.MatchConfig(patch_size=1)
    with pytest.raises(ValueError, match="mode"):
        G.MatchConfig(mode="nope")
    with pytest.raises(ValueError, match="backend"):
        G.MatchConfig(backend="nope")
    with pytest.raises(ValueError, match="bm_window"):
        G.MatchConfig(mode="bm-uniform", patch_size=8, bm_window=4)
    cfg = G.MatchConfig(patch_size=8)
    assert cfg.sep == 2 and cfg.nms == 4
    cfg = G.MatchConfig(patch_size=12)
    assert cfg.sep == 3 and cfg.nms == 6
    cfg = G.MatchConfig(patch_size=5, min_separation=0, nms_radius=1)
    assert cfg.sep == 0 and cfg.nms == 1


def test_solver_config_validation_and_schedule():
    for bad in [dict(algorithm="sgd"), dict(regularizer="deep-prior"), dict(max_iters=0),
                dict(match_refresh_interval=0), dict(sigma0=0.001, sigma_min=0.01),
                dict(init="oracle")]:
        with pytest.raises(ValueError):
            G.SolverConfig(**bad)
    cfg = G.SolverConfig(sigma0=0.1, sigma_min=0.001, max_iters=100, peak=2.0)
    assert cfg.sigma_at(0) == pytest.approx(0.2)
    assert cfg.sigma_at(100) == pytest.approx(0.002)
    assert cfg.sigma_at(50) == pytest.approx(np.sqrt(0.1 * 0.001) * 2.0)


def test_wnnm_params_validation():
    for bad in [dict(c_weight=0.0), dict(eps=0.0), dict(noise_sigma=-1.0)]:
        with pytest.raises(ValueError):
            G.WnnmParams(**bad)


def test_mask_generators_match_reference_golden():
    g = load_golden("operators")
    np.testing.assert_array_equal(G.bernoulli_masks(9, 7, 3, seed=7), g["bern_seed7"])
    np.testing.assert_array_equal(G.msfa_pattern("periodic-4x4", 16, 16, 20), g["msfa_masks"])
    np.testing.assert_array_equal(G.radial_mask(16, 16, 5), g["four_mask"])
    np.testing.assert_array_equal(G.bernoulli_masks(16, 20, 8, seed=3), g["cacti_masks"])


def test_radial_mask_properties():
    for h, w, n in ((16, 16, 1), (32, 24, 5), (64, 64, 30)):
        m = np.fft.fftshift(G.radial_mask(h, w, n))
        assert m[h // 2, w // 2] == 1.0
        ys, xs = np.nonzero(m)
        for r, c in zip(ys, xs):
            r2, c2 = 2 * (h // 2) - r, 2 * (w // 2) - c
            if 0 <= r2 < h and 0 <= c2 < w:
                assert m[r2, c2] == 1.0
    m = np.fft.fftshift(G.radial_mask(17, 17, 1))
    assert np.array_equal(np.nonzero(m.sum(axis=1))[0], [8])
    assert G.radial_mask(64, 64, 128).mean() >= 0.95
    with pytest.raises(ValueError):
        G.radial_mask(8, 8, 0)


def test_msfa_pattern_and_partition_errors():
    with pytest.raises(ValueError, match="requires C"):
        G.msfa_pattern("periodic-4x4", 9, 8, 8)
    with pytest.raises(ValueError, match="out of range"):
        G.msfa_pattern("custom-tile", 2, 8, 8, tile=np.array([[0, 2], [1, 0]]))
    with pytest.raises(ValueError, match="unknown"):
        G.msfa_pattern("hexagonal", 4, 8, 8)
    with pytest.raises(ValueError, match="tile"):
        G.msfa_pattern("custom-tile", 4, 8, 8)
    with pytest.raises(ValueError, match="orthogonal"):
        G.msfa_operator(np.ones((4, 4, 2)))
    masks = np.zeros((4, 4, 2))
    masks[:, :, 0] = 1.0
    masks[0, 0, 0] = 0.0
    with pytest.raises(ValueError, match="partition"):
        G.msfa_operator(masks)
    for kind, c in [("bayer-like-2x2", 4), ("periodic-3x3", 9), ("periodic-4x4", 16)]:
        m = G.msfa_pattern(kind, c, 48, 48)
        assert np.array_equal(m.sum(axis=2), np.ones((48, 48)))


def test_validation_before_launch():
    with pytest.raises(ValueError, match="nonnegative"):
        G.binarize_gradients(np.zeros((3, 3, 1)), np.zeros((3, 3, 1)), th=-0.1)
    with pytest.raises(ValueError, match="differ"):
        G.binarize_gradients(np.zeros((3, 3, 1)), np.zeros((3, 4, 1)))
    with pytest.raises(ValueError, match="too small"):
        G.sobel_gradients(np.zeros((2, 5, 1)))
    with pytest.raises(ValueError, match="max_n"):
        G.detect_corners(np.zeros((8, 8, 1)), max_n=0)
    with pytest.raises(ValueError, match="exceeds"):
        G.select_exemplars([], (6, 6), 8)
    with pytest.raises(ValueError, match="anchor 1"):
        G.gather_group(np.zeros((4, 4, 1)), [(0, 0), (3, 0)], 2)
    g = G.PatchGroup(patch_size=2, positions=[(0, 0)], matrix=np.zeros((4, 1)))
    with pytest.raises(ValueError, match="accumulator"):
        G.scatter_group(np.zeros((4, 4, 1)), np.zeros((4, 5, 1)), g)
    m = np.ones((3, 3))
    m[1, 1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        G.wnnm_prox(m, G.WnnmParams())
    op = G.cacti_operator(G.bernoulli_masks(8, 8, 2, seed=0))
    with pytest.raises(ValueError, match="measurement shape"):
        G.gap_solve(op, np.zeros((8, 9, 1)), G.SolverConfig())
    with pytest.raises(ValueError, match="mask"):
        G.operators.cacti_forward(np.zeros((8, 8, 3)), np.zeros((8, 8, 4)))
    with pytest.raises(ValueError, match="integer overlap counts"):
        G.top_k_positions(np.full((4, 4), 0.5), (0, 0), 3, 1)
    with pytest.raises(ValueError, match="larger"):
        G.xcorr2_valid_batch(np.zeros((3, 3, 1)), np.zeros((1, 5, 5, 1)))
    with pytest.raises(ValueError, match="channel"):
        G.xcorr2_valid_batch(np.zeros((8, 8, 2)), np.zeros((1, 3, 3, 1)))
    with pytest.raises(ValueError, match="square"):
        G.xcorr2_valid_batch(np.zeros((8, 8, 1)), np.zeros((1, 3, 4, 1)))
    bmc = G.MatchConfig(patch_size=4, group_size=4, bm_window=4, mode="bm-uniform")
    ex = G.ExemplarSet(anchors=[(0, 0), (5, 0)], tags=["uniform"] * 2, patch_size=4)
    with pytest.raises(ValueError, match="anchor 1"):
        G.block_match(np.zeros((8, 8, 1)), ex, bmc)
    with pytest.raises(ValueError, match="bm_window"):
        G.MatchConfig(patch_size=8, bm_window=4, mode="bm-corner")


def test_block_match_has_no_cpu_fallback():
    """Valid block-matching input without a device: the native path raises,
    nothing computes on the host."""
    from paper_2301_03047_b200 import _native as N
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    bmc = G.MatchConfig(patch_size=4, group_size=4, bm_window=4, mode="bm-uniform")
    ex = G.ExemplarSet(anchors=[(0, 0)], tags=["uniform"], patch_size=4)
    with pytest.raises(N.NativeUnavailable):
        G.block_match(np.zeros((8, 8, 1)), ex, bmc)


def test_report_serialization():
    rep = G.ReconReport()
    rep.add(iteration=0, residual=1.5, match_ms=2.0, lowrank_ms=3.0, projection_ms=0.5)
    assert rep.to_csv().splitlines()[0].startswith("iteration,residual")
    assert rep.to_jsonl().strip().startswith("{")
    assert rep.final_psnr is None


def test_divergence_guard():
    from paper_2301_03047_b200.solvers import _check_divergence
    with pytest.raises(G.SolverDivergenceError, match="10x"):
        _check_divergence([1.0] + [20.0] * 20, y_norm=1.0)
    _check_divergence([1e-15] + [1e-9] * 20, y_norm=1.0)


def test_workload_solver_configs():
    """BASELINE configurations: iteration counts, group sizes and the MSFA
    configuration's init (the reference's own MSFA runs start from "interp",
    scripts/run_msfa_demo.py:38; from the adjoint the iterate is a fixed point)."""
    from paper_2301_03047_b200 import workloads
    expect = {"C1": (30, 64, "adjoint"), "C4": (30, 64, "interp")}
    for name, (iters, k, init) in expect.items():
        wl = workloads.make(name)
        cfg = wl.solver_config()
        assert (cfg.max_iters, cfg.match.group_size, cfg.init) == (iters, k, init)
        assert wl.solver_config(max_iters=3).max_iters == 3


def test_msfa_adjoint_start_is_a_fixed_point_of_the_reference_algorithm():
    """Why C4 runs from init="interp": from the adjoint start the edge maps of
    a (smooth) mosaic image repeat with the 4x4 pattern, every patch of a group
    shares the anchor's mosaic phase, so a row of the group matrix is sampled
    in all of its columns or in none: GAP-GLR iterations of the oracle
    (solvers.py:284-308) leave the unsampled entries at zero (to rounding) and
    return the sampled ones to the measurement."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
    import glr_oracle as O
    rng = np.random.default_rng(0)
    h = w = 48
    bands = 16
    yy, xx = np.mgrid[0:h, 0:w]
    scene = np.clip(0.5 + 0.2 * np.sin(yy / 9.0)[..., None] * np.cos(xx / 11.0)[..., None]
                    + 0.1 * np.linspace(0, 1, bands)[None, None, :]
                    + 0.01 * rng.standard_normal((h, w, bands)), 0, 1)
    masks = O.msfa_pattern_periodic(4, h, w)
    op = O.Operator("msfa", masks=masks)
    y = O.masksum_forward(scene, masks)
    x0 = np.clip(op.adjoint(y), 0.0, 1.0)
    x2, _, _ = O.gap_solve(op, y, 2, patch_size=8, group_size=8, max_corners=16,
                           exemplar_stride=4)
    assert np.abs(x2[masks == 0]).max() < 1e-12  # (exactly 0 on the device path: M Wm of a zero row)
    assert np.abs(x2 - x0).max() < 1e-12
    # the normalised-convolution start fills every band
    assert np.all(O.init_x(op, y, "interp") > 0.0)
