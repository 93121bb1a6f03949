"""Config-shaped parity (GPU): reduced versions of the BASELINE configs
checked end to end against the oracle, and the full-size C2 refresh checked
through size-independent properties (self-maximum, exchange symmetry,
separation, determinism, WNNM vs SVD on sampled groups)."""

import numpy as np
import pytest

import glr_oracle as O

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2301_03047_b200")
from paper_2301_03047_b200 import workloads  # noqa: E402


def _compare_runs(op_g, op_o, y, iters, mc, clip=True, ref=None):
    cfg = G.SolverConfig(max_iters=iters, match=mc)
    trace = []
    x, rep = G.gap_solve(op_g, y, cfg, trace=trace, ref=ref)
    otrace = []
    xo, res_o, _ = O.gap_solve(op_o, y, iters, patch_size=mc.patch_size,
                               group_size=mc.group_size, max_corners=mc.max_corners,
                               exemplar_stride=mc.exemplar_stride, clip=clip, trace=otrace)
    assert len(trace) == len(otrace)
    for j, ((a, p), (ao, po)) in enumerate(zip(trace, otrace)):
        assert np.array_equal(np.asarray(a), np.asarray(ao)), f"anchors differ at refresh {j}"
        assert np.array_equal(np.asarray(p), np.asarray(po)), f"positions differ at refresh {j}"
    assert np.abs(x - xo).max() <= 1e-6
    res = [r["residual"] for r in rep.rows]
    ynorm = float(np.linalg.norm(np.asarray(y).ravel()))
    np.testing.assert_allclose(res, res_o, rtol=1e-6, atol=1e-9 * ynorm)
    return x, xo


def test_c1_style_cacti_reduced():
    rng = np.random.default_rng(1)
    scene = workloads.cacti_scene(96, 96, 8, seed=3)
    masks = G.bernoulli_masks(96, 96, 8, seed=4)
    y = O.masksum_forward(scene, masks) + rng.normal(0, 0.01, (96, 96, 1))
    mc = G.MatchConfig(patch_size=8, group_size=64, max_corners=64, exemplar_stride=6)
    _compare_runs(G.cacti_operator(masks), O.Operator("cacti", masks=masks), y, 7, mc)


def test_c3_style_complex_mri_reduced():
    rng = np.random.default_rng(2)
    h = w = 64
    mag = workloads.ellipse_phantom(h, w, rng, n=8)
    ph = 0.5 * np.pi * np.tanh(workloads.smooth_field(h, w, rng))
    scene = np.stack([mag * np.cos(ph), mag * np.sin(ph)], 2).astype(np.float32).astype(float)
    mask = workloads.cartesian_vd_mask(h, w, 0.25, 8, seed=5)
    assert abs(mask.mean() - 0.25) < 0.02
    z = scene[:, :, 0] + 1j * scene[:, :, 1]
    y = mask * (np.fft.fft2(z, norm="ortho")
                + 0.005 * (rng.normal(size=(h, w)) + 1j * rng.normal(size=(h, w))))
    mc = G.MatchConfig(patch_size=8, group_size=48, max_corners=48, exemplar_stride=6)
    _compare_runs(G.fourier_operator(mask, channels=2),
                  O.Operator("fourier", mask=mask, channels=2), y, 6, mc, clip=False)


def test_c4_style_msfa_reduced():
    rng = np.random.default_rng(3)
    h = w = 64
    spectra = rng.random((6, 16))
    ab = np.stack([workloads.blob_texture_image(h, w, rng, n_blobs=6, tex=8) for _ in range(6)], 2)
    ab /= ab.sum(axis=2, keepdims=True)
    scene = np.clip(ab @ spectra, 0, 1).astype(np.float32).astype(float)
    masks = G.msfa_pattern("periodic-4x4", 16, h, w)
    y = O.masksum_forward(scene, masks) + rng.normal(0, 0.005, (h, w, 1))
    mc = G.MatchConfig(patch_size=8, group_size=64, max_corners=40, exemplar_stride=10)
    _compare_runs(G.msfa_operator(masks), O.Operator("msfa", masks=masks), y, 6, mc)


@pytest.fixture(scope="module")
def c2_refresh():
    from paper_2301_03047_b200.engine import GlrEngine
    from paper_2301_03047_b200 import _device as D
    wl = workloads.make("C2")
    eng = GlrEngine(wl.shape, wl.match)
    x = D.f64(wl.scene)
    n = eng.refresh(x)
    return wl, eng, x, n


def test_c2_full_size_heat_properties(c2_refresh):
    from paper_2301_03047_b200 import _device as D, _native as N
    import torch
    wl, eng, x, n = c2_refresh
    assert n >= 4096
    h, w, c = wl.shape
    p = wl.match.patch_size
    oh, ow = h - p + 1, w - p + 1
    # recompute the heat map for 256 sampled exemplars and check self-maximum
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(n, 256, replace=False))
    anc = D.host(eng.anchors[:n])[idx]
    anc_d = D.i32(anc)
    heat = D.empty((256, eng.stride), torch.int16)
    ws = D.empty((N.query("glr_heat_workspace", c, p, 256),), torch.uint8)
    N.call("glr_heat_map", eng.stack.data_ptr(), h, w, c, p, eng.expand, anc_d.data_ptr(), 256,
           None, heat.data_ptr(), ws.data_ptr(), ws.numel(), D.stream())
    hv = D.host(heat)[:, :oh * ow].view(np.uint16).astype(np.int64)
    flat = anc[:, 0] * ow + anc[:, 1]
    own = hv[np.arange(256), flat]
    assert np.array_equal(own, hv.max(axis=1)), "anchor score must be the slice maximum"
    # exchange symmetry: heat_a(anchor_b) == heat_b(anchor_a)
    sub = hv[:, flat]
    assert np.array_equal(sub, sub.T)
    # own score = edge count of the exemplar's own patch (oracle on the maps)
    gh, gv = O.sobel_gradients(wl.scene)
    maps = np.concatenate(O.binarize_gradients(gh, gv, 0.2), axis=2)
    for t in range(0, 256, 37):
        r, cc = anc[t]
        assert own[t] == int(maps[r:r + p, cc:cc + p, :].sum())


def test_c2_full_size_topk_properties(c2_refresh):
    wl, eng, x, n = c2_refresh
    anchors, pos, pad = eng.positions_host()
    sep = wl.match.sep
    assert np.array_equal(pos[:, 0, :], anchors)
    assert (pad == 0).all()
    for g in range(0, n, 97):
        q = pos[g]
        d = np.abs(q[:, None, :] - q[None, :, :]).max(axis=2)
        np.fill_diagonal(d, sep + 1)
        assert d.min() > sep, g


def test_c2_full_size_wnnm_sampled_vs_svd_and_determinism(c2_refresh):
    from paper_2301_03047_b200 import _device as D
    wl, eng, x, n = c2_refresh
    anchors, pos, _ = eng.positions_host()
    p = wl.match.patch_size
    sigma = 0.05
    for g in (0, n // 3, n - 1):
        m = O.gather_group(wl.scene, [tuple(t) for t in pos[g]], p)
        out = G.wnnm_prox(m, G.WnnmParams(noise_sigma=sigma))
        assert np.abs(out - O.wnnm_prox(m, sigma)).max() < 1e-9
    eng.regularize(x, sigma)
    a1 = D.host(eng.acc).copy()
    eng.warm = False
    eng.regularize(x, sigma)
    assert np.array_equal(a1, D.host(eng.acc))


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_configs_run(name):
    from paper_2301_03047_b200.solvers import GapRunner
    from paper_2301_03047_b200 import _device as D
    wl = workloads.make(name)
    cfg = G.SolverConfig(max_iters=6, match=wl.match)
    r = GapRunner(workloads.operator_for(wl), cfg)
    y = r.dop.upload_y(wl.y)
    trace = []
    xd = r.run(y, trace=trace)
    xh = D.host(xd)
    assert np.isfinite(xh).all()
    res = np.sqrt(D.host(r.resid_sq))
    # the GAP projection makes the data term consistent up to clipping/rounding
    assert res[-1] <= max(res[0], 1e-9 * float(np.linalg.norm(np.abs(wl.y).ravel())))
    # "2048 exemplars" (corners + reference grid) on the first refresh
    assert len(trace[0][0]) in (2048, 2049), len(trace[0][0])


def test_c1_full_size_free_running_parity():
    """C1 at full size (256x256x8, P=8, K=64, max_corners=512 + reference grid,
    N ~ 700): the first 10 GAP-GLR iterations (2 matching refreshes) against
    the oracle — every refresh's anchors and positions identical, max |x - x_o|
    <= 1e-6 and PSNR within 0.05 dB (SURVEY §8c levels L1-L3)."""
    wl = workloads.make("C1")
    iters = 10
    cfg = G.SolverConfig(max_iters=iters, match=wl.match)
    trace = []
    x, rep = G.gap_solve(G.cacti_operator(wl.masks), wl.y, cfg, trace=trace, ref=wl.scene)
    otrace = []
    xo, res_o, ps_o = O.gap_solve(O.Operator("cacti", masks=wl.masks), wl.y, iters,
                                  patch_size=8, group_size=64, max_corners=512,
                                  exemplar_stride=wl.match.exemplar_stride, trace=otrace,
                                  ref=wl.scene)
    assert len(trace) == len(otrace) == 2
    for (a, p), (ao, po) in zip(trace, otrace):
        assert len(a) > 600
        assert np.array_equal(np.asarray(a), np.asarray(ao))
        assert np.array_equal(np.asarray(p), np.asarray(po))
    assert np.abs(x - xo).max() <= 1e-6
    assert abs(rep.rows[-1]["psnr_db"] - ps_o[-1]) <= 0.05
