"""Pin the CPU oracle (oracle/glr_oracle.py) to golden vectors produced by
running the reference itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import glr_oracle as O
from conftest import load_golden


def test_edges_bitwise():
    g = load_golden("edges")
    for i in range(int(g["n"])):
        x = g[f"x{i}"]
        gh, gv = O.sobel_gradients(x)
        assert np.array_equal(gh, g[f"gh{i}"]) and np.array_equal(gv, g[f"gv{i}"]), i
        maps = np.stack(O.binarize_gradients(gh, gv, 0.2))
        assert np.array_equal(maps, g[f"maps{i}"]), i
        assert np.array_equal(O.corner_response(x), g[f"resp{i}"]), i
        corners = O.detect_corners(x, max_n=40, nms_radius=3)
        assert np.array_equal(np.array(corners, dtype=np.int32).reshape(-1, 2), g[f"corners{i}"])
        anchors, tags = O.select_exemplars(corners, x.shape[:2], 6, uniform_interval=7)
        assert np.array_equal(np.array(anchors, dtype=np.int32).reshape(-1, 2), g[f"anchors{i}"])
        assert np.array_equal(np.array([t == "uniform" for t in tags], dtype=np.uint8),
                              g[f"tags{i}"])


def test_heat_and_topk_bitwise():
    g = load_golden("heat_topk")
    for i in range(int(g["n"])):
        h, w, c, p, n, k, sep = (int(v) for v in g[f"meta{i}"])
        maps = list(g[f"maps{i}"])
        anchors = [tuple(a) for a in g[f"anchors{i}"].tolist()]
        heat = O.similarity_heatmap(maps, anchors, p)
        assert np.array_equal(heat, g[f"heat{i}"]), i
        pos, pads = O.match_positions(heat, anchors, k, sep)
        assert np.array_equal(np.array(pos, dtype=np.int32), g[f"positions{i}"]), i
        assert np.array_equal(np.array(pads), g[f"padded{i}"]), i
        for j, q in enumerate(pos):
            assert np.array_equal(O.gather_group(g[f"x{i}"], q, p), g[f"matrix{i}"][j])


def test_topk_slices_bitwise():
    g = load_golden("topk_slices")
    for i in range(int(g["n"])):
        ar, ac, k, sep, pad = (int(v) for v in g[f"meta{i}"])
        pos, padded = O.top_k_positions(g[f"s{i}"], (ar, ac), k, sep)
        assert padded == pad, i
        assert np.array_equal(np.array(pos, dtype=np.int32), g[f"pos{i}"]), i


def test_wnnm_and_regularize():
    g = load_golden("wnnm")
    for i in range(int(g["n"])):
        m = g[f"m{i}"]
        out = O.wnnm_prox(m, float(g[f"sigma{i}"]))
        np.testing.assert_allclose(out, g[f"out{i}"], atol=1e-12, rtol=0)
        uw = O.wnnm_prox(m, 0.0, uniform_weight=0.3)
        np.testing.assert_allclose(uw, g[f"uw{i}"], atol=1e-12, rtol=0)
    pos = [[tuple(p) for p in grp] for grp in g["reg_pos"].tolist()]
    z = O.glr_regularize(g["reg_x"], pos, 4, 0.05)
    np.testing.assert_allclose(z, g["reg_z"], atol=1e-12, rtol=0)


def test_operators():
    g = load_golden("operators")
    np.testing.assert_array_equal(O.bernoulli_masks(9, 7, 3, seed=7), g["bern_seed7"])
    op = O.Operator("cacti", masks=g["cacti_masks"])
    np.testing.assert_allclose(op.forward(g["cacti_x"]), g["cacti_y"], atol=1e-13)
    np.testing.assert_allclose(op.adjoint(g["cacti_y"]), g["cacti_adj"], atol=1e-13)
    np.testing.assert_allclose(op.gram, g["cacti_gram"], atol=0)
    np.testing.assert_array_equal(O.msfa_pattern_periodic(4, 16, 20), g["msfa_masks"])
    op = O.Operator("msfa", masks=g["msfa_masks"])
    np.testing.assert_allclose(op.forward(g["msfa_x"]), g["msfa_y"], atol=1e-13)
    np.testing.assert_allclose(op.adjoint(g["msfa_y"]), g["msfa_adj"], atol=1e-13)
    op = O.Operator("fourier", mask=g["four_mask"], channels=1)
    np.testing.assert_allclose(op.forward(g["four_x"]), g["four_y"], atol=1e-13)
    np.testing.assert_allclose(op.adjoint(g["four_y"]), g["four_adj"], atol=1e-13)


def test_complex_fourier_adjoint_identity(rng):
    mask = (rng.random((16, 12)) < 0.4).astype(float)
    op = O.Operator("fourier", mask=mask, channels=2)
    for _ in range(20):
        x = rng.standard_normal((16, 12, 2))
        y = rng.standard_normal((16, 12)) + 1j * rng.standard_normal((16, 12))
        lhs = np.vdot(op.forward(x), y).real
        rhs = np.vdot(x, op.adjoint(y)).real
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


@pytest.mark.parametrize("i", [0, 1, 2])
def test_gap_solve_matches_reference_run(i):
    g = load_golden("solves")
    kind = str(g[f"kind{i}"])
    p, k, mc, stride, iters = (int(v) for v in g[f"mc{i}"])
    op = O.Operator(kind, masks=g[f"masks{i}"])
    trace = []
    x, res, ps = O.gap_solve(op, g[f"y{i}"], iters, patch_size=p, group_size=k, max_corners=mc,
                             exemplar_stride=stride, ref=g[f"scene{i}"], trace=trace)
    assert len(trace) == int(g[f"nref{i}"])
    for j, (anc, pos) in enumerate(trace):
        assert np.array_equal(np.array(anc, dtype=np.int32), g[f"anchors{i}_{j}"])
        assert np.array_equal(np.array(pos, dtype=np.int32), g[f"positions{i}_{j}"])
    np.testing.assert_allclose(x, g[f"out{i}"], atol=1e-10, rtol=0)
    np.testing.assert_allclose(res, g[f"resid{i}"], rtol=1e-9)
    np.testing.assert_allclose(ps, g[f"psnr{i}"], atol=1e-8)


def test_admm_solve_matches_reference_run():
    g = load_golden("admm")
    op = O.Operator("cacti", masks=g["masks"])
    trace = []
    x, res, ps = O.admm_solve(op, g["y"], 7, patch_size=4, group_size=8, max_corners=24,
                              exemplar_stride=4, rho=0.01, ref=g["scene"], trace=trace)
    assert len(trace) == int(g["nref"])
    for j, (anc, pos) in enumerate(trace):
        assert np.array_equal(np.array(anc, dtype=np.int32), g[f"anchors_{j}"])
        assert np.array_equal(np.array(pos, dtype=np.int32), g[f"positions_{j}"])
    np.testing.assert_allclose(x, g["out"], atol=1e-10, rtol=0)
    np.testing.assert_allclose(ps, g["psnr"], atol=1e-8)


def test_interp_init_bitwise():
    g = load_golden("interp")
    op = O.Operator("msfa", masks=g["msfa_masks"])
    assert np.array_equal(O.interp_init(op, g["msfa_y"]), g["msfa_init"])
    op = O.Operator("cacti", masks=g["cacti_masks"])
    np.testing.assert_allclose(O.interp_init(op, g["cacti_y"]), g["cacti_init"], atol=1e-13, rtol=0)


def test_gap_solve_interp_init_matches_reference_run():
    g = load_golden("interp")
    op = O.Operator("msfa", masks=g["solve_masks"])
    trace = []
    x, res, ps = O.gap_solve(op, g["solve_y"], 6, patch_size=4, group_size=8, max_corners=24,
                             exemplar_stride=4, ref=g["solve_scene"], trace=trace, init="interp")
    assert len(trace) == int(g["solve_nref"])
    for j, (anc, pos) in enumerate(trace):
        assert np.array_equal(np.array(anc, dtype=np.int32), g[f"solve_anchors_{j}"])
        assert np.array_equal(np.array(pos, dtype=np.int32), g[f"solve_positions_{j}"])
    np.testing.assert_allclose(x, g["solve_out"], atol=1e-10, rtol=0)
    np.testing.assert_allclose(ps, g["solve_psnr"], atol=1e-8)


def test_ssim_psnr_vs_reference():
    g = load_golden("metrics")
    for i in range(int(g["n"])):
        a, b = g[f"a{i}"], np.clip(g[f"b{i}"], 0, 1)
        assert abs(O.ssim(a, b, 1.0) - float(g[f"ssim{i}"])) <= 1e-12
        assert abs(O.psnr(a, b, 1.0) - float(g[f"psnr{i}"])) <= 1e-12


def test_block_match_bitwise():
    g = load_golden("bm")
    for i in range(int(g["bm_n"])):
        p, k, win, st = (int(v) for v in g[f"bm_cfg{i}"])
        pos, pads = O.block_match(g[f"bm_x{i}"], g[f"bm_anchors{i}"], p, k, win, st)
        assert np.array_equal(np.array(pos, dtype=np.int32), g[f"bm_pos{i}"]), i
        assert np.array_equal(np.array(pads, dtype=np.int32), g[f"bm_pad{i}"]), i


def test_rerank_pixel_bitwise():
    g = load_golden("bm")
    for i in range(int(g["rr_n"])):
        p, k = (int(v) for v in g[f"rr_cfg{i}"])
        out = O.rerank_pixel(g[f"rr_x{i}"], g[f"rr_plain{i}"], p)
        assert np.array_equal(np.array(out, dtype=np.int32), g[f"rr_pos{i}"]), i


def _bm_solve_kwargs(g, i):
    import ast
    mc = ast.literal_eval(str(g[f"sv_mc{i}"]))
    kw = dict(patch_size=mc["patch_size"], group_size=mc["group_size"],
              max_corners=mc.get("max_corners", 512), exemplar_stride=mc.get("exemplar_stride", 6),
              bm_window=mc.get("bm_window", 20), bm_stride=mc.get("bm_stride", 1),
              rerank=mc.get("rerank_pixel", False), regularizer=str(g[f"sv_reg{i}"]))
    return kw


@pytest.mark.parametrize("i", range(5))
def test_bm_solves_match_reference_run(i):
    g = load_golden("bm")
    kw = _bm_solve_kwargs(g, i)
    op = O.Operator("cacti", masks=g[f"sv_masks{i}"])
    solve = O.gap_solve if str(g[f"sv_alg{i}"]) == "gap" else O.admm_solve
    extra = {} if str(g[f"sv_alg{i}"]) == "gap" else {"rho": 0.01}
    trace = []
    x, res, ps = solve(op, g[f"sv_y{i}"], int(g[f"sv_iters{i}"]), ref=g[f"sv_scene{i}"],
                       trace=trace, **kw, **extra)
    assert len(trace) == int(g[f"sv_nref{i}"])
    for j, (anc, pos) in enumerate(trace):
        assert np.array_equal(np.array(anc, dtype=np.int32), g[f"sv_anchors{i}_{j}"])
        assert np.array_equal(np.array(pos, dtype=np.int32), g[f"sv_positions{i}_{j}"])
    np.testing.assert_allclose(x, g[f"sv_out{i}"], atol=1e-10, rtol=0)
    np.testing.assert_allclose(res, g[f"sv_resid{i}"], rtol=1e-9)
    np.testing.assert_allclose(ps, g[f"sv_psnr{i}"], atol=1e-8)


def test_tv_denoise_bitwise():
    g = load_golden("tv")
    for i in range(int(g["tv_n"])):
        wgt, iters = g[f"tv_cfg{i}"]
        assert np.array_equal(O.tv_denoise(g[f"tv_x{i}"], float(wgt), int(iters)),
                              g[f"tv_out{i}"]), i


@pytest.mark.parametrize("i,alg", [(0, "gap"), (1, "admm")])
def test_tv_solves_match_reference_run(i, alg):
    g = load_golden("tv")
    op = O.Operator("cacti", masks=g[f"sv_masks{i}"])
    solve = O.gap_solve if alg == "gap" else O.admm_solve
    extra = {} if alg == "gap" else {"rho": 0.01}
    x, res, ps = solve(op, g[f"sv_y{i}"], 12, regularizer="tv", tv_weight=0.03, tv_iters=15,
                       ref=g[f"sv_scene{i}"], **extra)
    np.testing.assert_allclose(x, g[f"sv_out{i}"], atol=1e-12, rtol=0)
    np.testing.assert_allclose(res, g[f"sv_resid{i}"], rtol=1e-9)
    np.testing.assert_allclose(ps, g[f"sv_psnr{i}"], atol=1e-9)
