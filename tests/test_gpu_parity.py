"""CUDA path vs the oracle and the reference's golden vectors (GPU only).

Integer / decision stages (edges, corners, anchors, heat map, top-K) must be
bit-identical; fp64 stages carry the tolerance written in each test.
"""

import numpy as np
import pytest

import glr_oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2301_03047_b200")


def test_device_is_b200_class():
    from paper_2301_03047_b200 import _native as N
    import ctypes as C
    lib = N.load(require_gpu=True)
    sm, ma, mi = C.c_int(), C.c_int(), C.c_int()
    assert lib.glr_device_info(C.byref(sm), C.byref(ma), C.byref(mi)) == 0
    assert ma.value == 10


def test_edges_corners_anchors_bitwise_vs_golden():
    g = load_golden("edges")
    for i in range(int(g["n"])):
        x = g[f"x{i}"]
        gh, gv = G.sobel_gradients(x)
        assert np.array_equal(gh, g[f"gh{i}"]) and np.array_equal(gv, g[f"gv{i}"]), i
        em = G.binarize_gradients(gh, gv, 0.2)
        assert np.array_equal(np.stack(em.as_tuple()).astype(np.uint8), g[f"maps{i}"]), i
        corners = G.detect_corners(x, max_n=40, nms_radius=3)
        assert np.array_equal(np.array(corners, dtype=np.int32).reshape(-1, 2),
                              g[f"corners{i}"]), i
        ex = G.select_exemplars(corners, x.shape[:2], 6, uniform_interval=7)
        assert np.array_equal(np.array(ex.anchors, dtype=np.int32).reshape(-1, 2),
                              g[f"anchors{i}"]), i
        assert [t == "uniform" for t in ex.tags] == g[f"tags{i}"].astype(bool).tolist()


@pytest.mark.parametrize("shape,max_n,radius", [((300, 280, 3), 500, 4), ((1300, 1300, 1), 60, 4),
                                              ((97, 131, 2), 5000, 2), ((64, 64, 1), 10, 17),
                                              ((2048, 1100, 1), 3000, 4)])
def test_detect_corners_vs_oracle(shape, max_n, radius, rng):
    """Greedy NMS (edges.py:100-128): the batched kernel with its bitmap in
    shared memory, and in global memory for images beyond ~1.8 MPixel (the
    2048 x 1100 case, C5's path), vs the oracle."""
    h, w, c = shape
    base = rng.random((h // 4 + 2, w // 4 + 2, c))
    x = np.kron(base, np.ones((4, 4, 1)))[:h, :w] + 0.05 * rng.random((h, w, c))
    got = G.detect_corners(x, max_n=max_n, nms_radius=radius)
    want = O.detect_corners(x, max_n=max_n, nms_radius=radius)
    assert [tuple(p) for p in got] == [tuple(p) for p in want]


def test_corner_response_bitwise_vs_oracle(rng):
    from paper_2301_03047_b200 import _device as D, _native as N
    import torch
    for (h, w, c) in [(64, 48, 1), (40, 40, 8), (33, 65, 24), (20, 21, 9), (16, 16, 130)]:
        x = rng.random((h, w, c)).astype(np.float32).astype(np.float64)
        x_d = D.f64(x)
        resp = D.empty((h, w), torch.float64)
        ws = D.workspace().get("cr", N.query("glr_corner_workspace", h, w, c))
        N.call("glr_corner_response", x_d.data_ptr(), h, w, c, resp.data_ptr(),
               ws.data_ptr(), D.stream())
        want = O.corner_response(x)
        assert np.array_equal(D.host(resp), want), (h, w, c)
        # the engine's entry: the same response from stored Sobel gradients
        gh, gv = D.empty((h, w, c), torch.float64), D.empty((h, w, c), torch.float64)
        N.call("glr_sobel", x_d.data_ptr(), h, w, c, gh.data_ptr(), gv.data_ptr(), D.stream())
        resp2 = D.empty((h, w), torch.float64)
        N.call("glr_corner_response_grad", gh.data_ptr(), gv.data_ptr(), h, w, c,
               resp2.data_ptr(), ws.data_ptr(), D.stream())
        assert np.array_equal(D.host(resp2), want), (h, w, c)


def test_heat_topk_global_match_bitwise_vs_golden():
    g = load_golden("heat_topk")
    for i in range(int(g["n"])):
        h, w, c, p, n, k, sep = (int(v) for v in g[f"meta{i}"])
        maps = g[f"maps{i}"].astype(np.float64)
        edge = G.EdgeMaps(*maps)
        anchors = [tuple(a) for a in g[f"anchors{i}"].tolist()]
        ex = G.ExemplarSet(anchors=anchors, tags=["corner"] * n, patch_size=p)
        hm = G.similarity_heatmap(edge, ex)
        assert np.array_equal(hm.values, g[f"heat{i}"].astype(np.float64)), i
        cfg = G.MatchConfig(patch_size=p, group_size=k, min_separation=sep)
        groups = G.global_match(g[f"x{i}"], ex, cfg, edge)
        assert np.array_equal(np.array([q.positions for q in groups], dtype=np.int32),
                              g[f"positions{i}"]), i
        assert [q.padded for q in groups] == g[f"padded{i}"].tolist(), i
        for j, q in enumerate(groups):
            assert np.array_equal(q.matrix, g[f"matrix{i}"][j]), (i, j)


def test_topk_slices_bitwise_vs_golden():
    g = load_golden("topk_slices")
    for i in range(int(g["n"])):
        ar, ac, k, sep, pad = (int(v) for v in g[f"meta{i}"])
        pos, padded = G.top_k_positions(g[f"s{i}"], (ar, ac), k, sep)
        assert padded == pad, i
        assert np.array_equal(np.array(pos, dtype=np.int32), g[f"pos{i}"]), i


@pytest.mark.parametrize("seed", range(6))
def test_topk_random_vs_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(20):
        oh, ow = int(rng.integers(2, 60)), int(rng.integers(2, 60))
        s = rng.integers(0, int(rng.choice([2, 4, 30, 500])), size=(oh, ow)).astype(np.float64)
        anchor = (int(rng.integers(0, oh)), int(rng.integers(0, ow)))
        k = int(rng.integers(1, 65))
        sep = int(rng.integers(0, 4))
        assert G.top_k_positions(s, anchor, k, sep) == O.top_k_positions(s, anchor, k, sep)


def test_heat_map_vs_oracle_random_shapes(rng):
    for (h, w, c, p, n) in [(37, 29, 1, 8, 5), (30, 44, 2, 8, 9), (26, 26, 3, 5, 4),
                            (40, 50, 24, 8, 3), (34, 31, 16, 8, 300), (50, 52, 1, 12, 7),
                            (13, 300, 4, 8, 2), (9, 9, 1, 3, 2)]:
        maps = [(rng.random((h, w, c)) < 0.3).astype(np.uint8) for _ in range(4)]
        anchors = [(int(rng.integers(0, h - p + 1)), int(rng.integers(0, w - p + 1)))
                   for _ in range(n)]
        ex = G.ExemplarSet(anchors=anchors, tags=["corner"] * n, patch_size=p)
        got = G.similarity_heatmap(G.EdgeMaps(*[m.astype(float) for m in maps]), ex).values
        assert np.array_equal(got, O.similarity_heatmap(maps, anchors, p)), (h, w, c, p, n)


def test_wnnm_vs_golden_and_oracle():
    g = load_golden("wnnm")
    for i in range(int(g["n"])):
        m = g[f"m{i}"]
        sigma = float(g[f"sigma{i}"])
        out = G.wnnm_prox(m, G.WnnmParams(noise_sigma=sigma))
        np.testing.assert_allclose(out, g[f"out{i}"], atol=1e-9, rtol=0)
        uw = G.wnnm_prox(m, G.WnnmParams(uniform_weight=0.3))
        np.testing.assert_allclose(uw, g[f"uw{i}"], atol=1e-9, rtol=0)
    pos = [[tuple(p) for p in grp] for grp in g["reg_pos"].tolist()]
    groups = [G.gather_group(g["reg_x"], q, 4) for q in pos]
    z = G.glr_regularize(g["reg_x"], groups, G.WnnmParams(noise_sigma=0.05))
    np.testing.assert_allclose(z, g["reg_z"], atol=1e-9, rtol=0)


def test_wnnm_acceptance4_style(rng):
    """acceptance #4: 100 random matrices vs the SVD oracle, zero-noise identity."""
    worst = 0.0
    for _ in range(100):
        m = rng.standard_normal((int(rng.integers(2, 65)), int(rng.integers(2, 65))))
        sigma = float(rng.uniform(0.01, 0.8))
        out = G.wnnm_prox(m, G.WnnmParams(noise_sigma=sigma))
        worst = max(worst, float(np.abs(out - O.wnnm_prox(m, sigma)).max()))
        ident = G.wnnm_prox(m, G.WnnmParams(noise_sigma=0.0))
        assert np.abs(ident - m).max() < 1e-10
    assert worst < 1e-8, worst


def test_operators_vs_golden():
    g = load_golden("operators")
    op = G.cacti_operator(g["cacti_masks"])
    np.testing.assert_allclose(op.forward(g["cacti_x"]), g["cacti_y"], atol=1e-13, rtol=0)
    np.testing.assert_allclose(op.adjoint(g["cacti_y"]), g["cacti_adj"], atol=1e-13, rtol=0)
    op = G.msfa_operator(g["msfa_masks"])
    np.testing.assert_allclose(op.forward(g["msfa_x"]), g["msfa_y"], atol=1e-13, rtol=0)
    op = G.fourier_operator(g["four_mask"])
    np.testing.assert_allclose(op.forward(g["four_x"]), g["four_y"], atol=1e-13, rtol=0)
    np.testing.assert_allclose(op.adjoint(g["four_y"]), g["four_adj"], atol=1e-13, rtol=0)


@pytest.mark.parametrize("shape", [(16, 16), (24, 24), (12, 20), (64, 32)])
def test_fourier_adjoint_identity_and_oracle(shape, rng):
    h, w = shape
    mask = (rng.random((h, w)) < 0.4).astype(float)
    for ch in (1, 2):
        op = G.fourier_operator(mask, channels=ch)
        oop = O.Operator("fourier", mask=mask, channels=ch)
        x = rng.standard_normal((h, w, ch))
        y = rng.standard_normal((h, w)) + 1j * rng.standard_normal((h, w))
        np.testing.assert_allclose(op.forward(x), oop.forward(x), atol=1e-12)
        np.testing.assert_allclose(op.adjoint(y), oop.adjoint(y), atol=1e-12)
        lhs = np.vdot(op.forward(x), y).real
        rhs = np.vdot(x, op.adjoint(y)).real
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))


@pytest.mark.parametrize("i", [0, 1, 2])
def test_gap_solve_vs_reference_run(i):
    """L3 free-running end-to-end parity against a recorded reference run."""
    g = load_golden("solves")
    kind = str(g[f"kind{i}"])
    p, k, mc, stride, iters = (int(v) for v in g[f"mc{i}"])
    masks = g[f"masks{i}"]
    op = G.cacti_operator(masks) if kind == "cacti" else G.msfa_operator(masks)
    cfg = G.SolverConfig(regularizer="glr", max_iters=iters,
                         match=G.MatchConfig(patch_size=p, group_size=k, max_corners=mc,
                                             exemplar_stride=stride))
    trace = []
    x, rep = G.gap_solve(op, g[f"y{i}"], cfg, ref=g[f"scene{i}"], trace=trace)
    assert len(trace) == int(g[f"nref{i}"])
    for j, (anc, pos) in enumerate(trace):
        assert np.array_equal(np.array(anc, dtype=np.int32), g[f"anchors{i}_{j}"]), j
        assert np.array_equal(np.array(pos, dtype=np.int32), g[f"positions{i}_{j}"]), j
    assert np.abs(x - g[f"out{i}"]).max() <= 1e-6
    ps = [r["psnr_db"] for r in rep.rows]
    assert abs(ps[-1] - float(g[f"psnr{i}"][-1])) <= 0.05
    # residuals of a noiseless CACTI/MSFA projection sit at rounding level:
    # compare relative to ||y||
    ynorm = float(np.linalg.norm(g[f"y{i}"]))
    np.testing.assert_allclose([r["residual"] for r in rep.rows], g[f"resid{i}"], rtol=1e-6,
                               atol=1e-9 * ynorm)


def test_gap_solve_deterministic(rng):
    scene = rng.random((40, 44, 4)).astype(np.float32).astype(np.float64)
    op = G.cacti_operator(G.bernoulli_masks(40, 44, 4, seed=2))
    y = op.forward(scene)
    cfg = G.SolverConfig(max_iters=7, match=G.MatchConfig(patch_size=4, group_size=16,
                                                          max_corners=40))
    a, ra = G.gap_solve(op, y, cfg)
    b, rb = G.gap_solve(op, y, cfg)
    assert np.array_equal(a, b)
    assert [r["residual"] for r in ra.rows] == [r["residual"] for r in rb.rows]


def test_admm_solve_vs_reference_run():
    """ADMM-GLR (solvers.py:311-341) on device vs a recorded reference run:
    identical refresh traces, max |x - x_ref| <= 1e-6, PSNR within 0.05 dB."""
    g = load_golden("admm")
    op = G.cacti_operator(g["masks"])
    cfg = G.SolverConfig(algorithm="admm", max_iters=7, admm_rho=0.01,
                         match=G.MatchConfig(patch_size=4, group_size=8, max_corners=24,
                                             exemplar_stride=4))
    x, rep = G.solve(op, g["y"], cfg, ref=g["scene"])
    assert np.abs(x - g["out"]).max() <= 1e-6
    assert abs(rep.rows[-1]["psnr_db"] - float(g["psnr"][-1])) <= 0.05
    ynorm = float(np.linalg.norm(g["y"]))
    np.testing.assert_allclose([r["residual"] for r in rep.rows], g["resid"], rtol=1e-6,
                               atol=1e-9 * ynorm)


def test_interp_init_vs_golden():
    """init="interp" (solvers.py:237-254) on device: the MSFA Gaussian
    normalised convolution is bit-identical to the reference (scipy), CACTI
    adjoint / max(gram, 1e-12) within 1e-13."""
    from paper_2301_03047_b200.engine import DeviceOperator
    import torch
    g = load_golden("interp")
    for kind, build, atol in (("msfa", G.msfa_operator, 0.0), ("cacti", G.cacti_operator, 1e-13)):
        op = build(g[f"{kind}_masks"])
        dop = DeviceOperator(op)
        x = torch.empty(dop.shape, dtype=torch.float64, device="cuda")
        dop.init_x(dop.upload_y(g[f"{kind}_y"]), x, "interp")
        out = x.cpu().numpy()
        if atol == 0.0:
            assert np.array_equal(out, g[f"{kind}_init"]), kind
        else:
            np.testing.assert_allclose(out, g[f"{kind}_init"], atol=atol, rtol=0)


def test_gap_solve_interp_init_vs_reference_run():
    g = load_golden("interp")
    op = G.msfa_operator(g["solve_masks"])
    cfg = G.SolverConfig(regularizer="glr", max_iters=6, init="interp",
                         match=G.MatchConfig(patch_size=4, group_size=8, max_corners=24,
                                             exemplar_stride=4))
    trace = []
    x, rep = G.gap_solve(op, g["solve_y"], cfg, ref=g["solve_scene"], trace=trace)
    assert len(trace) == int(g["solve_nref"])
    for j, (anc, pos) in enumerate(trace):
        assert np.array_equal(np.array(anc, dtype=np.int32), g[f"solve_anchors_{j}"]), j
        assert np.array_equal(np.array(pos, dtype=np.int32), g[f"solve_positions_{j}"]), j
    assert np.abs(x - g["solve_out"]).max() <= 1e-6
    assert abs(rep.rows[-1]["psnr_db"] - float(g["solve_psnr"][-1])) <= 0.05


def test_vcache_remap_reindexes_kept_positions(rng):
    """glr_vcache_remap: a group keeping its anchor gets its cached V^T with the
    coordinates permuted so every kept patch position keeps its coordinate
    (t-th occurrence to t-th occurrence), the rest in order: an orthogonal
    row permutation of V."""
    import torch
    from paper_2301_03047_b200 import _device as D, _native as N
    H, W, K = 40, 50, 12
    old_anc = np.array([[3, 4], [10, 20], [30, 5]], np.int32)
    new_anc = np.array([[10, 20], [7, 7], [3, 4]], np.int32)
    old_pos = rng.integers(0, 30, (3, K, 2)).astype(np.int32)
    old_pos[0, 5] = old_pos[0, 2]                      # a duplicated position
    new_pos = rng.integers(0, 30, (3, K, 2)).astype(np.int32)
    new_pos[0, [0, 3, 7]] = old_pos[1, [4, 0, 9]]      # kept by the second old group
    new_pos[2, [1, 2, 6]] = old_pos[0, [2, 5, 11]]     # includes the duplicate twice
    vc_old = np.zeros((3, 64, 64))
    for g in range(3):
        q, _ = np.linalg.qr(rng.standard_normal((64, 64)))
        vc_old[g] = q
    vo, vn = D.f64(vc_old), D.f64(np.zeros_like(vc_old))
    flags = D.zeros((3,), torch.uint8)
    amap = D.empty((H * W,), torch.int32).fill_(-1)
    oa, na, op, npd = D.i32(old_anc), D.i32(new_anc), D.i32(old_pos), D.i32(new_pos)
    N.call("glr_vcache_remap", oa.data_ptr(), 0, 3, na.data_ptr(), 0, 3, H, W, vo.data_ptr(),
           vn.data_ptr(), flags.data_ptr(), amap.data_ptr(), op.data_ptr(), npd.data_ptr(), K,
           D.stream())
    got, fl = D.host(vn), D.host(flags)
    assert fl.tolist() == [1, 0, 1]
    assert (D.host(amap) == -1).all()
    for g_new, g_old in ((0, 1), (2, 0)):
        perm = []
        for j in range(64):
            hits = [i for i in range(64) if np.array_equal(got[g_new][:, j], vc_old[g_old][:, i])]
            assert len(hits) == 1
            perm.append(hits[0])
        assert sorted(perm) == list(range(64)) and perm[K:] == list(range(K, 64))
        key = lambda p: (int(p[0]), int(p[1]))  # noqa: E731
        seen = {}
        for j in range(K):
            v = key(new_pos[g_new, j])
            t = seen.get(v, 0)
            seen[v] = t + 1
            occ = [i for i in range(K) if key(old_pos[g_old, i]) == v]
            if t < len(occ):
                assert perm[j] == occ[t], (g_new, j)


@pytest.mark.parametrize("cap", [None, 8])
def test_fused_heat_topk_matches_dense(cap, rng):
    """glr_heat_topk (candidate lists from the GEMM epilogue, low-memory mode)
    gives the same positions as the dense heat map + glr_topk; cap = 8 forces
    every exemplar through the overflow fallback (dense path)."""
    from paper_2301_03047_b200 import _device as D
    from paper_2301_03047_b200.engine import GlrEngine
    h, w, c = 150, 170, 4
    base = rng.random((h // 6 + 2, w // 6 + 2, c))
    x = np.kron(base, np.ones((6, 6, 1)))[:h, :w] + 0.1 * rng.random((h, w, c))
    mc = G.MatchConfig(patch_size=8, group_size=16, max_corners=60, exemplar_stride=6)
    xd = D.f64(x)
    dense = GlrEngine((h, w, c), mc)
    dense.refresh(xd)
    a0, p0, d0 = dense.positions_host()
    fused = GlrEngine((h, w, c), mc, low_memory_match=True)
    if cap is not None:
        fused.cand_cap = cap
    fused.refresh(xd)
    a1, p1, d1 = fused.positions_host()
    assert np.array_equal(a0, a1) and np.array_equal(p0, p1) and np.array_equal(d0, d1)
    if cap is not None:
        assert fused.n_fallback == len(a1)


def test_ssim_on_device_vs_reference():
    """f3: glr_ssim (device, clip(x, 0, peak) vs ref) against the reference's
    metrics.ssim values (tests/golden/metrics.npz) within 1e-10."""
    import torch
    from paper_2301_03047_b200 import _device as D, _native as N
    g = load_golden("metrics")
    ax = np.arange(11) - 5.0
    taps = np.exp(-(ax ** 2) / (2.0 * 1.5 ** 2))
    taps = np.ascontiguousarray(taps / taps.sum())
    for i in range(int(g["n"])):
        a, b = g[f"a{i}"], g[f"b{i}"]
        h, w, c = a.shape
        out = D.zeros((1,), torch.float64)
        ws = D.empty((N.query("glr_ssim_workspace", h, w, c),), torch.uint8)
        bd, ad = D.f64(b), D.f64(a)
        N.call("glr_ssim", bd.data_ptr(), ad.data_ptr(), h, w, c, 1.0, 1,
               taps.ctypes.data_as(N.C.POINTER(N.C.c_double)), 11, out.data_ptr(),
               ws.data_ptr(), D.stream())
        val = float(D.host(out)[0]) / (c * (h - 10) * (w - 10))
        assert abs(val - float(g[f"ssim{i}"])) <= 1e-10, i


def test_report_ssim_matches_host_formula():
    """gap_solve with ref: per-iteration SSIM from the device equals the
    oracle's SSIM of the reported iterate within 1e-10."""
    g = load_golden("solves")
    op = G.cacti_operator(g["masks0"])
    cfg = G.SolverConfig(regularizer="glr", max_iters=3,
                         match=G.MatchConfig(patch_size=4, group_size=8, max_corners=24,
                                             exemplar_stride=4))
    x, rep = G.gap_solve(op, g["y0"], cfg, ref=g["scene0"])
    assert abs(rep.rows[-1]["ssim"] - O.ssim(g["scene0"], x, 1.0)) <= 1e-10
    assert all(0.0 < r["ssim"] <= 1.0 for r in rep.rows)


def test_binary_mask_upload_path_is_bitwise_identical(rng):
    """Binary masks travel as their 1-byte copy (gram formed on device); the
    solve must not change bit for bit against the float64 upload."""
    h, w, t = 40, 36, 6
    scene = rng.random((h, w, t)).astype(np.float32).astype(np.float64)
    masks = G.bernoulli_masks(h, w, t, seed=7)
    op = G.cacti_operator(masks)
    assert "masks_u8" in op.meta
    y = op.forward(scene)
    cfg = G.SolverConfig(max_iters=6, match=G.MatchConfig(patch_size=4, group_size=16,
                                                          max_corners=30))
    a, _ = G.gap_solve(op, y, cfg)
    op_f64 = G.cacti_operator(masks)
    op_f64.meta.pop("masks_u8")
    b, _ = G.gap_solve(op_f64, y, cfg)
    assert np.array_equal(a, b)
    op_swapped = G.cacti_operator(masks)
    op_swapped.meta["masks"] = masks.copy()  # replaced: the u8 copy must not be used
    c, _ = G.gap_solve(op_swapped, y, cfg)
    assert np.array_equal(a, c)


@pytest.mark.parametrize("p,c,k,amp", [(8, 24, 64, 1.0), (4, 3, 16, 1.0), (8, 1, 64, 1.0),
                                       (5, 2, 37, 1.0), (6, 4, 64, 255.0), (8, 2, 64, 0.01),
                                       (4, 2, 64, 0.0)])
def test_wnnm_scatter_image_groups_vs_oracle(p, c, k, amp, rng):
    """glr_wnnm_scatter (image groups gathered at their positions, the solve's
    path: Gram -> Jacobi -> tensor-core split-integer apply -> int64 scatter)
    against the SVD oracle + an fp64 scatter (lowrank.py:68-87)."""
    from paper_2301_03047_b200 import _device as D, _native as N
    from paper_2301_03047_b200.lowrank import frac_bits_for
    t = D.torch()
    h, w, n, sigma = 37, 41, 9, 0.05 * amp
    x = (rng.random((h, w, c)) * 1.5 - 0.25) * amp
    x[rng.random((h, w, c)) < 0.05] = 0.0  # exact zeros and a flat region
    x[:8, :8] = 0.5 * amp
    pos = np.stack([rng.integers(0, h - p + 1, (n, k)), rng.integers(0, w - p + 1, (n, k))],
                   axis=2).astype(np.int32)
    pos[0, :] = 0  # one group of identical (flat) patches
    frac = frac_bits_for(amp * 1.5)
    x_d, pos_d = D.f64(x), D.i32(pos)
    acc = D.zeros((h, w, c), t.int64)
    ws = D.empty((N.query("glr_wnnm_workspace", n, k),), t.uint8)
    N.call("glr_wnnm_scatter", x_d.data_ptr(), h, w, c, p, pos_d.data_ptr(), n, None, k, sigma,
           2.0 * np.sqrt(2.0), 1e-16, frac, acc.data_ptr(), None, 0, None, ws.data_ptr(),
           ws.numel(), D.stream())
    got = D.host(acc).astype(np.float64) * 2.0 ** -frac
    ref = np.zeros((h, w, c))
    for g in range(n):
        cols = [x[r:r + p, q:q + p, :].ravel() for r, q in pos[g]]
        den = O.wnnm_prox(np.stack(cols, axis=1), sigma)
        for j, (r, q) in enumerate(pos[g]):
            ref[r:r + p, q:q + p, :] += den[:, j].reshape(p, p, c)
    # per term: 2^-frac rounding of the numerator + the WNNM agreement bar
    cnt = np.zeros((h, w))
    for g in range(n):
        for r, q in pos[g]:
            cnt[r:r + p, q:q + p] += 1
    tol = cnt[..., None] * (2.0 ** -frac + 1e-9 * amp)
    err = np.abs(got - ref)
    assert (err <= tol + 1e-15).all(), float((err - tol).max())


@pytest.mark.parametrize("sigmas", [(0.5, 0.45, 0.4), (0.1, 0.08, 0.06), (0.02, 0.015, 0.01),
                                    (0.002, 0.0015, 0.001)])
def test_wnnm_scatter_warm_start_across_kept_ranks(sigmas, rng):
    """The warm path of glr_wnnm_scatter (cached eigenvectors, zero-shrinkage
    exemption with its gap rule, partial sweeps, first-order finish) against
    the SVD oracle on a smooth image + noise, at noise levels that keep from
    3 to all 64 of the components (oracle ranks: ~3, ~8, ~44, ~63), with the
    iterate perturbed between calls as in a solve (lowrank.py:46-65 per group, :68-87 aggregated)."""
    from paper_2301_03047_b200 import _device as D, _native as N
    from paper_2301_03047_b200.lowrank import frac_bits_for
    t = D.torch()
    h, w, c, p, k, n = 48, 52, 2, 8, 64, 24
    yy, xx = np.mgrid[0:h, 0:w]
    base = 0.5 + 0.3 * np.sin(yy / 5.0)[..., None] * np.cos(xx / 7.0)[..., None] \
        + 0.1 * np.stack([np.sin(xx / 3.0), np.cos(yy / 4.0)], axis=2)
    x = base + 0.02 * rng.standard_normal((h, w, c))
    pos = np.stack([rng.integers(0, h - p + 1, (n, k)), rng.integers(0, w - p + 1, (n, k))],
                   axis=2).astype(np.int32)
    frac = frac_bits_for(1.5)
    pos_d = D.i32(pos)
    vc = D.zeros((n, 64, 64), t.float64)
    ws = D.empty((N.query("glr_wnnm_workspace", n, k),), t.uint8)
    cnt = np.zeros((h, w))
    for g in range(n):
        for r, q in pos[g]:
            cnt[r:r + p, q:q + p] += 1
    for step, sigma in enumerate(sigmas):
        if step:
            x = x + 2e-3 * rng.standard_normal((h, w, c))  # the iterate moves between calls
        acc = D.zeros((h, w, c), t.int64)
        x_d = D.f64(x)
        N.call("glr_wnnm_scatter", x_d.data_ptr(), h, w, c, p, pos_d.data_ptr(), n, None, k,
               float(sigma), 2.0 * np.sqrt(2.0), 1e-16, frac, acc.data_ptr(), vc.data_ptr(),
               1 if step else 0, None, ws.data_ptr(), ws.numel(), D.stream())
        got = D.host(acc).astype(np.float64) * 2.0 ** -frac
        ref = np.zeros((h, w, c))
        for g in range(n):
            m = np.stack([x[r:r + p, q:q + p, :].ravel() for r, q in pos[g]], axis=1)
            den = O.wnnm_prox(m, sigma)
            for j, (r, q) in enumerate(pos[g]):
                ref[r:r + p, q:q + p, :] += den[:, j].reshape(p, p, c)
        tol = cnt[..., None] * (2.0 ** -frac + 1e-9)
        err = np.abs(got - ref)
        assert (err <= tol + 1e-15).all(), (step, sigma, float((err - tol).max()))
