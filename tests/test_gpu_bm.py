"""Block matching and the pixel re-rank on device vs the
reference's golden vectors and the oracle (GPU only).

Distances reproduce numpy's summation order, so positions, their order and
the padding counts must be bit-identical; solves carry the same end-to-end
bar as the GLR path (identical refresh traces, max |x - x_ref| <= 1e-6,
final PSNR within 0.05 dB)."""

import ast

import numpy as np
import pytest

import glr_oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2301_03047_b200")


def _ex(anchors, p):
    anchors = [tuple(map(int, a)) for a in anchors]
    return G.ExemplarSet(anchors=anchors, tags=["uniform"] * len(anchors), patch_size=p)


def test_block_match_bitwise_vs_golden():
    g = load_golden("bm")
    for i in range(int(g["bm_n"])):
        p, k, win, st = (int(v) for v in g[f"bm_cfg{i}"])
        x = g[f"bm_x{i}"]
        cfg = G.MatchConfig(patch_size=p, group_size=k, bm_window=win, bm_stride=st,
                            mode="bm-uniform")
        groups = G.block_match(x, _ex(g[f"bm_anchors{i}"], p), cfg)
        assert np.array_equal(np.array([gr.positions for gr in groups], dtype=np.int32),
                              g[f"bm_pos{i}"]), i
        assert [gr.padded for gr in groups] == g[f"bm_pad{i}"].tolist(), i
        for gr in groups:
            assert np.array_equal(gr.matrix, O.gather_group(x, gr.positions, p))


@pytest.mark.parametrize("shape,p,k,win,st", [
    ((96, 96, 24), 8, 64, 20, 1),    # C2-like patch (m = 1536)
    ((80, 72, 3), 6, 32, 30, 1),     # 61x61 window: chunked selection (> 2048 candidates)
    ((64, 60, 16), 8, 64, 12, 2),
    ((50, 52, 1), 12, 16, 25, 3),
    ((20, 18, 2), 4, 300, 20, 1),    # whole image < K: padding
])
def test_block_match_vs_oracle(shape, p, k, win, st, rng):
    h, w, c = shape
    x = rng.random(shape)
    if c > 1:  # a few exact duplicates and flat areas: ties ordered row-major
        x[10:30, 10:30] = 0.25
        x[:, -8:] = x[:, :8]
    x = x.astype(np.float32).astype(np.float64)
    anchors = [(int(rng.integers(0, h - p + 1)), int(rng.integers(0, w - p + 1)))
               for _ in range(37)] + [(0, 0), (h - p, w - p), (12, 12)]
    cfg = G.MatchConfig(patch_size=p, group_size=k, bm_window=win, bm_stride=st,
                        mode="bm-uniform")
    groups = G.block_match(x, _ex(anchors, p), cfg)
    pos, pads = O.block_match(x, anchors, p, k, win, st)
    assert [gr.positions for gr in groups] == pos
    assert [gr.padded for gr in groups] == pads


def test_rerank_pixel_bitwise_vs_golden():
    g = load_golden("bm")
    for i in range(int(g["rr_n"])):
        p, k = (int(v) for v in g[f"rr_cfg{i}"])
        x = g[f"rr_x{i}"]
        gh, gv = G.sobel_gradients(x)
        edge = G.binarize_gradients(gh, gv, 0.2)
        ex = G.ExemplarSet(anchors=[tuple(a) for a in g[f"rr_anchors{i}"].tolist()],
                           tags=["corner"] * len(g[f"rr_anchors{i}"]), patch_size=p)
        plain = G.global_match(x, ex, G.MatchConfig(patch_size=p, group_size=k), edge)
        assert np.array_equal(np.array([gr.positions for gr in plain], dtype=np.int32),
                              g[f"rr_plain{i}"]), i
        rer = G.global_match(x, ex, G.MatchConfig(patch_size=p, group_size=k,
                                                  rerank_pixel=True), edge)
        assert np.array_equal(np.array([gr.positions for gr in rer], dtype=np.int32),
                              g[f"rr_pos{i}"]), i


@pytest.mark.parametrize("i", range(5))
def test_bm_solves_vs_reference_run(i):
    g = load_golden("bm")
    mc = ast.literal_eval(str(g[f"sv_mc{i}"]))
    alg = str(g[f"sv_alg{i}"])
    cfg = G.SolverConfig(regularizer=str(g[f"sv_reg{i}"]), algorithm=alg,
                         max_iters=int(g[f"sv_iters{i}"]), admm_rho=0.01,
                         match=G.MatchConfig(**mc))
    op = G.cacti_operator(g[f"sv_masks{i}"])
    trace = []
    solve = G.gap_solve if alg == "gap" else G.admm_solve
    x, rep = solve(op, g[f"sv_y{i}"], cfg, ref=g[f"sv_scene{i}"], trace=trace)
    assert len(trace) == int(g[f"sv_nref{i}"])
    for j, (anc, pos) in enumerate(trace):
        assert np.array_equal(np.array(anc, dtype=np.int32), g[f"sv_anchors{i}_{j}"]), j
        assert np.array_equal(np.array(pos, dtype=np.int32), g[f"sv_positions{i}_{j}"]), j
    assert np.abs(x - g[f"sv_out{i}"]).max() <= 1e-6
    assert abs(rep.rows[-1]["psnr_db"] - float(g[f"sv_psnr{i}"][-1])) <= 0.05


def test_block_match_solve_vs_oracle_larger(rng):
    """nlr-bm at a C1-like channel count, free-running vs the oracle."""
    h, w, c = 64, 72, 8
    yy, xx = np.mgrid[0:h, 0:w]
    base = 0.5 + 0.3 * np.sin(yy / 5.0) * np.cos(xx / 7.0) + 0.2 * rng.random((h, w))
    scene = np.stack([np.roll(base, t, axis=1) for t in range(c)], axis=2)
    scene = np.clip(scene, 0, 1).astype(np.float32).astype(np.float64)
    masks = G.bernoulli_masks(h, w, c, seed=5)
    op = G.cacti_operator(masks)
    y = O.masksum_forward(scene, masks)
    mc = G.MatchConfig(patch_size=8, group_size=32, exemplar_stride=6, bm_window=12)
    cfg = G.SolverConfig(regularizer="nlr-bm", max_iters=6, match=mc)
    trace = []
    x, _ = G.gap_solve(op, y, cfg, trace=trace)
    otrace = []
    xo, _, _ = O.gap_solve(O.Operator("cacti", masks=masks), y, 6, patch_size=8, group_size=32,
                           exemplar_stride=6, regularizer="nlr-bm", bm_window=12, trace=otrace)
    assert len(trace) == len(otrace)
    for (a, pz), (ao, po) in zip(trace, otrace):
        assert np.array_equal(np.asarray(a), np.asarray(ao))
        assert np.array_equal(np.asarray(pz), np.asarray(po))
    assert np.abs(x - xo).max() <= 1e-6


def _loop_xcorr(x, kernels):
    """The reference tests' kernel-index loop oracle (tests/test_matching.py:16-25
    of the reference, restated)."""
    h, w, c = x.shape
    n, p = kernels.shape[:2]
    out = np.zeros((h - p + 1, w - p + 1, n))
    for j in range(n):
        for dr in range(p):
            for dc in range(p):
                for ch in range(c):
                    out[:, :, j] += kernels[j, dr, dc, ch] * x[dr:dr + h - p + 1,
                                                              dc:dc + w - p + 1, ch]
    return out


@pytest.mark.parametrize("backend", ["direct", "im2col", "fft"])
def test_xcorr2_valid_batch_bitwise_vs_loop_oracle(backend, rng):
    x = rng.random((23, 19, 3))
    k = rng.standard_normal((5, 4, 4, 3))
    assert np.array_equal(G.xcorr2_valid_batch(x, k, backend=backend), _loop_xcorr(x, k))
    xb = (rng.random((16, 16, 2)) < 0.4).astype(np.float64)
    kb = (rng.random((3, 4, 4, 2)) < 0.4).astype(np.float64)
    assert np.array_equal(G.xcorr2_valid_batch(xb, kb, backend=backend), _loop_xcorr(xb, kb))
    d = np.zeros((1, 3, 3, 3))
    d[0, 0, 0, 0] = 1.0
    assert np.array_equal(G.xcorr2_valid_batch(x, d)[:, :, 0], x[:21, :17, 0])
