"""Parity at the BASELINE.json configurations at FULL size (GPU).

* C1 (256x256x8, 30 iterations): every refresh's anchors + positions, the
  residual trace and the final x against a golden produced by the
  UNMODIFIED reference gap_solve (tests/golden/make_golden.py gen_configs).
* C3 (512x512 complex, 40 it) and C4 (512x512x16, 30 it): the first two
  refreshes bitwise and the iterate after 10 free-running iterations against
  reference goldens (<= 1e-6 max-abs, PSNR within 0.05 dB).
* C2 (1024x1024x24, the headline): the first refresh's anchors against the
  oracle, 32 sampled exemplars' heat rows and ordered top-K lists bitwise
  against the oracle, then one full WNNM + aggregation + GAP iteration against
  the oracle at the device's positions (<= 1e-6).
* C5 (2048x2048x1 stage sweep): sampled heat rows and top-K at P = 8 and 12.

Goldens store x as float32 where the full array is kept; the tolerance adds
the float32 rounding of the stored value (|x| * 2^-24).
"""

import numpy as np
import pytest

import glr_oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2301_03047_b200")
from paper_2301_03047_b200 import _device as D, _native as N, workloads  # noqa: E402
from paper_2301_03047_b200.solvers import GapRunner  # noqa: E402


def _oracle_op(wl):
    if wl.kind == "fourier":
        return O.Operator("fourier", mask=wl.masks, channels=2)
    return O.Operator(wl.kind, masks=wl.masks)


def _run(wl, capture_after=None):
    """Device solve of the workload; returns (final x host, residuals,
    trace, x after `capture_after` iterations)."""
    cfg = wl.solver_config()
    runner = GapRunner(workloads.operator_for(wl), cfg)
    y_d = runner.dop.upload_y(wl.y)
    trace, cap = [], {}

    def on_iter(it, x):
        if capture_after is not None and it == capture_after - 1:
            cap["x"] = D.host(x)

    x = runner.run(y_d, trace=trace, on_iter=on_iter)
    res = np.sqrt(D.host(runner.resid_sq))
    return D.host(x), res, trace, cap.get("x")


def _check_traces(trace, gold, nref):
    assert len(trace) >= nref
    for j in range(nref):
        a, p = trace[j]
        ga = gold[f"anchors_{j}"].astype(np.int32)
        gp = gold[f"positions_{j}"].astype(np.int32)
        assert np.array_equal(np.asarray(a, dtype=np.int32), ga), f"anchors differ at refresh {j}"
        pa = np.asarray(p, dtype=np.int32)
        if not np.array_equal(pa, gp):
            bad = np.nonzero((pa != gp).any(axis=(1, 2)))[0]
            raise AssertionError(f"refresh {j}: {bad.size} of {len(gp)} groups differ "
                                 f"(first {bad[:5].tolist()})")


def _psnr(ref, x):
    return O.psnr(ref, np.clip(x, 0.0, 1.0), 1.0)


def test_c1_full_solve_vs_reference_golden():
    gold = load_golden("config_C1")
    wl = workloads.make("C1")
    assert wl.max_iters == int(gold["iters"]) == 30
    x, res, trace, _ = _run(wl)
    nref = int(gold["nref"])
    assert len(trace) == nref == 6
    _check_traces(trace, gold, nref)
    out = np.clip(x, 0.0, 1.0)
    gx = gold["x"].astype(np.float64)
    err = np.abs(out - gx) - np.abs(gx) * 2.0 ** -24
    assert err.max() <= 1e-6, err.max()
    np.testing.assert_allclose(res, gold["resid"], rtol=1e-6)
    assert abs(_psnr(wl.scene, out) - float(gold["psnr"])) <= 0.05


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_first_refreshes_and_10_iterations(name):
    gold = load_golden(f"config_{name}")
    wl = workloads.make(name)
    assert int(gold["iters"]) == 10
    _, res, trace, x10 = _run(wl, capture_after=10)
    _check_traces(trace, gold, 2)
    # C3's unclipped complex projection makes the data term exact: its
    # residuals sit at rounding level, hence the ||y||-relative floor
    ynorm = float(np.linalg.norm(np.abs(wl.y).ravel()))
    np.testing.assert_allclose(res[:10], gold["resid"], rtol=1e-6, atol=1e-12 * ynorm)
    if name == "C3":
        assert len(trace[0][0]) == 2048  # the config's exemplar count
        gx = gold["x"].astype(np.float64)
        err = np.abs(x10 - gx) - np.abs(gx) * 2.0 ** -24
        assert err.max() <= 1e-6, err.max()
    else:
        idx = gold["sample_idx"]
        assert np.abs(x10.ravel()[idx] - gold["sample"]).max() <= 1e-6
        n = x10.size
        assert abs(x10.sum() - float(gold["x_sum"])) <= 1e-6 * n
        assert abs((x10 * x10).sum() - float(gold["x_sumsq"])) <= 4e-6 * n
    assert abs(_psnr(wl.scene, x10) - float(gold["psnr"])) <= 0.05


# ---------------------------------------------------------------------------
# C2 / C5: sampled exemplars against the oracle

def _heat_topk_rows(eng, anchors):
    """Heat rows + top-K of `anchors` on the engine's edge stack (device)."""
    t = D.torch()
    h, w, c = eng.shape
    n = len(anchors)
    anc = D.i32(np.asarray(anchors, dtype=np.int32).reshape(n, 2))
    heat = D.empty((n, eng.stride), t.int16)
    ws = D.empty((N.query("glr_heat_workspace", c, eng.p, n),), t.uint8)
    s = D.stream()
    N.call("glr_heat_map", eng.stack.data_ptr(), h, w, c, eng.p, eng.expand, anc.data_ptr(), n,
           None, heat.data_ptr(), ws.data_ptr(), ws.numel(), s)
    pos = D.empty((n, eng.k, 2), t.int32)
    pad = D.empty((n,), t.int32)
    N.call("glr_topk", heat.data_ptr(), n, None, eng.oh, eng.ow, eng.max_score, anc.data_ptr(),
           eng.k, eng.mc.sep, pos.data_ptr(), pad.data_ptr(), None, 0, s)
    rows = D.host(heat)[:, :eng.oh * eng.ow].view(np.uint16).astype(np.int64)
    return rows.reshape(n, eng.oh, eng.ow), D.host(pos), D.host(pad)


def _edge_stack(eng, x_d):
    h, w, c = eng.shape
    N.call("glr_sobel", x_d.data_ptr(), h, w, c, eng.gh.data_ptr(), eng.gv.data_ptr(), D.stream())
    N.call("glr_edge_stack", eng.gh.data_ptr(), eng.gv.data_ptr(), h, w, c,
           float(eng.mc.edge_threshold), 1, eng.expand, None, eng.stack.data_ptr(),
           eng.ws_edge.data_ptr(), D.stream())


def test_c2_sampled_exemplars_and_one_iteration():
    wl = workloads.make("C2")
    mc = wl.match
    cfg = G.SolverConfig(max_iters=wl.max_iters, match=mc)
    runner = GapRunner(workloads.operator_for(wl), cfg)
    eng, dop = runner.eng, runner.dop
    y_d = dop.upload_y(wl.y)
    x_d = runner.xa
    dop.init_x(y_d, x_d, "adjoint")
    xh = D.host(x_d)
    n = eng.refresh(x_d)
    anchors, positions, padded = eng.positions_host()
    # exemplar detection at full size (A3/A4) vs the oracle
    o_anchors = O.build_exemplars(xh, mc.patch_size, mc.max_corners, mc.nms, mc.corner_quality,
                                  mc.exemplar_stride)
    assert n == len(o_anchors) == 4097
    assert np.array_equal(anchors, np.asarray(o_anchors, dtype=np.int32))
    # 32 sampled exemplars: heat rows and ordered top-K lists bitwise
    rng = np.random.default_rng(2024)
    idx = np.unique(np.concatenate([[0, n - 1], rng.choice(n, 30, replace=False)]))
    sub = [tuple(anchors[i]) for i in idx]
    rows, pos_s, pad_s = _heat_topk_rows(eng, sub)
    maps = O.binarize_gradients(*O.sobel_gradients(xh), mc.edge_threshold)
    heat_o = O.similarity_heatmap(maps, sub, mc.patch_size)
    for j in range(len(sub)):
        assert np.array_equal(rows[j], heat_o[:, :, j]), f"heat row of exemplar {idx[j]}"
    pos_o, pad_o = O.match_positions(heat_o, sub, mc.group_size, mc.sep)
    assert np.array_equal(positions[idx], np.asarray(pos_o, dtype=np.int32))
    assert np.array_equal(padded[idx], np.asarray(pad_o))
    assert np.array_equal(pos_s, positions[idx])
    # one full iteration (WNNM + aggregation + GAP) at these positions
    sigma = cfg.sigma_at(0)
    assert eng.regularize(x_d, sigma)
    x1_d = runner.xb
    dop.gap_update(eng.acc, eng.cnt, eng.frac, x_d, y_d, -0.5, 1.5, x1_d,
                   runner.resid_sq[0:1], eng.gap_ws)
    eng.consumed()
    x1 = D.host(x1_d)
    op = _oracle_op(wl)
    z = O.glr_regularize(xh, [list(map(tuple, p)) for p in positions], mc.patch_size, sigma)
    xo = np.clip(z + op.adjoint(O.safe_div(wl.y - op.forward(z), op.gram)), -0.5, 1.5)
    assert np.abs(x1 - xo).max() <= 1e-6
    # the numerator was consumed (read-and-clear): zero for the next iteration
    assert int(eng.acc.abs().max().item()) == 0


@pytest.mark.parametrize("p", [8, 12])
def test_c5_sampled_heat_rows_and_topk(p):
    wl = workloads.make("C5")
    mc = G.MatchConfig(patch_size=p, group_size=64, max_corners=64, exemplar_stride=683)
    eng = G.solvers.GlrEngine(wl.shape, mc)
    x_d = D.f64(wl.scene)
    _edge_stack(eng, x_d)
    h, w, _ = wl.shape
    rng = np.random.default_rng(55 + p)
    sub = [(0, 0), (h - p, w - p)] + [(int(rng.integers(0, h - p + 1)),
                                        int(rng.integers(0, w - p + 1))) for _ in range(10)]
    rows, pos, pad = _heat_topk_rows(eng, sub)
    maps = O.binarize_gradients(*O.sobel_gradients(wl.scene), mc.edge_threshold)
    heat_o = O.similarity_heatmap(maps, sub, p)
    for j in range(len(sub)):
        assert np.array_equal(rows[j], heat_o[:, :, j]), f"heat row {j}"
    pos_o, pad_o = O.match_positions(heat_o, sub, 64, mc.sep)
    assert np.array_equal(pos, np.asarray(pos_o, dtype=np.int32))
    assert np.array_equal(pad, np.asarray(pad_o))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_midsize_cacti_other_seeds_vs_oracle(seed):
    """The C1 generator at 112 x 96 x 8 with other seeds, 12 iterations (three
    refreshes, so the eigenvector carry-over, the warm starts with partial
    sweeps and the first-order finish all run) against the oracle's solve:
    every refresh's anchors and positions bit-identical, x within 1e-6."""
    h, w, t = 112, 96, 8
    rng = np.random.default_rng(1000 + seed)
    scene = workloads.cacti_scene(h, w, t, seed)
    masks = G.bernoulli_masks(h, w, t, seed=seed + 7)
    y = (masks * scene).sum(axis=2, keepdims=True) + rng.normal(0.0, 0.01, (h, w, 1))
    mc = G.MatchConfig(patch_size=8, group_size=64, max_corners=96, exemplar_stride=16)
    cfg = G.SolverConfig(max_iters=12, match=mc)
    trace = []
    x, rep = G.gap_solve(G.cacti_operator(masks), y, cfg, trace=trace)
    otrace = []
    xo, res_o, _ = O.gap_solve(O.Operator("cacti", masks=masks), y, 12, patch_size=8,
                               group_size=64, max_corners=96, exemplar_stride=16, trace=otrace)
    assert len(trace) == len(otrace) == 3
    for j, ((a, p), (ao, po)) in enumerate(zip(trace, otrace)):
        assert np.array_equal(np.asarray(a), np.asarray(ao)), f"anchors differ at refresh {j}"
        assert np.array_equal(np.asarray(p), np.asarray(po)), f"positions differ at refresh {j}"
    assert np.abs(x - xo).max() <= 1e-6
    np.testing.assert_allclose([r["residual"] for r in rep.rows], res_o, rtol=1e-6)
