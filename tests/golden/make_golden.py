"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference lives at /root/reference and does
not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small .npz files next to this script. Every array is produced by the
reference's own public functions (glr.*), so the oracle (oracle/glr_oracle.py)
and the CUDA path are pinned to the reference, not to each other.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = os.environ.get("GLR_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)

import glr  # noqa: E402  (the reference)
import glr.solvers as ref_solvers  # noqa: E402
from glr.edges import EdgeMaps, ExemplarSet  # noqa: E402

OUT = Path(__file__).resolve().parent


def f32(a):
    """Inputs are rounded once to fp32 and fed as float64 to both sides."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def blob_texture(rng, h, w, c):
    yy, xx = np.mgrid[0:h, 0:w]
    base = np.zeros((h, w))
    for _ in range(6):
        cy, cx = rng.uniform(0, h), rng.uniform(0, w)
        sy, sx = rng.uniform(2, h / 4), rng.uniform(2, w / 4)
        base += rng.uniform(0.2, 1.0) * np.exp(-((yy - cy) / sy) ** 2 - ((xx - cx) / sx) ** 2)
    tex = rng.random((8, 8))
    base += 0.3 * np.tile(tex, (h // 8 + 1, w // 8 + 1))[:h, :w]
    x = np.stack([np.roll(base, k, axis=1) for k in range(c)], axis=2)
    x = (x - x.min()) / (x.max() - x.min())
    return f32(x)


def random_maps(rng, h, w, c, density):
    m = lambda: (rng.random((h, w, c)) < density).astype(np.float64)  # noqa: E731
    hp, vp = m(), m()
    return EdgeMaps(h_pos=hp, h_neg=m() * (1 - hp), v_pos=vp, v_neg=m() * (1 - vp))


def gen_edges():
    rng = np.random.default_rng(101)
    cases = {}
    shapes = [(24, 31, 1), (32, 32, 3), (40, 36, 8), (29, 27, 9), (48, 40, 16), (20, 22, 24)]
    for i, (h, w, c) in enumerate(shapes):
        x = blob_texture(rng, h, w, c) if i % 2 == 0 else f32(rng.random((h, w, c)))
        gh, gv = glr.sobel_gradients(x)
        em = glr.binarize_gradients(gh, gv, 0.2)
        maps = np.stack([m.astype(np.uint8) for m in em.as_tuple()])
        from glr.edges import _shi_tomasi_response
        mag = np.sqrt(gh ** 2 + gv ** 2).mean(axis=2)
        resp = _shi_tomasi_response(mag)
        corners = glr.detect_corners(x, max_n=40, nms_radius=3)
        ex = glr.select_exemplars(corners, (h, w), 6, uniform_interval=7)
        cases.update({
            f"x{i}": x, f"gh{i}": gh, f"gv{i}": gv, f"maps{i}": maps, f"resp{i}": resp,
            f"corners{i}": np.array(corners, dtype=np.int32).reshape(-1, 2),
            f"anchors{i}": np.array(ex.anchors, dtype=np.int32).reshape(-1, 2),
            f"tags{i}": np.array([t == "uniform" for t in ex.tags], dtype=np.uint8),
        })
    cases["n"] = np.array(len(shapes))
    np.savez_compressed(OUT / "edges.npz", **cases)


def gen_heat_topk():
    """similarity_heatmap + global_match on random edge maps (acceptance #1
    style) and blob images; positions and padding from the reference."""
    rng = np.random.default_rng(202)
    cases = {}
    specs = [(20, 18, 2, 6, 3, 5, None), (33, 41, 1, 8, 6, 16, None), (28, 30, 3, 4, 5, 9, 1),
             (45, 40, 4, 8, 7, 24, None), (16, 16, 1, 8, 3, 40, None), (12, 11, 2, 3, 4, 30, 1)]
    for i, (h, w, c, p, n, k, sep) in enumerate(specs):
        edge = random_maps(rng, h, w, c, float(rng.uniform(0.1, 0.5)))
        anchors = [(int(rng.integers(0, h - p + 1)), int(rng.integers(0, w - p + 1)))
                   for _ in range(n)]
        ex = ExemplarSet(anchors=anchors, tags=["corner"] * n, patch_size=p)
        hm = glr.matching.similarity_heatmap(edge, ex)
        cfg = glr.MatchConfig(patch_size=p, group_size=k, min_separation=sep)
        x = f32(rng.random((h, w, c)))
        groups = glr.global_match(x, ex, cfg, edge)
        cases.update({
            f"maps{i}": np.stack([m.astype(np.uint8) for m in edge.as_tuple()]),
            f"anchors{i}": np.array(anchors, dtype=np.int32),
            f"heat{i}": hm.values.astype(np.int32),
            f"x{i}": x,
            f"positions{i}": np.array([g.positions for g in groups], dtype=np.int32),
            f"padded{i}": np.array([g.padded for g in groups], dtype=np.int32),
            f"matrix{i}": np.stack([g.matrix for g in groups]),
            f"meta{i}": np.array([h, w, c, p, n, k, cfg.sep]),
        })
    cases["n"] = np.array(len(specs))
    np.savez_compressed(OUT / "heat_topk.npz", **cases)


def gen_topk_slices():
    """top_k_positions on random integer slices (test_matching.py:134-143 style)."""
    rng = np.random.default_rng(303)
    cases = {}
    n = 60
    for i in range(n):
        oh, ow = int(rng.integers(2, 40)), int(rng.integers(2, 40))
        s = rng.integers(0, int(rng.choice([2, 6, 50])), size=(oh, ow)).astype(np.float64)
        anchor = (int(rng.integers(0, oh)), int(rng.integers(0, ow)))
        k = int(rng.integers(1, 40))
        sep = int(rng.integers(0, 4))
        pos, pad = glr.matching.top_k_positions(s, anchor, k, sep)
        cases.update({f"s{i}": s, f"meta{i}": np.array([anchor[0], anchor[1], k, sep, pad]),
                      f"pos{i}": np.array(pos, dtype=np.int32)})
    cases["n"] = np.array(n)
    np.savez_compressed(OUT / "topk_slices.npz", **cases)


def gen_wnnm():
    rng = np.random.default_rng(404)
    cases = {}
    shapes = [(64, 64), (128, 48), (12, 8), (5, 20), (64, 10), (512, 64), (2, 2), (33, 17)]
    for i, (m, k) in enumerate(shapes):
        a = rng.standard_normal((m, k)) if i % 2 else f32(rng.random((m, k)))
        sigma = float(rng.uniform(0.01, 0.5))
        out = glr.wnnm_prox(a, glr.WnnmParams(noise_sigma=sigma))
        uw = glr.wnnm_prox(a, glr.WnnmParams(uniform_weight=0.3))
        cases.update({f"m{i}": a, f"sigma{i}": np.array(sigma), f"out{i}": out, f"uw{i}": uw})
    cases["n"] = np.array(len(shapes))
    # glr_regularize on gathered groups (lowrank.py:68-87)
    x = blob_texture(rng, 30, 28, 3)
    pos = [[(int(rng.integers(0, 25)), int(rng.integers(0, 23))) for _ in range(6)]
           for _ in range(9)]
    groups = [glr.gather_group(x, q, 4) for q in pos]
    z = glr.glr_regularize(x, groups, glr.WnnmParams(noise_sigma=0.05))
    cases.update({"reg_x": x, "reg_pos": np.array(pos, dtype=np.int32), "reg_z": z})
    np.savez_compressed(OUT / "wnnm.npz", **cases)


def gen_operators():
    rng = np.random.default_rng(505)
    x8 = f32(rng.random((16, 20, 8)))
    masks = glr.bernoulli_masks(16, 20, 8, seed=3)
    cop = glr.cacti_operator(masks)
    y = cop.forward(x8)
    mm = glr.msfa_pattern("periodic-4x4", 16, 16, 20)
    mop = glr.msfa_operator(mm)
    x16 = f32(rng.random((16, 20, 16)))
    fmask = glr.radial_mask(16, 16, 5)
    fop = glr.fourier_operator(fmask)
    xf = f32(rng.random((16, 16, 1)))
    yf = fop.forward(xf)
    np.savez_compressed(
        OUT / "operators.npz",
        cacti_x=x8, cacti_masks=masks, cacti_y=y, cacti_adj=cop.adjoint(y), cacti_gram=cop.gram_diag,
        msfa_x=x16, msfa_masks=mm, msfa_y=mop.forward(x16), msfa_adj=mop.adjoint(mop.forward(x16)),
        four_x=xf, four_mask=fmask, four_y=yf, four_adj=fop.adjoint(yf),
        bern_seed7=glr.bernoulli_masks(9, 7, 3, seed=7),
    )


def gen_solves():
    """Small end-to-end gap_solve runs; the per-refresh anchors/positions are
    captured by wrapping the reference's own global_match."""
    rng = np.random.default_rng(606)
    captured = []
    orig = ref_solvers.global_match

    def spy(x, exemplars, cfg, edge):
        groups = orig(x, exemplars, cfg, edge)
        captured.append((list(exemplars.anchors), [g.positions for g in groups]))
        return groups

    ref_solvers.global_match = spy
    try:
        cases = {}
        runs = [
            ("cacti", (32, 32, 4), dict(patch_size=4, group_size=8, max_corners=24,
                                        exemplar_stride=4), 8),
            ("msfa", (32, 32, 4), dict(patch_size=4, group_size=8, max_corners=24,
                                       exemplar_stride=4), 6),
            ("cacti", (40, 36, 8), dict(patch_size=8, group_size=16, max_corners=30,
                                        exemplar_stride=6), 6),
        ]
        for i, (kind, (h, w, c), mc, iters) in enumerate(runs):
            scene = blob_texture(rng, h, w, c)
            if kind == "cacti":
                masks = glr.bernoulli_masks(h, w, c, seed=10 + i)
                op = glr.cacti_operator(masks)
            else:
                masks = glr.msfa_pattern("bayer-like-2x2", 4, h, w)
                op = glr.msfa_operator(masks)
            y = op.forward(scene)
            cfg = glr.SolverConfig(regularizer="glr", max_iters=iters, match=glr.MatchConfig(**mc))
            captured.clear()
            xr, rep = glr.gap_solve(op, y, cfg, ref=scene)
            cases.update({
                f"kind{i}": np.array(kind), f"scene{i}": scene, f"masks{i}": masks, f"y{i}": y,
                f"out{i}": xr, f"resid{i}": np.array([r["residual"] for r in rep.rows]),
                f"psnr{i}": np.array([r["psnr_db"] for r in rep.rows]),
                f"mc{i}": np.array([mc["patch_size"], mc["group_size"], mc["max_corners"],
                                    mc["exemplar_stride"], iters]),
                f"nref{i}": np.array(len(captured)),
            })
            for j, (anc, pos) in enumerate(captured):
                cases[f"anchors{i}_{j}"] = np.array(anc, dtype=np.int32)
                cases[f"positions{i}_{j}"] = np.array(pos, dtype=np.int32)
        cases["n"] = np.array(len(runs))
        np.savez_compressed(OUT / "solves.npz", **cases)
    finally:
        ref_solvers.global_match = orig


def gen_admm():
    """A small ADMM-GLR run (solvers.py:311-341), refresh positions captured."""
    rng = np.random.default_rng(707)
    captured = []
    orig = ref_solvers.global_match

    def spy(x, exemplars, cfg, edge):
        groups = orig(x, exemplars, cfg, edge)
        captured.append((list(exemplars.anchors), [g.positions for g in groups]))
        return groups

    ref_solvers.global_match = spy
    try:
        h, w, c = 32, 36, 4
        scene = blob_texture(rng, h, w, c)
        masks = glr.bernoulli_masks(h, w, c, seed=21)
        op = glr.cacti_operator(masks)
        y = op.forward(scene)
        mc = glr.MatchConfig(patch_size=4, group_size=8, max_corners=24, exemplar_stride=4)
        cfg = glr.SolverConfig(algorithm="admm", regularizer="glr", max_iters=7, match=mc,
                               admm_rho=0.01)
        xr, rep = glr.admm_solve(op, y, cfg, ref=scene)
        cases = {"scene": scene, "masks": masks, "y": y, "out": xr,
                 "resid": np.array([r["residual"] for r in rep.rows]),
                 "psnr": np.array([r["psnr_db"] for r in rep.rows]),
                 "nref": np.array(len(captured))}
        for j, (anc, pos) in enumerate(captured):
            cases[f"anchors_{j}"] = np.array(anc, dtype=np.int32)
            cases[f"positions_{j}"] = np.array(pos, dtype=np.int32)
        np.savez_compressed(OUT / "admm.npz", **cases)
    finally:
        ref_solvers.global_match = orig


def gen_metrics():
    """metrics.py: psnr / ssim of the reference on small random pairs."""
    rng = np.random.default_rng(909)
    cases = {}
    shapes = [(11, 11, 1), (24, 31, 3), (40, 36, 8)]
    for i, sh in enumerate(shapes):
        a = f32(rng.random(sh))
        b = np.clip(a + 0.1 * f32(rng.standard_normal(sh)), -0.2, 1.3)
        cases.update({f"a{i}": a, f"b{i}": b,
                      f"ssim{i}": np.array(glr.ssim(a, np.clip(b, 0, 1), 1.0)),
                      f"psnr{i}": np.array(glr.psnr(a, np.clip(b, 0, 1), 1.0))})
    cases["n"] = np.array(len(shapes))
    np.savez_compressed(OUT / "metrics.npz", **cases)


def gen_interp():
    """init="interp" (solvers.py:237-254): the reference's _interp_init on
    MSFA / CACTI / Fourier operators, and one MSFA gap_solve started from it."""
    rng = np.random.default_rng(808)
    cases = {}
    mm = glr.msfa_pattern("periodic-4x4", 16, 24, 20)
    x16 = f32(rng.random((24, 20, 16)))
    mop = glr.msfa_operator(mm)
    my = mop.forward(x16)
    cases.update(msfa_masks=mm, msfa_y=my, msfa_init=ref_solvers._interp_init(mop, my))
    masks = glr.bernoulli_masks(18, 22, 6, seed=5)
    cop = glr.cacti_operator(masks)
    cy = cop.forward(f32(rng.random((18, 22, 6))))
    cases.update(cacti_masks=masks, cacti_y=cy, cacti_init=ref_solvers._interp_init(cop, cy))
    captured = []
    orig = ref_solvers.global_match

    def spy(x, exemplars, cfg, edge):
        groups = orig(x, exemplars, cfg, edge)
        captured.append((list(exemplars.anchors), [g.positions for g in groups]))
        return groups

    ref_solvers.global_match = spy
    try:
        scene = blob_texture(rng, 32, 32, 16)
        sm = glr.msfa_pattern("periodic-4x4", 16, 32, 32)
        op = glr.msfa_operator(sm)
        y = op.forward(scene)
        mc = glr.MatchConfig(patch_size=4, group_size=8, max_corners=24, exemplar_stride=4)
        cfg = glr.SolverConfig(regularizer="glr", max_iters=6, match=mc, init="interp")
        xr, rep = glr.gap_solve(op, y, cfg, ref=scene)
        cases.update(solve_scene=scene, solve_masks=sm, solve_y=y, solve_out=xr,
                     solve_resid=np.array([r["residual"] for r in rep.rows]),
                     solve_psnr=np.array([r["psnr_db"] for r in rep.rows]),
                     solve_nref=np.array(len(captured)))
        for j, (anc, pos) in enumerate(captured):
            cases[f"solve_anchors_{j}"] = np.array(anc, dtype=np.int32)
            cases[f"solve_positions_{j}"] = np.array(pos, dtype=np.int32)
    finally:
        ref_solvers.global_match = orig
    np.savez_compressed(OUT / "interp.npz", **cases)


def gen_bm():
    """Block matching (matching.py:256-283), the pixel re-rank of global
    matching (matching.py:243-249) and small solves with the block-matching
    regularizers and glr+rerank (positions captured from the reference)."""
    rng = np.random.default_rng(808)
    cases = {}
    bm_runs = [  # (h, w, c, P, K, window, stride, quantise)
        (24, 20, 1, 4, 8, 5, 1, 0), (32, 32, 3, 6, 16, 8, 1, 0), (40, 36, 8, 8, 32, 20, 1, 0),
        (30, 30, 2, 5, 12, 7, 2, 0), (12, 12, 1, 4, 64, 20, 1, 0), (28, 26, 3, 4, 10, 6, 1, 4),
        (20, 24, 1, 4, 6, 9, 3, 2), (26, 26, 16, 8, 9, 8, 1, 0),
    ]
    for i, (h, w, c, p, k, win, st, q) in enumerate(bm_runs):
        x = blob_texture(rng, h, w, c) if q == 0 else f32(np.floor(rng.random((h, w, c)) * q) / q)
        anchors = [(int(rng.integers(0, h - p + 1)), int(rng.integers(0, w - p + 1)))
                   for _ in range(6)] + [(0, 0), (h - p, w - p)]
        ex = ExemplarSet(anchors=anchors, tags=["uniform"] * len(anchors), patch_size=p)
        cfg = glr.MatchConfig(patch_size=p, group_size=k, bm_window=max(win, p), bm_stride=st,
                              mode="bm-uniform")
        groups = glr.block_match(x, ex, cfg)
        cases.update({f"bm_x{i}": x, f"bm_anchors{i}": np.array(anchors, dtype=np.int32),
                      f"bm_cfg{i}": np.array([p, k, max(win, p), st]),
                      f"bm_pos{i}": np.array([g.positions for g in groups], dtype=np.int32),
                      f"bm_pad{i}": np.array([g.padded for g in groups], dtype=np.int32)})
    cases["bm_n"] = np.array(len(bm_runs))
    rr_runs = [(32, 28, 3, 4, 12), (40, 40, 8, 8, 16), (24, 24, 1, 6, 64)]
    for i, (h, w, c, p, k) in enumerate(rr_runs):
        x = blob_texture(rng, h, w, c)
        gh, gv = glr.sobel_gradients(x)
        edge = glr.binarize_gradients(gh, gv, 0.2)
        anchors = [(int(rng.integers(0, h - p + 1)), int(rng.integers(0, w - p + 1)))
                   for _ in range(10)]
        ex = ExemplarSet(anchors=anchors, tags=["corner"] * 10, patch_size=p)
        plain = glr.global_match(x, ex, glr.MatchConfig(patch_size=p, group_size=k), edge)
        rer = glr.global_match(x, ex, glr.MatchConfig(patch_size=p, group_size=k,
                                                      rerank_pixel=True), edge)
        cases.update({f"rr_x{i}": x, f"rr_anchors{i}": np.array(anchors, dtype=np.int32),
                      f"rr_cfg{i}": np.array([p, k]),
                      f"rr_plain{i}": np.array([g.positions for g in plain], dtype=np.int32),
                      f"rr_pos{i}": np.array([g.positions for g in rer], dtype=np.int32)})
    cases["rr_n"] = np.array(len(rr_runs))

    captured = []
    orig_gm, orig_bm = ref_solvers.global_match, ref_solvers.block_match

    def spy_gm(x, exemplars, cfg, edge):
        groups = orig_gm(x, exemplars, cfg, edge)
        captured.append((list(exemplars.anchors), [g.positions for g in groups]))
        return groups

    def spy_bm(x, exemplars, cfg):
        groups = orig_bm(x, exemplars, cfg)
        captured.append((list(exemplars.anchors), [g.positions for g in groups]))
        return groups

    ref_solvers.global_match, ref_solvers.block_match = spy_gm, spy_bm
    try:
        runs = [  # (regularizer, rerank, algorithm, match kwargs, iters)
            ("nlr-bm", False, "gap", dict(patch_size=4, group_size=8, exemplar_stride=5,
                                          bm_window=6), 7),
            ("nlr-corner-bm", False, "gap", dict(patch_size=4, group_size=8, max_corners=24,
                                                 bm_window=8), 6),
            ("nlr-corner-uniform-bm", False, "gap", dict(patch_size=4, group_size=8,
                                                         max_corners=20, exemplar_stride=4,
                                                         bm_window=5, bm_stride=2), 6),
            ("glr", True, "gap", dict(patch_size=4, group_size=8, max_corners=24,
                                      exemplar_stride=4, rerank_pixel=True), 6),
            ("nlr-bm", False, "admm", dict(patch_size=4, group_size=8, exemplar_stride=6,
                                           bm_window=6), 6),
        ]
        for i, (reg, rer, alg, mc, iters) in enumerate(runs):
            h, w, c = 32, 36, 4
            scene = blob_texture(rng, h, w, c)
            masks = glr.bernoulli_masks(h, w, c, seed=30 + i)
            op = glr.cacti_operator(masks)
            y = op.forward(scene)
            cfg = glr.SolverConfig(regularizer=reg, algorithm=alg, max_iters=iters,
                                   match=glr.MatchConfig(**mc), admm_rho=0.01)
            captured.clear()
            solve = glr.gap_solve if alg == "gap" else glr.admm_solve
            xr, rep = solve(op, y, cfg, ref=scene)
            cases.update({
                f"sv_reg{i}": np.array(reg), f"sv_alg{i}": np.array(alg),
                f"sv_mc{i}": np.array(repr(mc)), f"sv_iters{i}": np.array(iters),
                f"sv_scene{i}": scene, f"sv_masks{i}": masks, f"sv_y{i}": y, f"sv_out{i}": xr,
                f"sv_resid{i}": np.array([r["residual"] for r in rep.rows]),
                f"sv_psnr{i}": np.array([r["psnr_db"] for r in rep.rows]),
                f"sv_nref{i}": np.array(len(captured))})
            for j, (anc, pos) in enumerate(captured):
                cases[f"sv_anchors{i}_{j}"] = np.array(anc, dtype=np.int32)
                cases[f"sv_positions{i}_{j}"] = np.array(pos, dtype=np.int32)
        cases["sv_n"] = np.array(len(runs))
    finally:
        ref_solvers.global_match, ref_solvers.block_match = orig_gm, orig_bm
    np.savez_compressed(OUT / "bm.npz", **cases)


def gen_tens():
    """.tens files written by the reference (tensorio.py:47-56), kept as raw
    bytes, and a run config serialized by the reference (config.py:123-126)."""
    import tempfile
    from glr import tensorio, config
    rng = np.random.default_rng(909)
    arrays = [rng.random((5, 4, 3)), rng.random((7,)).astype(np.float32),
              (rng.random((3, 3)) * 255).astype(np.uint8),
              rng.random((2, 3)) + 1j * rng.random((2, 3)), np.float64(2.5) * np.ones(())]
    cases = {"n": np.array(len(arrays))}
    with tempfile.TemporaryDirectory() as d:
        for i, a in enumerate(arrays):
            path = f"{d}/t{i}.tens"
            tensorio.write_tensor(path, a)
            cases[f"bytes{i}"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
            cases[f"arr{i}"] = a
            cases[f"read{i}"] = tensorio.read_tensor(path)
    run = config.parse_run_config({"solver": {"max_iters": 7, "regularizer": "nlr-bm",
                                              "match": {"patch_size": 6, "bm_window": 9}},
                                   "operator": {"kind": "msfa", "channels": 4}})
    cases["config_json"] = np.array(config.serialize_run_config(run))
    np.savez_compressed(OUT / "tens.npz", **cases)


def gen_tv():
    """tv_denoise (solvers.py:121-139) and GAP / ADMM solves with the TV
    regularizer, run by the reference."""
    rng = np.random.default_rng(1010)
    cases = {}
    tv_runs = [((20, 24, 1), 0.05, 20), ((17, 13, 3), 0.2, 7), ((9, 9, 2), 0.0, 5)]
    for i, (shape, wgt, iters) in enumerate(tv_runs):
        x = f32(rng.random(shape))
        cases.update({f"tv_x{i}": x, f"tv_cfg{i}": np.array([wgt, iters]),
                      f"tv_out{i}": ref_solvers.tv_denoise(x, wgt, iters)})
    cases["tv_n"] = np.array(len(tv_runs))
    for i, alg in enumerate(("gap", "admm")):
        h, w, c = 32, 28, 4
        scene = blob_texture(rng, h, w, c)
        masks = glr.bernoulli_masks(h, w, c, seed=50 + i)
        op = glr.cacti_operator(masks)
        y = op.forward(scene)
        cfg = glr.SolverConfig(regularizer="tv", algorithm=alg, max_iters=12, tv_weight=0.03,
                               tv_iters=15, admm_rho=0.01)
        xr, rep = ref_solvers.solve(op, y, cfg, ref=scene)
        cases.update({f"sv_scene{i}": scene, f"sv_masks{i}": masks, f"sv_y{i}": y,
                      f"sv_out{i}": xr, f"sv_resid{i}": np.array([r["residual"] for r in rep.rows]),
                      f"sv_psnr{i}": np.array([r["psnr_db"] for r in rep.rows])})
    np.savez_compressed(OUT / "tv.npz", **cases)


class _StopSolve(Exception):
    pass


class _NoClip:
    """Stand-in for the reference module's ``np`` whose ``clip`` is the
    identity: the documented no-clip policy for complex (re, im) images
     applied to the UNMODIFIED gap_solve code."""

    def __getattr__(self, name):
        return getattr(np, name)

    @staticmethod
    def clip(a, lo, hi):
        return a


def _complex_fourier_operator(mask):
    """operators.py:65-89 minus ``.real`` on (H, W, 2) = (re, im)."""
    from glr.operators import SensingOperator
    mask = np.asarray(mask, dtype=np.float64)
    h, w = mask.shape

    def fwd(x):
        x = np.asarray(x, dtype=np.float64)
        return mask * np.fft.fft2(x[:, :, 0] + 1j * x[:, :, 1], norm="ortho")

    def adj(y):
        z = np.fft.ifft2(mask * y, norm="ortho")
        return np.stack([z.real, z.imag], axis=2)

    return SensingOperator(kind="fourier", forward=fwd, adjoint=adj, gram_diag=mask.copy(),
                           x_shape=(h, w, 2), meta={"mask": mask})


def gen_configs(names=("C1", "C3", "C4")):
    """BASELINE.json configurations at FULL size, run by the unmodified
    reference gap_solve on the package's seeded workloads (inputs are the
    same fp32-rounded arrays the GPU path sees):

      C1  all 30 iterations: every refresh's anchors + positions, the
          per-iteration residuals and the final clip(x, 0, 1)
      C3  first 10 of 40 iterations (complex operator, no-clip policy)
      C4  first 10 of 30 iterations (init="interp", the workload's setting)

    For C3/C4 the solve is stopped when iteration 10 begins (the iterate
    handed to regularize_dispatch = x after 10 iterations, with the
    max_iters of the config so the sigma schedule is the config's). Stored:
    the first two refreshes' anchors/positions (int16), the residuals, x
    (C3 full, float32; C4 a seeded sample of 2**18 entries, float64, plus
    sum / sum of squares / PSNR of the full array)."""
    import time
    sys.path.insert(0, str(OUT.parents[1]))
    from paper_2301_03047_b200 import workloads
    for name in names:
        wl = workloads.make(name)
        mc = wl.match
        stop_at = {"C1": None, "C3": 10, "C4": 10}[name]
        if wl.kind == "cacti":
            op = glr.cacti_operator(wl.masks)
        elif wl.kind == "msfa":
            op = glr.msfa_operator(wl.masks)
        else:
            op = _complex_fourier_operator(wl.masks)
        cfg = glr.SolverConfig(regularizer="glr", max_iters=wl.max_iters, init=wl.init,
                               match=glr.MatchConfig(patch_size=mc.patch_size,
                                                     group_size=mc.group_size,
                                                     max_corners=mc.max_corners,
                                                     exemplar_stride=mc.exemplar_stride))
        captured, resid, stopped = [], [], {}
        orig_gm, orig_rd, orig_rec = (ref_solvers.global_match, ref_solvers.regularize_dispatch,
                                      ref_solvers._record)
        orig_np = ref_solvers.np

        def spy_gm(x, exemplars, c, edge):
            groups = orig_gm(x, exemplars, c, edge)
            captured.append((list(exemplars.anchors), [g.positions for g in groups]))
            return groups

        def spy_rd(x, c, state, iteration=0, sigma=None):
            if stop_at is not None and iteration == stop_at:
                stopped["x"] = np.array(x, copy=True)
                raise _StopSolve()
            return orig_rd(x, c, state, iteration=iteration, sigma=sigma)

        def spy_rec(*a, **k):
            r = orig_rec(*a, **k)
            resid.append(r)
            return r

        ref_solvers.global_match, ref_solvers.regularize_dispatch = spy_gm, spy_rd
        ref_solvers._record = spy_rec
        if wl.kind == "fourier":
            ref_solvers.np = _NoClip()
        t0 = time.perf_counter()
        try:
            out, _ = glr.gap_solve(op, wl.y, cfg)
        except _StopSolve:
            out = stopped["x"]
        finally:
            ref_solvers.global_match, ref_solvers.regularize_dispatch = orig_gm, orig_rd
            ref_solvers._record = orig_rec
            ref_solvers.np = orig_np
        secs = time.perf_counter() - t0
        keep = len(captured) if stop_at is None else 2
        cases = {"name": np.array(name), "iters": np.array(len(resid)),
                 "resid": np.array(resid), "nref": np.array(keep),
                 "seconds": np.array(secs)}
        for j, (anc, pos) in enumerate(captured[:keep]):
            cases[f"anchors_{j}"] = np.array(anc, dtype=np.int16)
            cases[f"positions_{j}"] = np.array(pos, dtype=np.int16)
        if name == "C4":
            rng = np.random.default_rng(4242)
            idx = np.sort(rng.choice(out.size, size=1 << 18, replace=False))
            cases.update(sample_idx=idx.astype(np.int32), sample=out.ravel()[idx],
                         x_sum=np.array(out.sum()), x_sumsq=np.array((out * out).sum()),
                         psnr=np.array(glr.psnr(wl.scene, np.clip(out, 0, 1), 1.0)))
        else:
            cases.update(x=out.astype(np.float32),
                         psnr=np.array(glr.psnr(wl.scene, np.clip(out, 0, 1), 1.0)))
        np.savez_compressed(OUT / f"config_{name}.npz", **cases)
        print(name, f"{secs:.1f} s", len(resid), "iterations", len(captured), "refreshes",
              [len(a) for a, _ in captured], flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        sys.exit(0)
    gen_bm()
    gen_tv()
    gen_tens()
    gen_metrics()
    gen_interp()
    gen_admm()
    gen_edges()
    gen_heat_topk()
    gen_topk_slices()
    gen_wnnm()
    gen_operators()
    gen_solves()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
