"""TV baseline regularizer on device (glr_tv_denoise) vs the reference's
golden vectors: the prox is bit-identical (same rounding as numpy), solves
match the recorded reference runs (GPU only)."""

import numpy as np
import pytest

import glr_oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2301_03047_b200")


def test_tv_denoise_bitwise_vs_golden():
    g = load_golden("tv")
    for i in range(int(g["tv_n"])):
        wgt, iters = g[f"tv_cfg{i}"]
        assert np.array_equal(G.tv_denoise(g[f"tv_x{i}"], float(wgt), int(iters)),
                              g[f"tv_out{i}"]), i


def test_tv_denoise_bitwise_vs_oracle_large(rng):
    x = rng.random((300, 260, 8))
    assert np.array_equal(G.tv_denoise(x, 0.07, 20), O.tv_denoise(x, 0.07, 20))


@pytest.mark.parametrize("i,alg", [(0, "gap"), (1, "admm")])
def test_tv_solves_vs_reference_run(i, alg):
    g = load_golden("tv")
    cfg = G.SolverConfig(regularizer="tv", algorithm=alg, max_iters=12, tv_weight=0.03,
                         tv_iters=15, admm_rho=0.01)
    x, rep = G.solve(G.cacti_operator(g[f"sv_masks{i}"]), g[f"sv_y{i}"], cfg,
                     ref=g[f"sv_scene{i}"])
    assert np.abs(x - g[f"sv_out{i}"]).max() <= 1e-9
    assert abs(rep.rows[-1]["psnr_db"] - float(g[f"sv_psnr{i}"][-1])) <= 1e-6
    ynorm = float(np.linalg.norm(g[f"sv_y{i}"]))
    np.testing.assert_allclose([r["residual"] for r in rep.rows], g[f"sv_resid{i}"], rtol=1e-6,
                               atol=1e-9 * ynorm)
