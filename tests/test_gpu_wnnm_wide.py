"""WNNM for groups wider than 64 columns (lowrank.py:46-65 takes any K) on
the generic device path, against the SVD oracle (GPU)."""

import numpy as np
import pytest

import glr_oracle as O

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2301_03047_b200")
from paper_2301_03047_b200 import workloads  # noqa: E402


@pytest.mark.parametrize("m,k", [(96, 65), (200, 100), (64, 128), (33, 81), (300, 160)])
def test_wnnm_prox_wide_groups(m, k):
    rng = np.random.default_rng(m * 1000 + k)
    base = rng.standard_normal((m, 4)) @ rng.standard_normal((4, k))
    a = base + 0.05 * rng.standard_normal((m, k))
    for sigma in (0.02, 0.3):
        got = G.wnnm_prox(a, G.WnnmParams(noise_sigma=sigma))
        want = O.wnnm_prox(a, sigma)
        assert np.abs(got - want).max() <= 1e-9 * max(1.0, np.abs(want).max())
    got = G.wnnm_prox(a, G.WnnmParams(uniform_weight=0.5))
    want = O.wnnm_prox(a, 0.0, uniform_weight=0.5)
    assert np.abs(got - want).max() <= 1e-9 * max(1.0, np.abs(want).max())


def test_gap_solve_group_size_above_64():
    scene = workloads.cacti_scene(40, 36, 4, seed=9)
    masks = G.bernoulli_masks(40, 36, 4, seed=10)
    y = O.masksum_forward(scene, masks)
    mc = G.MatchConfig(patch_size=4, group_size=80, max_corners=12, exemplar_stride=5)
    cfg = G.SolverConfig(max_iters=4, match=mc)
    trace = []
    x, _ = G.gap_solve(G.cacti_operator(masks), y, cfg, trace=trace)
    otrace = []
    xo, _, _ = O.gap_solve(O.Operator("cacti", masks=masks), y, 4, patch_size=4, group_size=80,
                           max_corners=12, exemplar_stride=5, trace=otrace)
    for (a, p), (ao, po) in zip(trace, otrace):
        assert np.array_equal(np.asarray(a), np.asarray(ao))
        assert np.array_equal(np.asarray(p), np.asarray(po))
    assert np.abs(x - xo).max() <= 1e-6
