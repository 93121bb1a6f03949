"""The public regularize_dispatch (solvers.py:170-210) on device, and solve
repeatability (GPU).

* refresh at iteration 0 == the oracle's match + glr_regularize;
* non-refresh iterations re-gather at the CACHED positions
  (solvers.py:204-207), including a MatchState built by the caller (no
  engine attached) and one whose positions were edited: both must use
  ``state.positions``;
* two consecutive GapRunner.run() calls on the same y are bitwise equal (no
  eigenvector warm start leaks from one solve into the next)."""

import numpy as np
import pytest

import glr_oracle as O

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2301_03047_b200")
from paper_2301_03047_b200 import _device as D, workloads  # noqa: E402
from paper_2301_03047_b200.solvers import GapRunner, MatchState  # noqa: E402


def _image():
    scene = workloads.cacti_scene(48, 44, 4, seed=7)
    return scene


def _cfg():
    mc = G.MatchConfig(patch_size=6, group_size=12, max_corners=20, exemplar_stride=4)
    return G.SolverConfig(max_iters=10, match=mc)


def _oracle_z(x, positions, cfg, it):
    return O.glr_regularize(x, [list(map(tuple, p)) for p in positions], cfg.match.patch_size,
                            cfg.sigma_at(it))


def test_regularize_dispatch_refresh_and_cached_positions():
    cfg = _cfg()
    mc = cfg.match
    x0 = _image()
    st = MatchState()
    z0 = G.regularize_dispatch(x0, cfg, st, iteration=0)
    anchors, positions = O._glr_match(x0, mc.patch_size, mc.group_size, mc.max_corners,
                                      mc.exemplar_stride, mc.edge_threshold, mc.sep, "glr",
                                      20, 1, False)
    assert np.array_equal(np.asarray(st.positions), np.asarray(positions))
    assert np.abs(z0 - _oracle_z(x0, positions, cfg, 0)).max() <= 1e-9
    # non-refresh iteration: re-gather the NEW iterate at the cached positions
    x1 = np.clip(x0 + 0.05 * np.sin(np.arange(x0.size)).reshape(x0.shape), 0, 1)
    z1 = G.regularize_dispatch(x1, cfg, st, iteration=1)
    assert st.last_refresh == 0
    assert np.abs(z1 - _oracle_z(x1, positions, cfg, 1)).max() <= 1e-9
    # a caller-built state: positions but no engine
    st2 = MatchState(positions=[list(g) for g in st.positions], last_refresh=0)
    z2 = G.regularize_dispatch(x1, cfg, st2, iteration=2)
    assert np.abs(z2 - _oracle_z(x1, positions, cfg, 2)).max() <= 1e-9
    # edited positions on an existing state: the edit is honoured
    edited = [list(reversed(g)) for g in st.positions[::-1]][:-1]
    st.positions = edited
    z3 = G.regularize_dispatch(x1, cfg, st, iteration=3)
    assert np.abs(z3 - _oracle_z(x1, edited, cfg, 3)).max() <= 1e-9


def test_consecutive_runs_bitwise_equal():
    wl = workloads.make("C1")
    cfg = G.SolverConfig(max_iters=12, match=wl.match)
    runner = GapRunner(workloads.operator_for(wl), cfg)
    y_d = runner.dop.upload_y(wl.y)
    a = D.host(runner.run(y_d)).copy()
    ra = D.host(runner.resid_sq).copy()
    b = D.host(runner.run(y_d)).copy()
    rb = D.host(runner.resid_sq).copy()
    assert np.array_equal(a, b)
    assert np.array_equal(ra, rb)
    x, _ = G.gap_solve(workloads.operator_for(wl), wl.y, cfg)
    assert np.array_equal(np.clip(a, 0, 1), x)
