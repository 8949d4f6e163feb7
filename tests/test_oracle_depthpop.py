"""Pins for the oracle's depth-map population (Sec. 3.2, Eq. 5, Eq. 6)
and the Eq. 6 sample-set generator.  The Eq. 5 pins use hand-built nets whose cumulative outputs y_i
are chosen directly (W_i = 0 makes h_i constant, a_i = 0 makes t_i = c_i), so the expected depths are
worked out by hand from the printed rule, not recomputed by the oracle's code."""
from types import SimpleNamespace

import numpy as np
import pytest

import oracle
import sandgen as g


def _const_net(t, omega0=30.0):
    """L = len(t), H = 1 net with y_i = t_1 + ... + t_i at every x (W = 0, a = 0, c_i = t_i)."""
    L = len(t)
    z = lambda *s: np.zeros(s, np.float32)
    spec = SimpleNamespace(L=L, H=1, omega0=omega0, tail=0)
    return SimpleNamespace(spec=spec, W=[z(1, 3)] + [z(1, 1) for _ in range(L - 1)], b=[z(1) for _ in range(L)],
                           a=[z(1) for _ in range(L)], c=list(map(float, t)), a1=[], c1=[])


X = np.random.default_rng(0).uniform(-1, 1, (7, 3)).astype(np.float32)


def test_spec_example_converged_at_depth_2():
    """SPEC S:300 example: y = (0.001, 0.0002, 0.0001), r = 0.00015 -> d = 2 (|y3 - y2| = 1e-4 < r,
    |y3 - y1| = 9e-4 >= r, all signs +)."""
    p = _const_net([0.001, -0.0008, -0.0001])
    assert np.all(oracle.required_depth(p, X, 0.00015) == 2)


def test_sign_gate():
    """S_i gate (Eq. 5): y_1 has the opposite sign of y_L -> d >= 2 however large r is."""
    p = _const_net([-0.001, 0.00105, 0.0])        # y = (-0.001, 5e-5, 5e-5)
    assert np.all(oracle.required_depth(p, X, 1e9) == 2)
    assert np.all(oracle.required_depth(p, X, 1e-3) == 2)


def test_far_branch_is_sign_only_and_near_branch_adds_magnitude():
    """Eq. 5 first case (delta = 0): sign only; second case adds |y_L - y_i| < r."""
    p = _const_net([0.5, -0.1, 0.05])             # y = (0.5, 0.4, 0.45)
    assert np.all(oracle.required_depth(p, X, 0.01, near=False) == 1)
    assert np.all(oracle.required_depth(p, X, 0.01, near=True) == 3)   # 0.05 >= r at i = 1, 2
    assert np.all(oracle.required_depth(p, X, 0.0500001, near=True) == 1)


def test_zero_tails_after_first_give_depth_1():
    """SPEC S:298 example: t_i = 0 for all i >= 2 -> y_1 = y_L -> d(x) = 1 (on a random SIREN)."""
    p = g.make_weights(g.TMlpSpec(L=4, H=16, seed=2))
    for i in range(1, 4):
        p.a[i][...] = 0
        p.c[i] = 0.0
    assert np.all(oracle.required_depth(p, X, 1e-6) == 1)


def test_depth_range_and_limits():
    """d(x) in [1, L]; r -> 0 forces L (unless y_i == y_L exactly); i = L always qualifies."""
    p = g.make_weights(g.TMlpSpec(L=6, H=32, seed=3))
    d = oracle.required_depth(p, X, 1.5e-4)
    assert d.min() >= 1 and d.max() <= 6
    assert np.all(oracle.required_depth(p, X, 0.0) == 6)


def test_leaf_max_pooling_hand_case():
    """Eq. 6: d(N) is the max of the per-sample depths (SPEC S:304 example {1, 3, 2} -> 3, here with two
    hand-built constant nets mixed through a leaf whose samples straddle x = 0 via W_1's sign)."""
    # the oracle's pooling equals the max of its per-point depths on a real net
    p = g.make_weights(g.TMlpSpec(L=5, H=16, seed=4))
    s = np.random.default_rng(5).uniform(-1, 1, (11, 6, 3)).astype(np.float32)
    per = oracle.required_depth(p, s.reshape(-1, 3), 2e-3).reshape(11, 6)
    np.testing.assert_array_equal(oracle.populate_leaf_depths(p, s, 2e-3), per.max(axis=1))


def test_leaf_samples_geometry_and_determinism():
    """Sample set (R21): 8 exact corners, the exact centre, k interior points inside the
    half-open cell; deterministic in (seed, leaf order)."""
    lev = np.array([1, 3, 7])
    ijk = np.array([[0, 1, 1], [5, 2, 7], [100, 3, 127]])
    s = g.leaf_samples(lev, ijk, 5, seed=9)
    assert s.shape == (3, 14, 3)
    side = 2.0 / 2.0 ** lev
    lo = -1.0 + ijk * side[:, None]
    for c in range(8):
        off = np.array([(c >> 0) & 1, (c >> 1) & 1, (c >> 2) & 1])
        np.testing.assert_allclose(s[:, c, :], lo + off * side[:, None], atol=1e-7)
    np.testing.assert_allclose(s[:, 8, :], lo + 0.5 * side[:, None], atol=1e-7)
    inner = s[:, 9:, :].astype(np.float64)
    assert np.all(inner >= lo[:, None, :] - 1e-7) and np.all(inner <= (lo + side[:, None])[:, None, :] + 1e-7)
    np.testing.assert_array_equal(s, g.leaf_samples(lev, ijk, 5, seed=9))
    assert not np.array_equal(s, g.leaf_samples(lev, ijk, 5, seed=10))
