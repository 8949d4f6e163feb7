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


def hand_pool_net(H=1):
    """L = 3 net whose per-point Eq. 5 depth is set by the sign of y_1 = sin(x_0) (omega0 = 1, W_1 = (1, 0, 0),
    b_1 = 0, a_1 = 1, c_1 = 0) against constant residuals t_2 = t_3 = -0.01 (W_2 = W_3 = 0, b = pi/2, so
    h_2 = h_3 = sin(pi/2) = 1, a_2 = a_3 = -0.01).  Units beyond the first (H > 1, for kernels with a
    minimum width) have zero weights, biases and tail entries, so they contribute nothing."""
    z = lambda *s: np.zeros(s, np.float32)
    W = [z(H, 3), z(H, H), z(H, H)]
    W[0][0, 0] = 1.0
    b = [z(H), z(H), z(H)]
    b[1][0] = b[2][0] = np.float32(np.pi / 2)
    a = [z(H), z(H), z(H)]
    a[0][0], a[1][0], a[2][0] = 1.0, -0.01, -0.01
    spec = SimpleNamespace(L=3, H=H, omega0=1.0, tail=0)
    return SimpleNamespace(spec=spec, W=W, b=b, a=a, c=[0.0, 0.0, 0.0], a1=[], c1=[])


# y_1 = s, y_2 = s - 0.01, y_3 = s - 0.02; with r = 0.05 every |y_3 - y_i| <= 0.02 < r, so Eq. 5 reduces to the
# sign gate: s = 0.5 -> all signs agree -> d = 1; s = 0.015 -> y_3 < 0 < y_2 < y_1 -> d = 3;
# s = 0.005 -> y_1 > 0 > y_2, y_3 -> d = 2.  (Worked by hand from Eq. 5; margins >= 0.005 >> float error.)
HAND_S = (0.5, 0.015, 0.005)
HAND_D = (1, 3, 2)


def hand_pool_samples():
    x0 = np.arcsin(np.array(HAND_S)).astype(np.float32)
    return np.stack([x0, np.full(3, 0.25, np.float32), np.full(3, -0.5, np.float32)], 1)


def test_leaf_max_pooling_hand_case():
    """Eq. 6 max pooling, SPEC S:304's example: one leaf whose three samples have required depths
    {1, 3, 2} (worked by hand above) gets depth 3; leaves holding one sample each keep that sample's depth."""
    p = hand_pool_net()
    s = hand_pool_samples()
    np.testing.assert_array_equal(oracle.required_depth(p, s, 0.05), HAND_D)
    assert oracle.populate_leaf_depths(p, s[None, :, :], 0.05).tolist() == [3]
    np.testing.assert_array_equal(oracle.populate_leaf_depths(p, s[:, None, :], 0.05), HAND_D)
    # two-sample leaves: {1, 2} -> 2, {2, 1} -> 2, {1, 1} -> 1
    pairs = np.stack([s[[0, 2]], s[[2, 0]], s[[0, 0]]])
    assert oracle.populate_leaf_depths(p, pairs, 0.05).tolist() == [2, 2, 1]


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
