"""Pins for the oracle's dynamic-exit query ('SAND w/o Octree'; DESIGN.md reading
R23: stop at the first layer i >= 2 whose residual has |t_i| < r, else at L; sdf = y_d).  Hand-built
nets fix the residuals t_i directly (W_i = 0 makes h_i constant, a_i = 0 makes t_i = c_i), so the
expected exits are worked out by hand; the special cases r = 0 / r = inf reduce to the full-depth and
the depth-2 truncated networks."""
from types import SimpleNamespace

import numpy as np

import oracle
import sandgen as g


def _const_net(t, omega0=30.0):
    """L = len(t), H = 1: t_i = c_i at every x (W = 0, a = 0)."""
    L = len(t)
    z = lambda *s: np.zeros(s, np.float32)
    spec = SimpleNamespace(L=L, H=1, omega0=omega0, tail=0)
    return SimpleNamespace(spec=spec, W=[z(1, 3)] + [z(1, 1) for _ in range(L - 1)], b=[z(1) for _ in range(L)],
                           a=[z(1) for _ in range(L)], c=list(map(float, t)), a1=[], c1=[])


X = np.random.default_rng(0).uniform(-1, 1, (9, 3)).astype(np.float32)


def test_first_small_residual_from_layer_2():
    """t = (1e-6, 0.3, 0.01, 1e-4, 0.2): |t_1| < r is NOT a stop (reading R23); the first i >= 2 with
    |t_i| < 0.05 is i = 3 -> d = 3, sdf = 1e-6 + 0.3 + 0.01."""
    p = _const_net([1e-6, 0.3, 0.01, 1e-4, 0.2])
    s, d = oracle.query_dynamic(p, X, 0.05)
    assert np.all(d == 3)
    np.testing.assert_allclose(s, 1e-6 + 0.3 + 0.01, rtol=0, atol=1e-12)
    s, d = oracle.query_dynamic(p, X, 0.005)       # only |t_4| = 1e-4 < 0.005
    assert np.all(d == 4)
    np.testing.assert_allclose(s, 1e-6 + 0.3 + 0.01 + 1e-4, rtol=0, atol=1e-12)


def test_strict_threshold_and_negative_residuals():
    """|t| < r is strict and uses the magnitude: t_2 = -0.02 stops at r = 0.0200001, not at r = 0.02."""
    p = _const_net([0.5, -0.02, 0.7])
    assert np.all(oracle.query_dynamic(p, X, 0.0200001)[1] == 2)
    assert np.all(oracle.query_dynamic(p, X, 0.02)[1] == 3)


def test_r_zero_is_full_depth_and_r_inf_is_depth_two():
    """r = 0: no residual is < 0 -> every point runs to L and sdf = query_full.  r = inf: every point
    stops at layer 2 and sdf = the network truncated at depth 2 (Eq. 2)."""
    p = g.make_weights(g.TMlpSpec(L=5, H=32, seed=4))
    s, d = oracle.query_dynamic(p, X, 0.0)
    assert np.all(d == 5)
    np.testing.assert_allclose(s, oracle.query_full(p, X), rtol=0, atol=1e-12)
    s, d = oracle.query_dynamic(p, X, np.inf)
    assert np.all(d == 2)
    np.testing.assert_allclose(s, oracle.tmlp_forward(p, X, 2), rtol=0, atol=1e-12)


def test_agrees_with_full_trace_selection():
    """Early termination changes nothing for the points that continue: the exit layer and value equal
    those selected afterwards from the full trace t_1..t_L of every point."""
    p = g.make_weights(g.TMlpSpec(L=6, H=32, seed=5))
    x = np.random.default_rng(1).uniform(-1, 1, (400, 3)).astype(np.float32)
    _, ts, ys = oracle.tmlp_trace(p, x)
    r = float(np.median(np.abs(ts[1:])))           # about half the residuals below r
    stop = np.abs(ts[1:-1]) < r                   # candidates i = 2 .. L-1
    exp_d = np.where(stop.any(0), np.argmax(stop, 0) + 2, 6)
    s, d = oracle.query_dynamic(p, x, r)
    np.testing.assert_array_equal(d, exp_d)
    np.testing.assert_allclose(s, ys[exp_d - 1, np.arange(400)], rtol=0, atol=1e-12)
    assert 2 in d and 6 in d


def test_single_layer_and_nonfinite():
    p = g.make_weights(g.TMlpSpec(L=1, H=16, seed=6))
    s, d = oracle.query_dynamic(p, X, 1e9)
    assert np.all(d == 1)
    np.testing.assert_allclose(s, oracle.query_full(p, X), rtol=0, atol=1e-12)
    x = X.copy()
    x[2, 1] = np.nan
    s, d = oracle.query_dynamic(g.make_weights(g.TMlpSpec(L=3, H=16, seed=7)), x, 0.01)
    assert d[2] == oracle.NONFINITE_DEPTH and np.isnan(s[2])
    assert np.all(np.isfinite(np.delete(s, 2)))
