"""Pins for the oracle's T-MLP (Eq. 1-3, Appendix A) against things other than itself.

Each test names the paper passage and the kind of pin (closed form, library routine, hand
computation, invariant).  All CPU-only.
"""
import json
import os
from types import SimpleNamespace

import numpy as np
import pytest
import torch

import oracle
import sandgen as g

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _params(L, H, omega0=30.0, tail=0, seed=3):
    return g.make_weights(g.TMlpSpec(L=L, H=H, omega0=omega0, tail=tail, seed=seed))


def _hand_params(d, tail):
    spec = SimpleNamespace(L=2, H=1, omega0=d["omega0"], tail=tail)
    f = lambda v: np.array(v, np.float32)
    return SimpleNamespace(spec=spec, W=[f(d["W1"]), f(d["W2"])], b=[f(d["b1"]), f(d["b2"])],
                           a=[f(d["a1"]), f(d["a2"])], c=[d["c1"], d["c2"]],
                           a1=[f(d["a21"])], c1=[d["c21"]])


def test_hand_computed_L2_H1_linear_and_mult():
    """SPEC S:142 / Eq. 2-3: pencil-and-paper values (tests/golden/hand_L2_H1.json)."""
    d = json.load(open(os.path.join(GOLD, "hand_L2_H1.json")))
    x = np.array([d["x"]], np.float32)
    for tail, key in ((0, "y2_linear"), (1, "y2_mult")):
        p = _hand_params(d, tail)
        assert oracle.tmlp_forward(p, x, 1)[0] == pytest.approx(d["y1"], abs=1e-15)
        assert oracle.tmlp_forward(p, x, 2)[0] == pytest.approx(d[key], abs=1e-15)
        hs, ts, ys = oracle.tmlp_trace(p, x)
        assert hs[0][0, 0] == pytest.approx(d["h1"], abs=1e-15)
        assert hs[1][0, 0] == pytest.approx(d["h2"], abs=1e-15)
    p = _hand_params(d, 1)
    _, ts, _ = oracle.tmlp_trace(p, x)
    assert ts[1][0] == pytest.approx(d["t2_mult"], abs=1e-15)


def test_zero_params_give_zero():
    """all weights and biases zero -> y_i = 0 for every i (sin 0 = 0)."""
    p = _params(3, 8)
    for lst in (p.W, p.b, p.a):
        for arr in lst:
            arr[...] = 0
    p.c = [0.0] * 3
    x = np.random.default_rng(0).uniform(-1, 1, (50, 3)).astype(np.float32)
    _, ts, ys = oracle.tmlp_trace(p, x)
    assert np.all(ys == 0) and np.all(ts == 0)


@pytest.mark.parametrize("L,H", [(3, 8), (4, 64), (8, 32)])
def test_plain_siren_special_case_vs_torch_library(L, H):
    """Eq. 1 is Eq. 2 with tails 1..L-1 zero and tail L = (W^out, b^out): the oracle's
    y_L must equal a float64 SIREN built from torch.nn.functional.linear + torch.sin."""
    p = _params(L, H, omega0=30.0)
    for i in range(L - 1):
        p.a[i][...] = 0
        p.c[i] = 0.0
    x = np.random.default_rng(1).uniform(-1, 1, (257, 3)).astype(np.float32)
    y_or = oracle.query_full(p, x)
    h = torch.from_numpy(x.astype(np.float64))
    for i in range(L):
        h = torch.sin(30.0 * torch.nn.functional.linear(
            h, torch.from_numpy(p.W[i].astype(np.float64)), torch.from_numpy(p.b[i].astype(np.float64))))
    y_lib = torch.nn.functional.linear(h, torch.from_numpy(p.a[L - 1].astype(np.float64))[None, :],
                                       torch.tensor([p.c[L - 1]], dtype=torch.float64))[:, 0].numpy()
    np.testing.assert_allclose(y_or, y_lib, rtol=0, atol=1e-12)


def test_full_tmlp_vs_torch_sequential_all_tails():
    """Eq. 2 cumulative form vs a torch float64 module evaluation that sums every tail."""
    L, H = 5, 16
    p = _params(L, H)
    x = np.random.default_rng(2).uniform(-1, 1, (100, 3)).astype(np.float32)
    h = torch.from_numpy(x.astype(np.float64))
    y = torch.zeros(100, dtype=torch.float64)
    for i in range(L):
        lin = torch.nn.Linear(3 if i == 0 else H, H, dtype=torch.float64)
        tail = torch.nn.Linear(H, 1, dtype=torch.float64)
        with torch.no_grad():
            lin.weight.copy_(torch.from_numpy(p.W[i].astype(np.float64)))
            lin.bias.copy_(torch.from_numpy(p.b[i].astype(np.float64)))
            tail.weight.copy_(torch.from_numpy(p.a[i].astype(np.float64))[None])
            tail.bias.fill_(p.c[i])
            h = torch.sin(30.0 * lin(h))
            y = y + tail(h)[:, 0]
    np.testing.assert_allclose(oracle.query_full(p, x), y.numpy(), rtol=0, atol=1e-12)


@pytest.mark.parametrize("tail", [0, 1])
def test_prefix_consistency_and_truncation(tail):
    """Eq. 2: y_d - y_{d-1} = t_d and the depth-d output equals the full trace truncated at d
    (BJ north_star oracle check 1)."""
    L, H = 6, 24
    p = _params(L, H, tail=tail)
    x = np.random.default_rng(3).uniform(-1, 1, (200, 3)).astype(np.float32)
    _, ts, ys = oracle.tmlp_trace(p, x)
    prev = np.zeros(200)
    for d in range(1, L + 1):
        yd = oracle.tmlp_forward(p, x, d)
        np.testing.assert_array_equal(yd, ys[d - 1])
        np.testing.assert_array_equal(ys[d - 1] - prev, ts[d - 1]) if d == 1 else \
            np.testing.assert_allclose(ys[d - 1] - prev, ts[d - 1], rtol=0, atol=1e-15)
        prev = ys[d - 1]


@pytest.mark.parametrize("tail", [0, 1])
def test_nan_poisoning_of_unused_layers(tail):
    """SPEC S:184 depth-monotonic availability: forward at depth k never reads W_j, tails j > k."""
    L, H = 5, 16
    p = _params(L, H, tail=tail)
    x = np.random.default_rng(4).uniform(-1, 1, (64, 3)).astype(np.float32)
    for k in range(1, L + 1):
        q = _params(L, H, tail=tail)
        for j in range(k, L):
            q.W[j][...] = np.nan; q.b[j][...] = np.nan; q.a[j][...] = np.nan; q.c[j] = np.nan
            if tail == 1:
                q.a1[j - 1][...] = np.nan; q.c1[j - 1] = np.nan
        y = oracle.tmlp_forward(q, x, k)
        assert np.isfinite(y).all()
        np.testing.assert_array_equal(y, oracle.tmlp_forward(p, x, k))


def test_mixed_depths_equal_per_point():
    """Adaptive evaluation (Sec. 3.4) of a batch with mixed depths = per-point evaluation."""
    L, H = 6, 16
    p = _params(L, H)
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (300, 3)).astype(np.float32)
    d = rng.integers(1, L + 1, 300)
    y = oracle.tmlp_forward(p, x, d)
    for i in range(0, 300, 37):
        assert y[i] == pytest.approx(oracle.tmlp_forward(p, x[i:i + 1], d[i])[0], abs=1e-14)


def test_appendix_a_quadratic_form():
    """Appendix A: (a.h + c)(b.h + d) = h^T Q h + u^T h + s with Q = a b^T,
    u = d a + c b, s = c d; rank(Q) <= 1.  The oracle's MULT tail must equal the quadratic form."""
    L, H = 3, 32
    p = _params(L, H, tail=1)
    x = np.random.default_rng(6).uniform(-1, 1, (1000, 3)).astype(np.float32)
    hs, ts, _ = oracle.tmlp_trace(p, x)
    for i in (2, 3):
        a = p.a[i - 1].astype(np.float64); c = p.c[i - 1]
        b = p.a1[i - 2].astype(np.float64); dd = p.c1[i - 2]
        Q = np.outer(a, b); u = dd * a + c * b; s = c * dd
        h = hs[i - 1]
        quad = np.einsum("ni,ij,nj->n", h, Q, h) + h @ u + s
        np.testing.assert_allclose(ts[i - 1], quad, rtol=0, atol=1e-12)
        assert np.linalg.matrix_rank(Q) <= 1


def test_siren_init_bounds_and_moments():
    """SIREN init (BJ configs[0]): first layer |w| <= 1/3; hidden
    |w| <= sqrt(6/H)/30; empirical std within 10% of the uniform std bound/sqrt(3)."""
    for H in (64, 256):
        p = _params(8, H, omega0=30.0, seed=9)
        assert np.abs(p.W[0]).max() <= 1.0 / 3.0
        bnd = np.sqrt(6.0 / H) / 30.0
        for i in range(1, 8):
            assert np.abs(p.W[i]).max() <= np.float32(bnd)
        allh = np.concatenate([w.ravel() for w in p.W[1:]])
        assert abs(allh.std() / (bnd / np.sqrt(3.0)) - 1.0) < 0.10
        assert abs(allh.mean()) < 0.05 * bnd
        assert abs(p.W[0].std() / ((1 / 3) / np.sqrt(3.0)) - 1.0) < 0.10


def test_blob_roundtrip():
    for tail in (0, 1):
        p = _params(4, 16, tail=tail)
        blob = g.pack_blob(p)
        q = g.unpack_blob(blob, p.spec)
        np.testing.assert_array_equal(g.pack_blob(q), blob)
