"""Pins for the plain FP32 C oracle (oracle/sand_oracle_fp32.c, the oracle BASELINE.json's north star
names) against things other than itself: the float64 numpy oracle (itself pinned by
test_oracle_tmlp.py / test_oracle_lookup.py), hand-computed values, the Appendix-A closed form, a
brute-force leaf scan and the integer closed form of grid-point cells.  All CPU-only.

The FP32 oracle must agree with the float64 one to <= 1e-5 max-abs on the SDF (float32 rounding of
sequential sums of at most 256 terms and of sinf) and bit-exactly on every exit depth (both decide the
cell in float32, reading R1).
"""
import json
import os
from math import gcd
from types import SimpleNamespace

import numpy as np
import pytest

import oracle
import sandgen as g
from oracle import fp32 as of

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-5


def _tiny_octree(level=3, far_band=False, seed=5):
    sph = g.make_spheres(seed, n=3, rlo=0.2, rhi=0.4)
    return g.build_octree(sph, level, g.configs.BANDS_8, 8, score_seed=3, far_band=far_band)


def _pts(n, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, (n, 3)).astype(np.float32)


def _compare(p, dm, pts, cap=None, tol=TOL):
    s64, d64 = oracle.query(p, dm, pts, lod_cap=cap)
    s32, d32 = of.query_fp32(p, dm, pts, lod_cap=cap)
    np.testing.assert_array_equal(d32, d64)
    fin = np.isfinite(s64)
    np.testing.assert_array_equal(np.isfinite(s32), fin)
    err = np.abs(s32[fin].astype(np.float64) - s64[fin]).max() if fin.any() else 0.0
    assert err <= tol, f"FP32 oracle vs float64 oracle: max-abs {err:.3e} > {tol}"
    return err


def test_builds_with_strict_fp_flags():
    """The oracle is compiled with -ffp-contract=off (no FMA contraction) and OpenMP."""
    assert "-ffp-contract=off" in of.CFLAGS and "-fopenmp" in of.CFLAGS
    of.build()
    assert os.path.exists(of.LIB)
    assert of.threads() >= 1


def test_hand_computed_L2_H1():
    """SPEC S:142 / Eq. 2-3 pencil-and-paper values (tests/golden/hand_L2_H1.json), in float32."""
    d = json.load(open(os.path.join(GOLD, "hand_L2_H1.json")))
    x = np.array([d["x"]], np.float32)
    for tail, key in ((0, "y2_linear"), (1, "y2_mult")):
        spec = SimpleNamespace(L=2, H=1, omega0=d["omega0"], tail=tail)
        f = lambda v: np.array(v, np.float32)
        p = SimpleNamespace(spec=spec, W=[f(d["W1"]), f(d["W2"])], b=[f(d["b1"]), f(d["b2"])],
                            a=[f(d["a1"]), f(d["a2"])], c=[d["c1"], d["c2"]], a1=[f(d["a21"])], c1=[d["c21"]])
        for depth, want in ((1, d["y1"]), (2, d[key])):
            dm = g.VoxelMap(0, np.array([depth], np.uint8), None)
            s, e = of.query_fp32(p, dm, x)
            assert e[0] == depth
            assert float(s[0]) == pytest.approx(want, abs=2e-6)


def test_appendix_a_closed_form_mult_tail():
    """Eq. 3 / Appendix A: with W_2 = 0 the layer-2 features are constants h_j = sin(w0 b_j),
    and the multiplicative tail t_2 = (a0.h + c0)(a1.h + c1) = h^T Q h + u^T h + s with Q = a0 a1^T,
    u = c1 a0 + c0 a1, s = c0 c1 (computed here in float64 from the constants)."""
    H = 16
    spec = g.TMlpSpec(L=2, H=H, omega0=30.0, tail=1, seed=9)
    p = g.make_weights(spec)
    p.W[1][...] = 0
    pts = _pts(500, 4)
    dm1 = g.VoxelMap(0, np.array([1], np.uint8), None)
    dm2 = g.VoxelMap(0, np.array([2], np.uint8), None)
    y1, _ = of.query_fp32(p, dm1, pts)
    y2, _ = of.query_fp32(p, dm2, pts)
    h = np.sin(30.0 * p.b[1].astype(np.float64))
    a0, a1 = p.a[1].astype(np.float64), p.a1[0].astype(np.float64)
    c0, c1 = float(p.c[1]), float(p.c1[0])
    t2 = h @ np.outer(a0, a1) @ h + (c1 * a0 + c0 * a1) @ h + c0 * c1
    np.testing.assert_allclose(y2.astype(np.float64) - y1.astype(np.float64), t2, rtol=0, atol=2e-6)


@pytest.mark.parametrize("level", [1, 2, 3, 4])
def test_octree_exit_depth_equals_bruteforce_leaf_scan(level):
    """the FP32 oracle's descent gives the depth / cached SDF of the leaf a brute-force scan
    over the serialized leaf list finds, at random, cell-face and out-of-domain points."""
    oc = _tiny_octree(level, far_band=True)
    rng = np.random.default_rng(level)
    faces = -1.0 + np.arange((1 << level) + 1) * (2.0 / (1 << level))
    pts = np.concatenate([rng.uniform(-1, 1, (3000, 3)), rng.choice(faces, (1000, 3)),
                          rng.uniform(-1.5, 1.5, (500, 3))]).astype(np.float32)
    d_bf, f_bf, _ = oracle.lookup_bruteforce(oc.leaf_level, oc.leaf_ijk, oc.leaf_depth, oc.leaf_far_sdf, pts)
    p = g.make_weights(g.TMlpSpec(L=8, H=16, omega0=30.0, seed=2))
    s, d = of.query_fp32(p, oc, pts)
    np.testing.assert_array_equal(d, d_bf)
    far = d == 0
    np.testing.assert_array_equal(s[far], f_bf[far])


@pytest.mark.parametrize("level,R", [(5, 64), (7, 256)])
def test_grid_point_exit_depths_closed_form(level, R):
    """Grid queries (reading R15): the FP32 oracle's exit depth of vertex (i, j, k) is the voxel payload at
    integer cell (floor(G i/(R-1)), ...), clamped to G-1 -- integer arithmetic only."""
    G = 1 << level
    assert gcd(G, R - 1) == 1
    depth = np.random.default_rng(level).integers(1, 5, G ** 3).astype(np.uint8)
    dm = g.VoxelMap(level, depth, None)
    ax = g.grid_axis(R)
    rng = np.random.default_rng(R)
    ijk = rng.integers(0, R, (4000, 3))
    pts = np.stack([ax[ijk[:, 0]], ax[ijk[:, 1]], ax[ijk[:, 2]]], 1)
    p = g.make_weights(g.TMlpSpec(L=4, H=16, omega0=30.0, seed=3))
    _, d = of.query_fp32(p, dm, pts)
    c = np.minimum(G * ijk // (R - 1), G - 1)
    np.testing.assert_array_equal(d, depth[c[:, 0] + G * (c[:, 1] + G * c[:, 2])])


@pytest.mark.parametrize("H,L,tail", [(16, 1, 0), (64, 4, 0), (64, 4, 1), (256, 8, 0), (256, 8, 1), (336, 3, 0)])
def test_matches_float64_oracle_random_depths(H, L, tail):
    """Random depth mixes 1..L with ragged counts, voxel map: FP32 vs float64 <= 1e-5, depths bit-exact."""
    p = g.make_weights(g.TMlpSpec(L=L, H=H, omega0=30.0, tail=tail, seed=5 + H + L))
    dm = g.VoxelMap(3, np.random.default_rng(H).integers(1, L + 1, 512).astype(np.uint8), None)
    _compare(p, dm, _pts(3001 if H < 256 else 1201, H))


def test_matches_float64_oracle_octree_far_cap_nonfinite():
    """C2-style octree with a far band (cached SDF, Eq. 7), LOD caps, out-of-domain and non-finite points."""
    oc = g.build_octree(g.make_spheres(7), 5, g.configs.BANDS_8, 8, score_seed=11, far_band=True)
    p = g.make_weights(g.TMlpSpec(L=8, H=64, omega0=30.0, seed=1))
    pts = np.concatenate([_pts(4000, 1), _pts(300, 2, -1.4, 1.4)])
    pts[5] = [np.nan, 0, 0]
    pts[9] = [0, -np.inf, 0]
    for cap in (None, 1, 3, 8):
        _compare(p, oc, pts, cap=cap)
    s, d = of.query_fp32(p, oc, pts)
    assert d[5] == 255 and d[9] == 255 and np.isnan(s[5]) and np.isnan(s[9])
    for cap in (None, 2):   # the lookup-only entry point gives the same depths as the full query
        np.testing.assert_array_equal(of.lookup_fp32(oc, pts, lod_cap=cap), oracle.query(p, oc, pts, lod_cap=cap)[1])
    assert (d == 0).any(), "the far band must produce depth-0 points"


def test_nan_poisoned_unused_layers_leave_output_finite():
    """layers beyond a point's exit depth are never evaluated (NaN weights there do not leak)."""
    p = g.make_weights(g.TMlpSpec(L=5, H=32, omega0=30.0, seed=6))
    for i in (3, 4):
        p.W[i][...] = np.nan
        p.b[i][...] = np.nan
    dm = g.VoxelMap(2, np.random.default_rng(1).integers(1, 4, 64).astype(np.uint8), None)
    s, d = of.query_fp32(p, dm, _pts(1000, 3))
    assert d.max() == 3 and np.isfinite(s).all()
