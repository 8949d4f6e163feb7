"""Pins for the oracle's depth-map lookup and adaptive query (Sec. 3.2, 3.4; Eq. 7)."""
from math import gcd

import numpy as np
import pytest

import oracle
import sandgen as g


def _tiny_octree(level=3, far_band=False, seed=5):
    sph = g.make_spheres(seed, n=3, rlo=0.2, rhi=0.4)
    return g.build_octree(sph, level, g.configs.BANDS_8, 8, score_seed=3, far_band=far_band)


def _adversarial_points(level, n_rand=10000, seed=0):
    rng = np.random.default_rng(seed)
    pts = [rng.uniform(-1, 1, (n_rand, 3))]
    faces = -1.0 + np.arange((1 << level) + 1) * (2.0 / (1 << level))   # every cell face
    f = rng.choice(faces, (4000, 3))
    mix = rng.uniform(-1, 1, (4000, 3))
    m = rng.integers(0, 2, (4000, 3)).astype(bool)
    pts.append(np.where(m, f, mix))
    pts.append(rng.uniform(-1.5, 1.5, (1000, 3)))        # outside the domain -> boundary clamp
    pts.append(np.array([[1, 1, 1], [-1, -1, -1], [1, -1, 1], [0, 0, 0]], np.float64))
    return np.concatenate(pts).astype(np.float32)


@pytest.mark.parametrize("level", [1, 2, 3, 4])
def test_octree_descent_equals_bruteforce_leaf_scan(level):
    """SPEC S:317 / S:608: traversal lookup equals brute-force linear scan over the leaf list at
    10^4 random points plus points on every cell face (half-open [lo,hi)) and outside."""
    oc = _tiny_octree(level, far_band=True)
    pts = _adversarial_points(level)
    d1, f1, l1 = oracle.lookup_octree(oc.level, oc.nodes, oc.leaf_depth, oc.leaf_far_sdf, pts)
    d2, f2, l2 = oracle.lookup_bruteforce(oc.leaf_level, oc.leaf_ijk, oc.leaf_depth, oc.leaf_far_sdf, pts)
    np.testing.assert_array_equal(l1, l2)
    np.testing.assert_array_equal(d1, d2)
    np.testing.assert_array_equal(f1, f2)


def test_leaves_tile_the_domain():
    """the union of leaf cells tiles [-1,1]^3 exactly (volumes sum to 8, disjoint by
    the brute-force scan's 'exactly one owner' assertion above)."""
    oc = _tiny_octree(4)
    vol = ((2.0 / 2.0 ** oc.leaf_level.astype(np.float64)) ** 3).sum()
    assert vol == pytest.approx(8.0, abs=1e-12)


@pytest.mark.parametrize("level,R", [(5, 64), (7, 256), (7, 512)])
def test_grid_point_cells_closed_form(level, R):
    """For the R^3 vertex grid and G = 2^level with gcd(G, R-1) = 1 (BJ configs), the float32 cell
    of coordinate i is floor(G*i/(R-1)) (integer arithmetic), clamped to G-1 at x = +1 (DESIGN.md
    reading R15): no grid point lies within float32 rounding of a cell face."""
    G = 1 << level
    assert gcd(G, R - 1) == 1
    ax = g.grid_axis(R)
    pts = np.stack([ax, ax[::-1], ax], axis=1)
    c = oracle.cell_coords(pts, level)
    i = np.arange(R)
    ref = np.minimum(G * i // (R - 1), G - 1)
    np.testing.assert_array_equal(c[:, 0], ref)
    np.testing.assert_array_equal(c[:, 1], ref[::-1])


def test_octree_descent_equals_painted_leaf_grid():
    """Descent at the max level equals a dense grid painted leaf-by-leaf from the leaf list (an
    independent formulation of 'the leaf containing x'), on C2-like trees at 2^18 points."""
    oc = g.build_octree(g.make_spheres(7), 6, g.configs.BANDS_8, 8, score_seed=11)
    G = 1 << oc.level
    grid = np.full((G, G, G), -1, np.int64)          # [z][y][x]
    for li in range(oc.n_leaves):
        s = 1 << (oc.level - oc.leaf_level[li])
        i, j, k = oc.leaf_ijk[li] * s
        grid[k:k + s, j:j + s, i:i + s] = li
    assert (grid >= 0).all()
    pts = np.random.default_rng(1).uniform(-1, 1, (1 << 18, 3)).astype(np.float32)
    _, _, leaf = oracle.lookup_octree(oc.level, oc.nodes, oc.leaf_depth, None, pts)
    c = oracle.cell_coords(pts, oc.level)
    np.testing.assert_array_equal(leaf, grid[c[:, 2], c[:, 1], c[:, 0]])


def _small_net(L=4, H=16):
    return g.make_weights(g.TMlpSpec(L=L, H=H, omega0=30.0, seed=2))


def test_query_all_far_zero_passes():
    """SPEC S:371 / Eq. 7: all points in far leaves -> cached SDF, no network evaluation
    (NaN-poisoned weights must not matter)."""
    p = _small_net()
    for lst in (p.W, p.b, p.a):
        for arr in lst:
            arr[...] = np.nan
    vm = g.VoxelMap(3, np.zeros(512, np.uint8), np.linspace(-1, 1, 512).astype(np.float32))
    pts = np.random.default_rng(0).uniform(-1, 1, (1000, 3)).astype(np.float32)
    sdf, ed = oracle.query(p, vm, pts)
    assert (ed == 0).all()
    c = oracle.cell_coords(pts, 3)
    np.testing.assert_array_equal(sdf, vm.far_sdf[c[:, 0] + 8 * (c[:, 1] + 8 * c[:, 2])].astype(np.float64))


def test_query_all_max_depth_equals_full_and_cap_noop():
    """BJ oracle check 2 / SPEC S:372: an all-L map reproduces the full-depth T-MLP;
    cap = L is a no-op; LOD nesting; conservation."""
    L = 4
    p = _small_net(L)
    vm = g.VoxelMap(3, np.full(512, L, np.uint8), None)
    pts = np.random.default_rng(1).uniform(-1, 1, (2000, 3)).astype(np.float32)
    sdf, ed = oracle.query(p, vm, pts)
    np.testing.assert_array_equal(sdf, oracle.query_full(p, pts))
    sdf2, ed2 = oracle.query(p, vm, pts, lod_cap=L)
    np.testing.assert_array_equal(sdf2, sdf)
    rng = np.random.default_rng(2)
    vm2 = g.VoxelMap(3, rng.integers(0, L + 1, 512).astype(np.uint8), rng.normal(size=512).astype(np.float32))
    prev = None
    for cap in range(1, L + 1):
        _, e = oracle.query(p, vm2, pts, lod_cap=cap)
        assert np.bincount(e, minlength=L + 1).sum() == len(pts)
        if prev is not None:
            assert (prev <= e).all()
        prev = e


def test_query_nonfinite_points():
    p = _small_net()
    vm = g.VoxelMap(3, np.full(512, 2, np.uint8), None)
    pts = np.array([[np.nan, 0, 0], [0, np.inf, 0], [0.1, 0.2, 0.3]], np.float32)
    sdf, ed = oracle.query(p, vm, pts)
    assert ed.tolist() == [255, 255, 2]
    assert np.isnan(sdf[:2]).all() and np.isfinite(sdf[2])


def test_config_depth_mix_matches_recipe():
    """The C0 recipe (BJ configs[0]): depth 4 iff |d(centre)| < 0.05 etc.; bands are monotone in
    distance; all depths in 1..4."""
    c = g.make_config("C0")
    dm = c.depthmap
    G = dm.G
    ax = -1.0 + (np.arange(G) + 0.5) * (2.0 / G)
    zz, yy, xx = np.meshgrid(ax, ax, ax, indexing="ij")
    r = np.abs(np.sqrt(xx ** 2 + yy ** 2 + zz ** 2) - 0.5).ravel()
    exp = np.where(r < 0.05, 4, np.where(r < 0.15, 3, np.where(r < 0.4, 2, 1)))
    np.testing.assert_array_equal(dm.depth, exp)
