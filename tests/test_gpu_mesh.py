"""GPU parity for marching cubes (reading R24) through the C ABI:
sand_marching_cubes on analytic sdf grids against oracle.marching_cubes (same rule, independent code),
and the fused slab-by-slab extraction sand_mesh_grid against the unfused pipeline (sand_query on the
whole grid, then sand_marching_cubes) on the same weights and depth map.

The triangulation is unique under R24, so the triangle sets are compared exactly (vertex coordinates
within FP32 interpolation error); the output order is not (atomic placement), so triangles are sorted
canonically before comparing."""
import numpy as np
import pytest

import oracle
import sandgen as g
from _engine import make_ctx

pytestmark = pytest.mark.gpu


def _grid(R):
    ax = (2.0 * np.arange(R) / (R - 1) - 1.0).astype(np.float32).astype(np.float64)
    Z, Y, X = np.meshgrid(ax, ax, ax, indexing="ij")
    return X, Y, Z


def _canon(T, q=1e-4):
    """Sort triangles by their quantised vertex tuples (vertex order within a triangle kept: it is
    fixed by R24 up to the fan's start, which R24 also fixes)."""
    T = np.asarray(T, np.float64).reshape(-1, 9)
    key = np.round(T / q).astype(np.int64)
    return T[np.lexsort(key.T[::-1])]


def _gpu_mc(ctx, sdf_np, R):
    import torch
    s = torch.from_numpy(np.ascontiguousarray(sdf_np, np.float32)).cuda()
    n = ctx.sand_marching_cubes(s.data_ptr(), R, 0, 0)
    tris = torch.empty(max(n, 1) * 9, dtype=torch.float32, device="cuda")
    n2 = ctx.sand_marching_cubes(s.data_ptr(), R, tris.data_ptr(), n)
    assert n2 == n
    return tris[: 9 * n].cpu().numpy().reshape(-1, 3, 3)


def _watertight(T):
    keys = {}
    idx = [[keys.setdefault(tuple(v), len(keys)) for v in map(tuple, tri)] for tri in np.asarray(T, np.float32)]
    directed = {}
    for a, b, c in idx:
        for u, v in ((a, b), (b, c), (c, a)):
            directed[(u, v)] = directed.get((u, v), 0) + 1
    return all(n == 1 and directed.get((v, u), 0) == 1 for (u, v), n in directed.items()), len(keys), len(directed) // 2, len(idx)


@pytest.mark.parametrize("shape,R", [("sphere", 33), ("torus", 40), ("two", 29)])
def test_marching_cubes_matches_oracle(shape, R):
    X, Y, Z = _grid(R)
    if shape == "sphere":
        sdf = np.sqrt(X ** 2 + Y ** 2 + Z ** 2) - 0.61
    elif shape == "torus":
        sdf = np.sqrt((np.sqrt(X ** 2 + Y ** 2) - 0.55) ** 2 + Z ** 2) - 0.22
    else:
        sdf = np.minimum(np.sqrt((X - 0.45) ** 2 + Y ** 2 + Z ** 2), np.sqrt((X + 0.45) ** 2 + Y ** 2 + Z ** 2)) - 0.3
    sdf = sdf.astype(np.float32)
    spec = g.TMlpSpec(L=2, H=64, omega0=30.0, seed=1)
    with make_ctx(spec, 2) as ctx:
        T = _gpu_mc(ctx, sdf.ravel(), R)
    To = oracle.marching_cubes(sdf.ravel().astype(np.float64), R)
    assert T.shape == To.shape
    np.testing.assert_allclose(_canon(T), _canon(To), rtol=0, atol=2e-6)
    ok, V, E, F = _watertight(T)                      # bit-identical shared vertices on the GPU too
    assert ok and V - E + F == {"sphere": 2, "torus": 0, "two": 4}[shape]


@pytest.mark.parametrize("R", [131, 132])
def test_marching_cubes_across_sign_word_groups(R):
    """Grids wider than one 128-vertex sign-word group (csrc/mesh.cu): the surface crosses vertex columns 127 /
    128 (the x + 1 neighbour of a group's last vertex lives in the next group's first word) and leaves the domain
    through the x = +1 face (cubes end at column R - 2); R = 132 takes the 16-byte row loads, R = 131 the
    unaligned path.  Triangle set against oracle.marching_cubes, as above."""
    X, Y, Z = _grid(R)
    sdf = (np.sqrt((X - 0.6) ** 2 + (Y + 0.1) ** 2 + (Z - 0.05) ** 2) - 0.45).astype(np.float32)
    spec = g.TMlpSpec(L=2, H=64, omega0=30.0, seed=1)
    with make_ctx(spec, 2) as ctx:
        T = _gpu_mc(ctx, sdf.ravel(), R)
    To = oracle.marching_cubes(sdf.ravel().astype(np.float64), R)
    assert T.shape == To.shape and T.shape[0] > 10000
    np.testing.assert_allclose(_canon(T), _canon(To), rtol=0, atol=2e-6)
    assert T[:, :, 0].max() == 1.0   # the mesh reaches the domain face


def test_marching_cubes_large_grid_invariants_and_unaligned_buffer():
    """R = 260 (three sign-word groups per row, too large for the Python oracle in the default suite): properties
    that hold at any size -- two disjoint spheres inside the domain give a watertight mesh with Euler
    characteristic 2 + 2, every vertex lies on a grid edge with the sdf changing sign across it, and the same sdf
    read through a buffer that is NOT 16-byte aligned (the scalar load path of the sign pass) gives the same
    triangle set bit for bit."""
    import torch
    R = 260
    X, Y, Z = _grid(R)
    sdf = np.minimum(np.sqrt((X - 0.5) ** 2 + (Y - 0.1) ** 2 + Z ** 2) - 0.37,
                     np.sqrt((X + 0.55) ** 2 + (Y + 0.2) ** 2 + (Z - 0.3) ** 2) - 0.31).astype(np.float32)
    spec = g.TMlpSpec(L=2, H=64, omega0=30.0, seed=1)
    with make_ctx(spec, 2) as ctx:
        T = _gpu_mc(ctx, sdf.ravel(), R)
        buf = torch.empty(R ** 3 + 1, dtype=torch.float32, device="cuda")
        view = buf[1:]
        view.copy_(torch.from_numpy(sdf.ravel()))
        assert view.data_ptr() % 16 == 4
        n = ctx.sand_marching_cubes(view.data_ptr(), R, 0, 0)
        tris = torch.empty(n * 9, dtype=torch.float32, device="cuda")
        assert ctx.sand_marching_cubes(view.data_ptr(), R, tris.data_ptr(), n) == n
        Tu = tris.cpu().numpy().reshape(-1, 3, 3)
    assert T.shape == Tu.shape and T.shape[0] > 100000
    key = lambda A: A.reshape(-1, 9)[np.lexsort(A.reshape(-1, 9).T[::-1])]
    np.testing.assert_array_equal(key(T), key(Tu))
    ok, V, E, F = _watertight(T)
    assert ok and V - E + F == 4
    # every vertex sits on a grid line: two of its coordinates are grid coordinates
    ax = (2.0 * np.arange(R) / (R - 1) - 1.0).astype(np.float32)
    on_grid = np.isin(T.reshape(-1, 3), ax).sum(axis=1)
    assert (on_grid >= 2).all()


def test_capacity_and_empty():
    R = 21
    X, Y, Z = _grid(R)
    sdf = (np.sqrt(X ** 2 + Y ** 2 + Z ** 2) - 0.5).astype(np.float32).ravel()
    import torch
    spec = g.TMlpSpec(L=2, H=64, omega0=30.0, seed=1)
    with make_ctx(spec, 2) as ctx:
        s = torch.from_numpy(sdf).cuda()
        n = ctx.sand_marching_cubes(s.data_ptr(), R, 0, 0)
        guard = torch.full((9 * (n // 2) + 9,), 7.0, device="cuda")
        assert ctx.sand_marching_cubes(s.data_ptr(), R, guard.data_ptr(), n // 2) == n   # count, partial write
        assert torch.all(guard[9 * (n // 2):] == 7.0)                                  # nothing past cap
        pos = torch.ones(R ** 3, device="cuda")
        assert ctx.sand_marching_cubes(pos.data_ptr(), R, guard.data_ptr(), 1) == 0    # no surface


@pytest.mark.parametrize("slab", [0, 7, 64])
def test_fused_mesh_equals_unfused(slab):
    """sand_mesh_grid (slab-wise, device-generated grid points) == sand_query over the whole grid then
    sand_marching_cubes, exactly (same sdf values, same triangles)."""
    import torch
    c = g.make_config("C0")
    p = c.params()
    R = 65
    with make_ctx(c.spec, 0) as ctx:
        ctx.sand_load_weights(g.pack_blob(p))
        ctx.sand_load_depthmap(c.depthmap)
        pts = torch.from_numpy(g.grid_points(R)).cuda()
        sdf, _ = ctx.query_tensor(pts)
        torch.cuda.synchronize()
        n = ctx.sand_marching_cubes(sdf.data_ptr(), R, 0, 0)
        a = torch.empty(9 * n, device="cuda")
        ctx.sand_marching_cubes(sdf.data_ptr(), R, a.data_ptr(), n)
        m = ctx.sand_mesh_grid(R, slab, 0, 0)
        b = torch.empty(9 * max(m, 1), device="cuda")
        assert ctx.sand_mesh_grid(R, slab, b.data_ptr(), m) == m == n
        A, B = _canon(a.cpu().numpy()), _canon(b[: 9 * m].cpu().numpy())
        np.testing.assert_array_equal(A, B)
        assert n > 1000
        # the SIREN surface leaves the [-1, 1]^3 domain: every directed edge occurs once, and an edge
        # without its reverse must lie on the domain boundary
        Tv = B.reshape(-1, 3, 3).astype(np.float32)
        directed = {}
        for tri in Tv:
            vs = [tuple(v) for v in tri]
            for u, v in ((vs[0], vs[1]), (vs[1], vs[2]), (vs[2], vs[0])):
                directed[(u, v)] = directed.get((u, v), 0) + 1
        assert max(directed.values()) == 1
        on_face = lambda v: np.any(np.abs(np.abs(np.array(v)) - 1.0) < 1e-6)
        assert all(on_face(u) and on_face(v) for (u, v) in directed if (v, u) not in directed)


def test_edge_grids_match_oracle():
    """R = 2 (one cube) for every one of the 256 corner configurations, and a plane through grid vertices
    (sdf exactly 0 at vertices: strict 'inside iff sdf < 0')."""
    import torch
    spec = g.TMlpSpec(L=2, H=64, omega0=30.0, seed=1)
    with make_ctx(spec, 2) as ctx:
        vals = np.array([-0.75, 0.5], np.float32)
        for case in range(256):
            sdf = np.array([vals[(case >> v) & 1 ^ 1] for v in range(8)], np.float32)   # bit v set -> inside
            T = _gpu_mc(ctx, sdf, 2)
            To = oracle.marching_cubes(sdf.astype(np.float64), 2)
            assert T.shape == To.shape, case
            if len(T):
                np.testing.assert_allclose(_canon(T), _canon(To), rtol=0, atol=1e-6)
        R = 9
        X, Y, Z = _grid(R)
        sdf = (X - X[0, 0, 4]).astype(np.float32).ravel()     # zero exactly on the plane of vertex column 4
        T = _gpu_mc(ctx, sdf, R)
        To = oracle.marching_cubes(sdf.astype(np.float64), R)
        assert T.shape == To.shape
        np.testing.assert_allclose(_canon(T), _canon(To), rtol=0, atol=1e-6)


def test_fused_mesh_matches_oracle_mc_of_oracle_query():
    """The whole mesh pipeline against the oracle end to end: sand_mesh_grid on C0's
    T-MLP (FP32 path, grid R = 33, slabs of 8 cube planes) vs oracle.marching_cubes applied to the FP32 C
    oracle's SDF of the same grid.  Corner signs must agree wherever |sdf_oracle| exceeds the FP32 tolerance;
    then the triangle sets must match one to one, vertices within interpolation error."""
    import torch
    from scipy.spatial import cKDTree
    from oracle import fp32 as ofp
    c = g.make_config("C0")
    p = c.params()
    R = 33
    pts = g.grid_points(R)
    s_or, _ = ofp.query_fp32(p, c.depthmap, pts)
    T_or = oracle.marching_cubes(s_or.astype(np.float64), R).reshape(-1, 3, 3)
    with make_ctx(c.spec, 0) as ctx:
        ctx.sand_load_weights(g.pack_blob(p))
        ctx.sand_load_depthmap(c.depthmap)
        sdf, _ = ctx.query_tensor(torch.from_numpy(pts).cuda())
        m = ctx.sand_mesh_grid(R, 8, 0, 0)
        b = torch.empty(9 * max(m, 1), device="cuda")
        assert ctx.sand_mesh_grid(R, 8, b.data_ptr(), m) == m
        torch.cuda.synchronize()
        s_gpu = sdf.cpu().numpy()
        T_gpu = b[: 9 * m].cpu().numpy().reshape(-1, 3, 3).astype(np.float64)
    robust = np.abs(s_or) > 1e-4
    assert np.array_equal(np.sign(s_gpu[robust]), np.sign(s_or[robust]))
    flips = int((np.sign(s_gpu) != np.sign(s_or)).sum())
    assert flips == 0, f"{flips} near-zero corners changed sign: triangulations differ locally"
    assert m == T_or.shape[0] > 5000
    # R24 fixes each triangle's vertex order, so triangles are compared as points in R^9
    tree = cKDTree(T_or.reshape(-1, 9))
    _, j = tree.query(T_gpu.reshape(-1, 9))
    d = np.linalg.norm(T_gpu - T_or[j], axis=-1).max(axis=1)
    assert np.unique(j).size == m, "one-to-one triangle correspondence"
    assert d.max() <= 1e-3 and np.median(d) <= 1e-5, (d.max(), np.median(d))
