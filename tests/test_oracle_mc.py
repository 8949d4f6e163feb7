"""Pins for the oracle's marching cubes (reading R24) on analytic SDFs
whose surfaces have known topology and area: the mesh of a closed surface must be watertight and
consistently oriented (every directed edge met once, its reverse once), its Euler characteristic must
be 2 per sphere and 0 for a torus, its normals must point to positive SDF, its area must approach the
analytic area, and every vertex must be a zero of the linear interpolant on its grid edge."""
import numpy as np
import pytest

import oracle
from oracle import sand_oracle as so


def _grid(R):
    ax = (2.0 * np.arange(R) / (R - 1) - 1.0).astype(np.float32).astype(np.float64)
    Z, Y, X = np.meshgrid(ax, ax, ax, indexing="ij")
    return X, Y, Z


def _topology(T):
    """(V, E, F, directed edges balanced?) of a triangle soup with exactly shared vertices."""
    keys = {}
    idx = np.array([[keys.setdefault(tuple(np.round(v, 12)), len(keys)) for v in tri] for tri in T])
    directed = {}
    for a, b, c in idx:
        for u, v in ((a, b), (b, c), (c, a)):
            directed[(u, v)] = directed.get((u, v), 0) + 1
    balanced = all(cnt == 1 and directed.get((v, u), 0) == 1 for (u, v), cnt in directed.items())
    E = len(directed) // 2
    return len(keys), E, len(idx), balanced


def test_case_table_properties():
    """Every configuration: each crossing edge is used exactly once over the loops; loops have >= 3
    edges; complementary single-corner cases give one triangle; at most 5 triangles per cube."""
    edges = so._mc_edges()
    for case in range(256):
        loops = so.mc_loops(case)
        used = sorted(e for l in loops for e in l)
        crossing = sorted(i for i, (a, b) in enumerate(edges) if ((case >> a) & 1) != ((case >> b) & 1))
        assert used == crossing, case
        assert all(len(l) >= 3 for l in loops)
        assert sum(len(l) - 2 for l in loops) <= 5
    for v in range(8):
        assert [len(l) for l in so.mc_loops(1 << v)] == [3]
        assert [len(l) for l in so.mc_loops(255 ^ (1 << v))] == [3]


@pytest.mark.parametrize("R", [17, 24])
def test_sphere_closed_oriented_genus0(R):
    X, Y, Z = _grid(R)
    sdf = np.sqrt(X ** 2 + Y ** 2 + Z ** 2) - 0.6
    T = oracle.marching_cubes(sdf.ravel(), R)
    V, E, F, bal = _topology(T)
    assert bal and V - E + F == 2
    n = np.cross(T[:, 1] - T[:, 0], T[:, 2] - T[:, 0])
    assert np.all(np.einsum("ij,ij->i", n, T.mean(1)) > 0)       # outward = toward sdf > 0


def test_two_spheres_and_torus_euler():
    X, Y, Z = _grid(25)
    two = np.minimum(np.sqrt((X - 0.45) ** 2 + Y ** 2 + Z ** 2), np.sqrt((X + 0.45) ** 2 + Y ** 2 + Z ** 2)) - 0.3
    V, E, F, bal = _topology(oracle.marching_cubes(two.ravel(), 25))
    assert bal and V - E + F == 4
    X, Y, Z = _grid(33)
    torus = np.sqrt((np.sqrt(X ** 2 + Y ** 2) - 0.55) ** 2 + Z ** 2) - 0.22
    V, E, F, bal = _topology(oracle.marching_cubes(torus.ravel(), 33))
    assert bal and V - E + F == 0


def test_area_converges_and_vertices_on_zero_set():
    areas = []
    for R in (17, 33):
        X, Y, Z = _grid(R)
        sdf = np.sqrt(X ** 2 + Y ** 2 + Z ** 2) - 0.7
        T = oracle.marching_cubes(sdf.ravel(), R)
        areas.append(0.5 * np.linalg.norm(np.cross(T[:, 1] - T[:, 0], T[:, 2] - T[:, 0]), axis=1).sum())
        # each vertex is where the linear interpolant of the (exactly radial) sdf along its edge is 0:
        # the radial sdf is not linear, so check |r - 0.7| is within the interpolation error h^2 / r
        h = 2.0 / (R - 1)
        assert np.abs(np.linalg.norm(T.reshape(-1, 3), axis=1) - 0.7).max() < h * h / 0.7
    exact = 4 * np.pi * 0.7 ** 2
    e17, e33 = abs(areas[0] - exact) / exact, abs(areas[1] - exact) / exact
    assert e33 < 0.02 and e33 < e17


def test_linear_field_gives_a_plane():
    """sdf = x - c (linear): every vertex has x = c exactly (to rounding) and the mesh is a flat
    grid-spanning sheet with normals along +x."""
    R = 9
    X, Y, Z = _grid(R)
    T = oracle.marching_cubes((X - 0.123).ravel(), R)
    assert np.abs(T[..., 0] - 0.123).max() < 1e-12
    n = np.cross(T[:, 1] - T[:, 0], T[:, 2] - T[:, 0])
    assert np.all(n[:, 0] > 0) and np.allclose(n[:, 1:], 0, atol=1e-12)
    assert len(T) == 2 * (R - 1) ** 2
