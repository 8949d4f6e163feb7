"""Query point sets (BASELINE.json configs; readings R8, R13).

Grid: the R^3 uniform grid of vertex positions in [-1,1]^3 (the paper's marching-cubes evaluation
set): x_i = float32(2.0*i/(R-1) - 1.0) computed in float64, linear index
p = i + R*(j + R*k) (x fastest).  Points are float32 AoS [n][3].
"""
import numpy as np

from .geometry import SphereSet
from .rng import u01, normal


def grid_axis(R: int) -> np.ndarray:
    i = np.arange(R, dtype=np.float64)
    return (2.0 * i / (R - 1) - 1.0).astype(np.float32)


def grid_points_slab(R: int, k0: int, k1: int, Rz: int = None) -> np.ndarray:
    """Points of z-planes [k0, k1) of an R x R x Rz grid (Rz defaults to R), float32 [n][3]."""
    ax = grid_axis(R)
    az = ax if Rz is None else grid_axis(Rz)
    nz = k1 - k0
    out = np.empty((nz, R, R, 3), np.float32)
    out[..., 0] = ax[None, None, :]
    out[..., 1] = ax[None, :, None]
    out[..., 2] = az[k0:k1, None, None]
    return out.reshape(-1, 3)


def grid_points(R: int) -> np.ndarray:
    return grid_points_slab(R, 0, R)


def cloud_points(spheres: SphereSet, seed: int, n_uniform: int, n_near: int,
                 sigma: float = 0.01) -> np.ndarray:
    """BJ configs[3]: n_uniform points U[-1,1]^3 followed by n_near near-surface points
    c_s + r_s*u + N(0, sigma^2 I), s ~ U{0..S-1}, u uniform on S^2 (normalised Gaussian)."""
    uni = (2.0 * u01(seed, 2001, 3 * n_uniform) - 1.0).reshape(n_uniform, 3)
    S = spheres.radii.size
    s = np.minimum((u01(seed, 2002, n_near) * S).astype(np.int64), S - 1)
    g = normal(seed, 2003, 3 * n_near).reshape(n_near, 3)
    u = g / np.linalg.norm(g, axis=1, keepdims=True)
    eps = normal(seed, 2004, 3 * n_near).reshape(n_near, 3) * sigma
    near = spheres.centres[s] + spheres.radii[s, None] * u + eps
    return np.concatenate([uni, near], axis=0).astype(np.float32)


def leaf_samples(leaf_level, leaf_ijk, k: int, seed: int) -> np.ndarray:
    """Eq. 6 sample set of octree leaves (SPEC S:289 design decision; reading R21): per leaf,
    the 8 cell corners, the cell centre and k seeded interior points U[lo, hi)^3 (counter stream
    3001, counter = leaf * k * 3 + sample * 3 + axis).  Returns float32 [n_leaves, 9 + k, 3]."""
    lev = np.asarray(leaf_level, np.int64)
    ijk = np.asarray(leaf_ijk, np.int64).reshape(-1, 3)
    n = lev.size
    side = 2.0 / (2.0 ** lev)                          # float64
    lo = -1.0 + ijk * side[:, None]
    out = np.empty((n, 9 + k, 3), np.float64)
    for c in range(8):
        off = np.array([(c >> 0) & 1, (c >> 1) & 1, (c >> 2) & 1], np.float64)
        out[:, c, :] = lo + off[None, :] * side[:, None]
    out[:, 8, :] = lo + 0.5 * side[:, None]
    if k:
        cnt = (np.arange(n, dtype=np.uint64)[:, None, None] * np.uint64(3 * k)
               + np.arange(k, dtype=np.uint64)[None, :, None] * np.uint64(3)
               + np.arange(3, dtype=np.uint64)[None, None, :])
        u = u01(seed, 3001, cnt.reshape(-1)).reshape(n, k, 3)
        out[:, 9:, :] = lo[:, None, :] + u * side[:, None, None]
    return out.astype(np.float32)
