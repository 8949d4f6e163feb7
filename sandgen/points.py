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
