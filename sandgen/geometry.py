"""Analytic sphere-union shapes standing in for the paper's meshes (BASELINE.json configs).

The paper's shapes (Stanford / Thingi32 meshes) and Open3D ground-truth SDF
 are not available; the configs use an analytic union of spheres instead.
SDF of a union: min_s (||p - c_s|| - r_s), evaluated in float64.
"""
from dataclasses import dataclass

import numpy as np

from .rng import uniform


@dataclass
class SphereSet:
    centres: np.ndarray  # [S][3] float64
    radii: np.ndarray    # [S] float64


def make_spheres(seed: int, n: int = 16, lo: float = -0.7, hi: float = 0.7,
                 rlo: float = 0.1, rhi: float = 0.3) -> SphereSet:
    """BJ configs[1]: 16 seeded spheres, centres U[-0.7,0.7]^3, radii U[0.1,0.3]."""
    c = uniform(seed, 1001, 3 * n, lo, hi).reshape(n, 3)
    r = uniform(seed, 1002, n, rlo, rhi)
    return SphereSet(c, r)


def single_sphere(radius: float = 0.5) -> SphereSet:
    """BJ configs[0]: analytic sphere of radius 0.5 at the origin."""
    return SphereSet(np.zeros((1, 3)), np.array([radius], np.float64))


def union_sdf(spheres: SphereSet, p: np.ndarray, chunk: int = 1 << 20) -> np.ndarray:
    """min_s ||p - c_s|| - r_s in float64; p is [...][3]."""
    p = np.asarray(p, np.float64)
    shp = p.shape[:-1]
    p = p.reshape(-1, 3)
    out = np.empty(p.shape[0], np.float64)
    for s0 in range(0, p.shape[0], chunk):
        q = p[s0:s0 + chunk]
        d = np.full(q.shape[0], np.inf)
        for c, r in zip(spheres.centres, spheres.radii):
            dd = np.sqrt(((q - c) ** 2).sum(axis=1)) - r
            np.minimum(d, dd, out=d)
        out[s0:s0 + chunk] = d
    return out.reshape(shp)
