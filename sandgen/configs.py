"""BASELINE.json configs[0..4] as concrete seeded inputs.

C0: T-MLP 4x64, w0=30, FP32; 32^3 voxel map of a radius-0.5 sphere, bands {0.05,0.15,0.4} -> 4..1;
    queries = 64^3 grid.
C1: T-MLP 8x256, BF16; 128^3 voxel map of a 16-sphere union, bands {.005,...,.32} -> 8..1;
    queries = 256^3 grid.
C2: same net; octree to level 7 (subdivide iff |d| < diagonal), leaf bands + 1 if score > 0.7
    (cap 8); queries = 512^3 grid (the marching-cubes set of PAPER.md P:415/P:423).
C3: T-MLP 8x336, BF16; C2's octree; 2^22 uniform + 2^22 near-surface points.
C4: 8x256 BF16; C2's octree extended to level 8; queries = 1024^3 grid (z-slab sharded).
"""
from dataclasses import dataclass
from typing import Callable, Optional, Union

import numpy as np

from .depthmaps import Octree, VoxelMap, build_octree, build_voxel_map
from .geometry import make_spheres, single_sphere
from .points import cloud_points, grid_points_slab
from .weights import LINEAR, TMlpSpec, make_weights

WEIGHT_SEED = 1
SPHERE_SEED = 7
SCORE_SEED = 11
CLOUD_SEED = 13

BANDS_C0 = (0.05, 0.15, 0.4)
BANDS_8 = (0.005, 0.01, 0.02, 0.04, 0.08, 0.16, 0.32)

# precision codes (include/sand.h sand_precision)
FP32 = 0
BF16 = 2


@dataclass
class Config:
    name: str
    spec: TMlpSpec
    precision: int
    depthmap: Union[VoxelMap, Octree]
    n_points: int
    grid_R: Optional[int]                     # None for clouds
    points_fn: Callable[..., np.ndarray]      # points_fn() -> all points; grid: points_fn(k0, k1)
    description: str

    def params(self):
        return make_weights(self.spec)


CONFIGS = ("C0", "C1", "C2", "C3", "C4")


def make_config(name: str, tail: int = LINEAR, far_band: bool = False,
                weight_seed: int = WEIGHT_SEED) -> Config:
    if name == "C0":
        spec = TMlpSpec(L=4, H=64, omega0=30.0, tail=tail, seed=weight_seed)
        dm = build_voxel_map(single_sphere(0.5), 5, BANDS_C0, far_band=far_band)
        R = 64
        return Config(name, spec, FP32, dm, R ** 3, R,
                      lambda k0=0, k1=R: grid_points_slab(R, k0, k1),
                      "4x64 SIREN T-MLP FP32, 32^3 voxel sphere map, 64^3 grid")
    spheres = make_spheres(SPHERE_SEED)
    if name == "C1":
        spec = TMlpSpec(L=8, H=256, omega0=30.0, tail=tail, seed=weight_seed)
        dm = build_voxel_map(spheres, 7, BANDS_8, far_band=far_band)
        R = 256
        return Config(name, spec, BF16, dm, R ** 3, R,
                      lambda k0=0, k1=R: grid_points_slab(R, k0, k1),
                      "8x256 SIREN T-MLP BF16, 128^3 voxel 16-sphere map, 256^3 grid")
    if name in ("C2", "C3", "C4"):
        lev = 8 if name == "C4" else 7
        H = 336 if name == "C3" else 256
        spec = TMlpSpec(L=8, H=H, omega0=30.0, tail=tail, seed=weight_seed)
        dm = build_octree(spheres, lev, BANDS_8, spec.L, score_seed=SCORE_SEED, far_band=far_band)
        if name == "C3":
            n = 1 << 23
            return Config(name, spec, BF16, dm, n, None,
                          lambda: cloud_points(spheres, CLOUD_SEED, 1 << 22, 1 << 22),
                          "8x336 SIREN T-MLP BF16, level-7 octree, 8M mixed cloud")
        R = 1024 if name == "C4" else 512
        return Config(name, spec, BF16, dm, R ** 3, R,
                      lambda k0=0, k1=R: grid_points_slab(R, k0, k1),
                      f"8x256 SIREN T-MLP BF16, level-{lev} octree, {R}^3 grid")
    raise ValueError(name)
