"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no T-MLP evaluation, no
depth-map lookup).  It only manufactures inputs: SIREN-init weights, analytic
sphere-union SDF depth maps (voxel and octree), and query point sets, following
the recipes in BASELINE.json ``configs`` and the readings listed in DESIGN.md
("Input recipe").  Both the oracle (``oracle/``) and the product path
(``paper_2604_25936_b200``) consume these arrays; neither imports the other.

Randomness is a counter-based splitmix64 generator (reading R7), so
every consumer can regenerate bit-identical inputs from ``(seed, stream, idx)``.
"""
from .rng import splitmix64, u01, uniform, normal
from .weights import TMlpSpec, make_weights, pack_blob, unpack_blob, blob_len
from .geometry import SphereSet, make_spheres, single_sphere, union_sdf
from .depthmaps import VoxelMap, Octree, build_voxel_map, build_octree, bands_depth
from .points import grid_axis, grid_points, cloud_points, grid_points_slab, leaf_samples
from .configs import CONFIGS, make_config

__all__ = [
    "splitmix64", "u01", "uniform", "normal",
    "TMlpSpec", "make_weights", "pack_blob", "unpack_blob", "blob_len",
    "SphereSet", "make_spheres", "single_sphere", "union_sdf",
    "VoxelMap", "Octree", "build_voxel_map", "build_octree", "bands_depth",
    "grid_axis", "grid_points", "cloud_points", "grid_points_slab", "leaf_samples",
    "CONFIGS", "make_config",
]
