"""Synthetic volumetric network-depth maps (voxel grid and octree).

These stand in for the paper's trained depth maps (Eq. 5-7), which need a
trained T-MLP and a mesh.  The recipe is BASELINE.json's:

* voxel grid (configs[0], [1]): G = 2^level cells per axis over [-1,1]^3, x-fastest; the depth of a
  cell is a distance band of the union SDF at the cell centre (strict '<').
* octree (configs[2]-[4]): root = level 0 = [-1,1]^3; a cell at level l < max_level is subdivided iff
  |sdf(centre)| < cell diagonal (BJ rule, reading R10); leaf depth = band(|sdf(leaf centre)|) + 1 if a
  seeded per-leaf score U[0,1) > 0.7, capped at L (reading R11).
* far-field option (reading R18): cells/leaves whose band depth would be 1 become depth 0 (Eq. 7
  "far" leaves) with the analytic SDF at the centre cached as float32.

Node encoding (include/sand.h, sand_depthmap): nodes[i] has bit31 = 1 for a leaf (low 31 bits = leaf
index) else the index of the first of 8 contiguous children, octant = xbit | ybit<<1 | zbit<<2.
"""
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .geometry import SphereSet, union_sdf
from .rng import splitmix64

LEAF_BIT = np.uint32(1 << 31)


def bands_depth(absd: np.ndarray, thresholds: Sequence[float]) -> np.ndarray:
    """depth = 1 + #{t : |d| < t}  (C1/C2: {.005,...,.32} -> 8..1; C0: {.05,.15,.4} -> 4..1)."""
    d = np.ones(absd.shape, np.int32)
    for t in thresholds:
        d += (absd < t).astype(np.int32)
    return d


@dataclass
class VoxelMap:
    level: int
    depth: np.ndarray              # [G^3] uint8, x-fastest
    far_sdf: Optional[np.ndarray]  # [G^3] float32 or None

    @property
    def G(self):
        return 1 << self.level


@dataclass
class Octree:
    level: int                     # max level (root = 0)
    nodes: np.ndarray              # [n_nodes] uint32
    leaf_depth: np.ndarray         # [n_leaves] uint8
    leaf_far_sdf: Optional[np.ndarray]  # [n_leaves] float32 or None
    leaf_level: np.ndarray         # [n_leaves] int32   (for brute-force scans / tests)
    leaf_ijk: np.ndarray           # [n_leaves][3] int64 cell coords at leaf_level

    @property
    def n_nodes(self):
        return int(self.nodes.size)

    @property
    def n_leaves(self):
        return int(self.leaf_depth.size)


def _centres(level: int, ijk: np.ndarray) -> np.ndarray:
    side = 2.0 / (1 << level)
    return -1.0 + (ijk.astype(np.float64) + 0.5) * side


def build_voxel_map(spheres: SphereSet, level: int, thresholds: Sequence[float],
                    far_band: bool = False) -> VoxelMap:
    G = 1 << level
    ax = -1.0 + (np.arange(G, dtype=np.float64) + 0.5) * (2.0 / G)
    zz, yy, xx = np.meshgrid(ax, ax, ax, indexing="ij")  # x fastest in C order
    p = np.stack([xx, yy, zz], axis=-1).reshape(-1, 3)
    sd = union_sdf(spheres, p)
    dep = bands_depth(np.abs(sd), thresholds)
    far = None
    if far_band:
        isfar = dep == 1
        dep = np.where(isfar, 0, dep)
        far = np.where(isfar, sd, 0.0).astype(np.float32)
    return VoxelMap(level, dep.astype(np.uint8), far)


def _morton3(ijk: np.ndarray) -> np.ndarray:
    """Interleave the low 20 bits of (i, j, k) -> 60-bit key (x in bit 0)."""
    out = np.zeros(ijk.shape[0], np.uint64)
    for b in range(20):
        for a in range(3):
            bit = (ijk[:, a].astype(np.uint64) >> np.uint64(b)) & np.uint64(1)
            out |= bit << np.uint64(3 * b + a)
    return out


def leaf_scores(seed: int, level: np.ndarray, ijk: np.ndarray) -> np.ndarray:
    """Per-leaf complexity score U[0,1) = U01(splitmix64(seed ^ (level<<60 | morton(ijk))))."""
    key = (level.astype(np.uint64) << np.uint64(60)) | _morton3(ijk)
    with np.errstate(over="ignore"):
        u = splitmix64(np.uint64(seed) ^ key)
    return (u >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def build_octree(spheres: SphereSet, max_level: int, thresholds: Sequence[float], L: int,
                 score_seed: Optional[int] = None, score_threshold: float = 0.7,
                 far_band: bool = False, subdivide_factor: float = 1.0) -> Octree:
    """Breadth-first octree build; node 0 is the root.

    subdivide iff level < max_level and |sdf(centre)| < subdivide_factor * diagonal.
    """
    nodes = [np.zeros(1, np.uint32)]  # per-level node payloads, concatenated at the end
    level_ijk = np.zeros((1, 3), np.int64)
    first_id = 0              # node id of the first node at the current level
    next_id = 1               # next free node id
    leaf_level, leaf_ijk, leaf_sd = [], [], []
    n_leaves = 0
    payload_levels = []
    for lev in range(max_level + 1):
        n = level_ijk.shape[0]
        sd = union_sdf(spheres, _centres(lev, level_ijk))
        diag = (2.0 / (1 << lev)) * np.sqrt(3.0)
        sub = (np.abs(sd) < subdivide_factor * diag) if lev < max_level else np.zeros(n, bool)
        payload = np.zeros(n, np.uint32)
        # leaves, in node order
        lf = ~sub
        nl = int(lf.sum())
        payload[lf] = LEAF_BIT | (np.arange(n_leaves, n_leaves + nl, dtype=np.uint32))
        n_leaves += nl
        leaf_level.append(np.full(nl, lev, np.int32))
        leaf_ijk.append(level_ijk[lf])
        leaf_sd.append(sd[lf])
        # children, 8 contiguous per subdivided node in node order
        ns = int(sub.sum())
        payload[sub] = (next_id + 8 * np.arange(ns, dtype=np.int64)).astype(np.uint32)
        payload_levels.append(payload)
        par = level_ijk[sub]
        ch = np.empty((ns, 8, 3), np.int64)
        for o in range(8):
            ch[:, o, 0] = 2 * par[:, 0] + (o & 1)
            ch[:, o, 1] = 2 * par[:, 1] + ((o >> 1) & 1)
            ch[:, o, 2] = 2 * par[:, 2] + ((o >> 2) & 1)
        first_id = next_id
        next_id += 8 * ns
        level_ijk = ch.reshape(-1, 3)
        if ns == 0:
            break
    nodes = np.concatenate(payload_levels).astype(np.uint32)
    assert nodes.size == next_id
    leaf_level = np.concatenate(leaf_level)
    leaf_ijk = np.concatenate(leaf_ijk, axis=0)
    leaf_sd = np.concatenate(leaf_sd)
    dep = bands_depth(np.abs(leaf_sd), thresholds)
    if score_seed is not None:
        sc = leaf_scores(score_seed, leaf_level, leaf_ijk)
        dep = dep + (sc > score_threshold).astype(np.int32)
    dep = np.minimum(dep, L)
    far = None
    if far_band:
        isfar = bands_depth(np.abs(leaf_sd), thresholds) == 1
        dep = np.where(isfar, 0, dep)
        far = np.where(isfar, leaf_sd, 0.0).astype(np.float32)
    return Octree(max_level, nodes, dep.astype(np.uint8), far, leaf_level, leaf_ijk)
