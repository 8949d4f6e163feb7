"""Multi-GPU host logic: work-balanced z-slab sharding of a marching-cubes grid and the per-rank
record exchanged after a query.

Points are independent (Sec. 3.4), so ranks share nothing but the (replicated) weights and
depth map.  A rank's shard is a contiguous range of z-planes [k0, k1) of an R x R x Rz grid; with
x-fastest indexing that is a contiguous index range, so each rank generates its own points.  The
cut positions equalise *estimated work* (not plane counts): the depth mix varies strongly with z
(equal-thickness slabs are 1.35-1.54x imbalanced at 8 GPUs on C2-like maps).

The work model is the fused kernel's: a point of exit depth d costs d epilogue passes (sin + tail
per hidden unit, the bound pipe) plus (d - 1) H x H MMAs overlapping them, i.e. cost(d) ~ d + eps.
"""
import numpy as np


def dense_depth_grid(depthmap):
    """u8 [G][G][G] (z, y, x) depth grid at the map's level (octree leaves painted)."""
    if not hasattr(depthmap, "nodes"):
        G = 1 << depthmap.level
        return np.asarray(depthmap.depth, np.uint8).reshape(G, G, G)
    lev = depthmap.level
    G = 1 << lev
    grid = np.zeros((G, G, G), np.uint8)
    for L_ in np.unique(depthmap.leaf_level):
        sel = np.nonzero(depthmap.leaf_level == L_)[0]
        s = 1 << (lev - int(L_))
        ijk = depthmap.leaf_ijk[sel] * s
        dep = depthmap.leaf_depth[sel]
        if s == 1:
            grid[ijk[:, 2], ijk[:, 1], ijk[:, 0]] = dep
        else:
            for n in range(sel.size):
                i, j, k = ijk[n]
                grid[k:k + s, j:j + s, i:i + s] = dep[n]
    return grid


def _cells_of_axis(R, G):
    x = (2.0 * np.arange(R) / (R - 1) - 1.0).astype(np.float32).astype(np.float64)
    return np.clip(np.floor((x + 1.0) * (G / 2.0)), 0, G - 1).astype(np.int64)


def plane_work(depthmap, R, Rz, eps=0.5):
    """Estimated work of each of the Rz z-planes of an R x R x Rz vertex grid over [-1,1]^3."""
    dg = dense_depth_grid(depthmap).astype(np.float64)
    G = dg.shape[0]
    cost = np.where(dg > 0, dg + eps, 0.05)               # far (depth 0) points: lookup only
    cx = np.bincount(_cells_of_axis(R, G), minlength=G).astype(np.float64)
    per_cell_plane = np.einsum("zyx,y,x->z", cost, cx, cx)
    return per_cell_plane[_cells_of_axis(Rz, G)]


def balanced_cuts(work, nparts):
    """Contiguous cuts k_0 = 0 < k_1 < ... < k_n = len(work) equalising sum(work[k_r:k_{r+1}])."""
    work = np.asarray(work, np.float64)
    Rz = work.size
    if nparts > Rz:
        raise ValueError("more ranks than planes")
    cum = np.concatenate([[0.0], np.cumsum(work)])
    tgt = cum[-1] * np.arange(1, nparts) / nparts
    cuts = np.searchsorted(cum, tgt, side="left")
    cuts = np.concatenate([[0], cuts, [Rz]]).astype(np.int64)
    for r in range(1, nparts + 1):               # every rank gets at least one plane
        cuts[r] = max(cuts[r], cuts[r - 1] + 1)
    for r in range(nparts - 1, -1, -1):
        cuts[r] = min(cuts[r], cuts[r + 1] - 1)
    return cuts


def shard_planes(depthmap, R, world, rank, weak=True):
    """z-plane range [k0, k1) of `rank` and the grid's Rz.  Weak scaling: Rz = R * world (the grid
    is refined along z so every rank holds ~R^3 points); strong: Rz = R."""
    Rz = R * world if weak else R
    if world == 1:
        return 0, Rz, Rz
    cuts = balanced_cuts(plane_work(depthmap, R, Rz), world)
    return int(cuts[rank]), int(cuts[rank + 1]), Rz


RECORD_FIELDS = 8 + 33


def make_record(n, per_depth, ms, sdf_fx, depth_hash, k0, k1, queries, ms_full=0.0):
    """Fixed-size int64 record a rank contributes to the NCCL all-gather: point count, timed-region device
    time (ns), fixed-point SDF checksum sum(round(sdf * 2^24)), position-weighted depth hash, shard range,
    query count, full-depth comparison time (ns), per-depth counts.  Integer sums are exact and
    order-independent, so the totals over ranks are identical for any number of GPUs."""
    rec = np.zeros(RECORD_FIELDS, np.int64)
    rec[:8] = [int(n), int(round(ms * 1e6)), int(sdf_fx), int(depth_hash), int(k0), int(k1), int(queries),
               int(round(ms_full * 1e6))]
    pd = np.asarray(per_depth, np.int64)
    rec[8:8 + pd.size] = pd
    return rec


def summarize(records):
    r = np.asarray(records, np.int64).reshape(-1, RECORD_FIELDS)
    return dict(n_total=int(r[:, 0].sum()), ms_max=float(r[:, 1].max()) / 1e6, ms_min=float(r[:, 1].min()) / 1e6,
                sdf_fx=int(r[:, 2].sum()), depth_hash=int(r[:, 3].sum()), ms_full_max=float(r[:, 7].max()) / 1e6,
                per_depth=r[:, 8:].sum(0).astype(np.int64).tolist(),
                ranges=[(int(a), int(b)) for a, b in r[:, 4:6]])
