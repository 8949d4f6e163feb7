"""SAND oracle (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

Every function cites the PAPER.md passage it restates.  No blocking, fusion or reordering beyond
the definitions: the network is evaluated layer by layer exactly as Eq. 2 / Eq. 3 are written, with
numpy float64 matrix-vector products as the only library primitive.

Parameters are passed duck-typed (any object with the attributes below), so this module imports
nothing from the product package or from the input generators:
    W[i-1] : [H][fan_in] float32   (fan_in = 3 for i = 1, else H)      -- W_i of Eq. 2
    b[i-1] : [H] float32                                               -- b_i of Eq. 2
    a[i-1] : [H] float32, c[i-1] : float  -- LINEAR tail W_i^out, b_i^out (Eq. 2); for MULT, the
                                              t_{i0} factor W_{i0}^out, b_{i0}^out (Eq. 3, i >= 2)
    a1[i-2], c1[i-2]                        -- MULT only: the t_{i1} factor (Eq. 3, i >= 2)
    spec.omega0, spec.tail (0 = LINEAR, 1 = MULT), spec.L, spec.H
"""
import numpy as np

NONFINITE_DEPTH = 255   # include/sand.h: non-finite query points report exit depth 255, sdf NaN
LINEAR, MULT = 0, 1


# --------------------------------------------------------------------------------------------
# Volumetric network-depth map lookup   (Sec. 3.4 "we first query the
# volumetric network-depth map (octree) for all points"; octree = Sec. 3.2, Eq. 7)
# --------------------------------------------------------------------------------------------
def cell_coords(points: np.ndarray, level: int) -> np.ndarray:
    """Integer cell (ix, iy, iz) of each point in the 2^level grid over [-1,1]^3.

    DESIGN.md reading R1 (the paper gives no cell arithmetic; SPEC S:318/S:337 fixes half-open
    [lo, hi) with the global upper face closed).  The cell index is decided in float32, the
    kernel's precision:  u = fl32(x + 1);  v = u * 2^(level-1) (exact);  v = min(max(v, 0),
    2^level - 1);  c = floor(v).   Points outside [-1,1]^3 clamp to the boundary cell.
    """
    p = np.asarray(points, np.float32)
    with np.errstate(over="ignore", invalid="ignore"):
        u = p + np.float32(1.0)                              # one float32 rounding
        v = u * np.float32(2.0 ** (level - 1))               # exact (power of two)
        v = np.minimum(np.maximum(v, np.float32(0.0)), np.float32((1 << level) - 1))
    return np.floor(v).astype(np.int64)


def _finite_rows(points):
    return np.isfinite(np.asarray(points, np.float32)).all(axis=1)


def lookup_voxel(level, depth, far_sdf, points):
    """Dense voxel depth map (BJ configs[0], [1]): payload of cell i + G*(j + G*k)."""
    G = 1 << level
    c = cell_coords(np.nan_to_num(points, nan=0.0), level)
    lin = c[:, 0] + G * (c[:, 1] + G * c[:, 2])
    d = np.asarray(depth, np.uint8)[lin]
    f = np.asarray(far_sdf, np.float32)[lin] if far_sdf is not None else np.zeros(len(lin), np.float32)
    return d, f, lin


def lookup_octree(level, nodes, leaf_depth, leaf_far, points):
    """Root-to-leaf descent (Sec. 3.2: the octree's leaf O(x) containing x, Eq. 5-7).

    At step k the child octant is bit (level-1-k) of the level-`level` cell coordinates,
    octant = xbit | ybit<<1 | zbit<<2 (include/sand.h node encoding).
    """
    nodes = np.asarray(nodes, np.uint32)
    c = cell_coords(np.nan_to_num(points, nan=0.0), level)
    n = c.shape[0]
    node = np.zeros(n, np.int64)
    leaf = np.full(n, -1, np.int64)
    active = np.ones(n, bool)
    for k in range(level + 1):
        payload = nodes[node[active]]
        is_leaf = (payload >> np.uint32(31)) == 1
        idx_active = np.nonzero(active)[0]
        done = idx_active[is_leaf]
        leaf[done] = (payload[is_leaf] & np.uint32(0x7FFFFFFF)).astype(np.int64)
        active[done] = False
        if not active.any():
            break
        go = idx_active[~is_leaf]
        child = payload[~is_leaf].astype(np.int64)
        bit = level - 1 - k
        oct_ = (((c[go, 0] >> bit) & 1) | (((c[go, 1] >> bit) & 1) << 1) | (((c[go, 2] >> bit) & 1) << 2))
        node[go] = child + oct_
    assert not active.any(), "octree deeper than its declared level"
    d = np.asarray(leaf_depth, np.uint8)[leaf]
    f = np.asarray(leaf_far, np.float32)[leaf] if leaf_far is not None else np.zeros(n, np.float32)
    return d, f, leaf


def lookup_bruteforce(leaf_level, leaf_ijk, leaf_depth, leaf_far, points):
    """Brute-force linear scan over the leaf list (SPEC S:317 'traversal result equals linear scan
    over serialized leaf list'): a leaf (l, i, j, k) contains x iff x's level-l cell is (i, j, k).
    For tiny inputs only (O(n_points * n_leaves))."""
    pts = np.nan_to_num(np.asarray(points, np.float32), nan=0.0)
    n = pts.shape[0]
    owner = np.full(n, -1, np.int64)
    hits = np.zeros(n, np.int64)
    for li in range(len(leaf_level)):
        c = cell_coords(pts, int(leaf_level[li]))
        inside = (c == np.asarray(leaf_ijk[li])[None, :]).all(axis=1)
        owner[inside] = li
        hits += inside
    assert (hits == 1).all(), "leaves do not partition the domain"
    d = np.asarray(leaf_depth, np.uint8)[owner]
    f = np.asarray(leaf_far, np.float32)[owner] if leaf_far is not None else np.zeros(n, np.float32)
    return d, f, owner


def lookup(depthmap, points):
    """Dispatch on a VoxelMap-like (level, depth, far_sdf) or Octree-like (level, nodes, ...)."""
    if hasattr(depthmap, "nodes"):
        return lookup_octree(depthmap.level, depthmap.nodes, depthmap.leaf_depth,
                             depthmap.leaf_far_sdf, points)
    return lookup_voxel(depthmap.level, depthmap.depth, depthmap.far_sdf, points)


# --------------------------------------------------------------------------------------------
# T-MLP   (Eq. 2; Eq. 3; sigma = sin(omega0 * .), SIREN)
# --------------------------------------------------------------------------------------------
def _layer(params, i, h):
    """h_i = sigma(W_i h_{i-1} + b_i), sigma(z) = sin(omega0 z)  (Eq. 2; reading R4)."""
    W = np.asarray(params.W[i - 1], np.float64)
    b = np.asarray(params.b[i - 1], np.float64)
    return np.sin(params.spec.omega0 * (h @ W.T + b))


def _tail(params, i, h):
    """t_i.  LINEAR: W_i^out h_i + b_i^out (Eq. 2).  MULT (i >= 2): t_{i0} * t_{i1} with
    t_{i0} = W_{i0}^out h_i + b_{i0}^out, t_{i1} = W_{i1}^out h_i + b_{i1}^out (Eq. 3); the first
    tail is always linear (Eq. 3 starts at i = 2)."""
    a = np.asarray(params.a[i - 1], np.float64)
    t = h @ a + float(params.c[i - 1])
    if params.spec.tail == MULT and i >= 2:
        a1 = np.asarray(params.a1[i - 2], np.float64)
        t = t * (h @ a1 + float(params.c1[i - 2]))
    return t


def tmlp_trace(params, x):
    """All cumulative outputs: returns (h list, t [L][n], y [L][n]) for h_0 = x, y_0 = 0,
    y_i = y_{i-1} + t_i, i = 1..L (Eq. 2)."""
    h = np.asarray(x, np.float64)
    L = params.spec.L
    n = h.shape[0]
    y = np.zeros(n)
    ts, ys, hs = [], [], []
    for i in range(1, L + 1):
        h = _layer(params, i, h)
        t = _tail(params, i, h)
        y = y + t
        hs.append(h); ts.append(t); ys.append(y)
    return hs, np.array(ts), np.array(ys)


def tmlp_forward(params, x, depth):
    """y_{d(x)}(x) = sum_{k <= d(x)} t_k(x) for a per-point depth d >= 1 (Eq. 2 truncated at the
    exit depth; Sec. 3.4 P:368 'network evaluation with point-wise adaptive depths').  Layers
    beyond a point's depth are never evaluated for that point (only rows with d >= i enter layer i).
    """
    x = np.asarray(x, np.float64)
    depth = np.broadcast_to(np.asarray(depth, np.int64), (x.shape[0],))
    n = x.shape[0]
    H = params.spec.H
    y = np.zeros(n)
    h = np.zeros((n, H))
    dmax = int(depth.max()) if n else 0
    for i in range(1, dmax + 1):
        act = np.nonzero(depth >= i)[0]
        hin = x[act] if i == 1 else h[act]
        hi = _layer(params, i, hin)
        h[act] = hi
        y[act] = y[act] + _tail(params, i, hi)
    return y


def query(params, depthmap, points, lod_cap=None):
    """SAND adaptive inference (Sec. 3.4):
      1. look up every point in the depth map;
      2. far leaves (depth 0, Eq. 7): return the cached sdf(c_N), no network evaluation;
      3. near leaves: evaluate the T-MLP to d = min(d(N), cap) (LOD cap) and return y_d.
    Non-finite points -> (NaN, 255) (include/sand.h).  Returns (sdf float64 [n], exit depth u8 [n]).
    """
    pts = np.asarray(points, np.float32)
    n = pts.shape[0]
    fin = _finite_rows(pts)
    d, far, _ = lookup(depthmap, pts)
    d = d.astype(np.int64)
    if lod_cap is not None:
        d = np.where(d > 0, np.minimum(d, int(lod_cap)), d)   # reading R16: cap only d >= 1
    sdf = np.zeros(n)
    isfar = fin & (d == 0)
    sdf[isfar] = far[isfar].astype(np.float64)
    near = np.nonzero(fin & (d > 0))[0]
    if near.size:
        sdf[near] = tmlp_forward(params, pts[near], d[near])
    sdf[~fin] = np.nan
    ed = np.where(fin, d, NONFINITE_DEPTH).astype(np.uint8)
    return sdf, ed


def query_full(params, points):
    """Uniform full-depth evaluation y_L for every point (Eq. 2 at i = L; SPEC query_full S:374)."""
    return tmlp_forward(params, np.asarray(points, np.float32), params.spec.L)


# --------------------------------------------------------------------------------------------
# Volumetric network-depth map population   (Sec. 3.2, Eq. 5 and Eq. 6)
# --------------------------------------------------------------------------------------------
def required_depth(params, x, r, near=True):
    """Eq. 5:  d(x) = min{ i : |y_L(x) - y_i(x)| < r  and  S_i(x) }  for near-surface points
    (delta = 1), d(x) = min{ i : S_i(x) } for far points (delta = 0), with
    S_i(x) := sign(y_i(x)) = sign(y_L(x)).  i runs over 1..L; i = L always qualifies.
    Evaluated in float64 (R14).  Returns int64 [n]."""
    _, _, ys = tmlp_trace(params, x)           # ys[i-1] = y_i, shape [L][n]
    yL = ys[-1]
    ok = np.sign(ys) == np.sign(yL)[None, :]
    if near:
        ok &= np.abs(yL[None, :] - ys) < r
    ok[-1, :] = True
    return np.argmax(ok, axis=0).astype(np.int64) + 1


def populate_leaf_depths(params, samples, r):
    """Eq. 6: d(N) = max over the leaf's sample points x of d(x) (near branch of Eq. 5).
    samples: [n_leaves, spl, 3] (the sample set is an input; R21).  Returns int64 [n_leaves]."""
    s = np.asarray(samples, np.float32)
    n, spl = s.shape[0], s.shape[1]
    d = required_depth(params, s.reshape(-1, 3), r, near=True).reshape(n, spl)
    return d.max(axis=1)


# --------------------------------------------------------------------------------------------
# Dynamic-exit inference without a depth map   (Sec. 5 ablation "Necessity of
# the Octree Structure", "SAND w/o Octree", Tab. octree)
# --------------------------------------------------------------------------------------------
def query_dynamic(params, points, r):
    """'SAND w/o Octree': no depth map; every point proceeds layer by layer and 'if the
    absolute value of the predicted residual at the current layer falls below the error threshold r,
    the computation is terminated; otherwise, it proceeds to the next layer until the maximum depth
    is reached'.  The residual of layer i is t_i = y_i - y_{i-1} (Eq. 2); reading R23: the
    test applies from i = 2 (t_1 = y_1 is the first prediction itself, not a residual), so
      d(x) = min{ i >= 2 : |t_i(x)| < r }  (L if none; 1 if L = 1),   sdf = y_{d(x)}(x).
    Layer i is evaluated only for the points still running.  Non-finite points -> (NaN, 255).
    Returns (sdf float64 [n], exit depth u8 [n])."""
    pts = np.asarray(points, np.float32)
    n = pts.shape[0]
    L = params.spec.L
    fin = _finite_rows(pts)
    sdf = np.zeros(n)
    dep = np.full(n, L, np.int64)
    act = np.nonzero(fin)[0]
    h = np.asarray(pts[act], np.float64)
    y = np.zeros(act.size)
    for i in range(1, L + 1):
        h = _layer(params, i, h)
        t = _tail(params, i, h)
        y = y + t
        if i == L:
            sdf[act] = y
            break
        if i >= 2:
            stop = np.abs(t) < r
            sdf[act[stop]] = y[stop]
            dep[act[stop]] = i
            keep = ~stop
            act, h, y = act[keep], h[keep], y[keep]
            if act.size == 0:
                break
    sdf[~fin] = np.nan
    dep[~fin] = NONFINITE_DEPTH
    return sdf, dep.astype(np.uint8)


# --------------------------------------------------------------------------------------------
# Marching cubes on the query grid   (meshes are extracted from the SDF on a
# 512^3 grid with Marching Cubes [Lorensen and Cline])
# --------------------------------------------------------------------------------------------
# DESIGN.md reading R24.  The per-configuration triangulation is derived here from the cube itself
# (no stored table): a corner is inside iff sdf < 0; on each of the 6 faces, walked counter-clockwise
# as seen from outside the cube, every crossing edge entered from an outside corner starts a segment
# that ends at the next crossing edge of the walk, so a face with two diagonal inside corners keeps
# them separated (a rule that depends on the face's own corners only, hence watertight across
# cubes).  Every crossing edge starts one segment and ends one, the segments chain into closed loops,
# and each loop of k edge points becomes a fan of k - 2 triangles.
def _mc_edges():
    """Cube corners v = x + 2y + 4z; the 12 edges as (v0, v1), v1 = v0 + 2^axis, axis-major."""
    return [(v, v | (1 << a)) for a in range(3) for v in range(8) if not (v >> a) & 1]


def _mc_faces():
    """6 faces as corner cycles, counter-clockwise seen from outside the cube."""
    faces = []
    for a in range(3):
        u, w = (a + 1) % 3, (a + 2) % 3                  # e_u x e_w = e_a
        for side in (0, 1):
            cyc = [(0, 0), (1, 0), (1, 1), (0, 1)]       # CCW about +e_a
            if side == 0:
                cyc = cyc[::-1]                          # CCW about -e_a
            faces.append([(side << a) | (cu << u) | (cw << w) for cu, cw in cyc])
    return faces


def mc_loops(case):
    """Closed loops (lists of edge ids) of the iso-surface inside one cube; bit v of case = corner v
    inside."""
    edges = _mc_edges()
    eid = {frozenset(e): i for i, e in enumerate(edges)}
    inside = [(case >> v) & 1 for v in range(8)]
    nxt = {}
    for cyc in _mc_faces():
        cross = []                                       # (edge, entering?) in walk order
        for k in range(4):
            p, q = cyc[k], cyc[(k + 1) % 4]
            if inside[p] != inside[q]:
                cross.append((eid[frozenset((p, q))], inside[q] == 1))
        for k, (e, entering) in enumerate(cross):
            if entering:
                nxt[e] = cross[(k + 1) % len(cross)][0]
    loops, seen = [], set()
    for e0 in sorted(nxt):
        if e0 in seen:
            continue
        loop, e = [], e0
        while e not in seen:
            seen.add(e)
            loop.append(e)
            e = nxt[e]
        loops.append(loop)
    return loops


def marching_cubes(sdf, R):
    """Triangles of the sdf = 0 surface of an R x R x R vertex grid (sdf[i + R (j + R k)], vertex
    (i, j, k) at (x_i, x_j, x_k), x_i = fl32(2 i / (R - 1) - 1), reading R8).  A vertex on a crossing
    edge (v0, v1) lies at P0 + t (P1 - P0), t = s0 / (s0 - s1), computed from the edge's lower corner
    (so both cubes sharing the edge produce the same point).  Float64.  Returns [T, 3, 3]."""
    s = np.asarray(sdf, np.float64).reshape(R, R, R)     # [k][j][i]
    ax = (2.0 * np.arange(R) / (R - 1) - 1.0).astype(np.float32).astype(np.float64)
    edges = _mc_edges()
    tris = []
    for k in range(R - 1):
        for j in range(R - 1):
            for i in range(R - 1):
                vals = [s[k + (v >> 2), j + ((v >> 1) & 1), i + (v & 1)] for v in range(8)]
                case = sum(1 << v for v in range(8) if vals[v] < 0)
                if case == 0 or case == 255:
                    continue
                def point(e):
                    v0, v1 = edges[e]
                    s0, s1 = vals[v0], vals[v1]
                    t = s0 / (s0 - s1)
                    p0 = np.array([ax[i + (v0 & 1)], ax[j + ((v0 >> 1) & 1)], ax[k + (v0 >> 2)]])
                    p1 = np.array([ax[i + (v1 & 1)], ax[j + ((v1 >> 1) & 1)], ax[k + (v1 >> 2)]])
                    return p0 + t * (p1 - p0)
                for loop in mc_loops(case):
                    pts = [point(e) for e in loop]
                    for m in range(1, len(pts) - 1):
                        tris.append([pts[0], pts[m], pts[m + 1]])
    return np.array(tris).reshape(-1, 3, 3)
