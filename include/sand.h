/*
 * sand.h -- C ABI of libsand, the B200 (sm_100a) engine for SAND's adaptive-depth T-MLP query path.
 *
 * Method: SAND, "Spatially Adaptive Network Depth for Fast Sampling of Neural Implicit Surfaces"
 * (arxiv 2604.25936; /root/reference/PAPER.md = "P:<line>").  A query point x first looks up its
 * required network depth d(x) in a volumetric network-depth map (Sec. 3.2; inference
 * Sec. 3.4); far leaves (d = 0) return a cached SDF value (Eq. 7); near
 * points evaluate the tailed MLP (T-MLP, Eq. 2; multiplicative tails Eq. 3)
 * only up to layer d and return the cumulative output y_d = sum_{k<=d} t_k.
 *
 * Conventions for every entry point:
 *   - Return value: 0 (SAND_OK) on success, a negative sand_status on error.  No C++ exception
 *     crosses the ABI.  sand_last_error(ctx) returns a human-readable message for the last error.
 *   - Ownership: the caller owns every pointer it passes in; libsand copies what it keeps (weights,
 *     depth map).  The context owns its device copies and its workspace.
 *   - Threading: one context per device; calls on one context must not race.  Different contexts
 *     are independent (the multi-GPU driver uses one context per rank/GPU).
 *   - No collective communication happens inside the library.
 *   - Device pointers ("d_" prefix) must be CUDA device memory of the context's device.
 */
#ifndef SAND_H_
#define SAND_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAND_ABI_VERSION 1
#define SAND_MAX_L 32
#define SAND_DEPTH_NONFINITE 255

typedef enum {
  SAND_OK = 0,
  SAND_ERR_ARG = -1,         /* NULL where not allowed, negative size, out-of-range knob      */
  SAND_ERR_STATE = -2,       /* e.g. sand_query before both sand_load_weights and _depthmap    */
  SAND_ERR_SIZE = -3,        /* weight blob length does not match (L, H, tail)                  */
  SAND_ERR_DEPTHMAP = -4,    /* malformed depth map (depth > L, bad node index, cycle, level)   */
  SAND_ERR_CUDA = -5,        /* a CUDA runtime error; message via sand_last_error               */
  SAND_ERR_OOM = -6,         /* device allocation failed                                         */
  SAND_ERR_UNSUPPORTED = -7  /* configuration not supported by this build (e.g. H for a precision) */
} sand_status;

/* Arithmetic of the H x H layers.
 *   SAND_FP32  : FP32 SIMT kernels (FFMA; sine to ~5e-7: Cody-Waite reduction to [-pi, pi] +
 *                MUFU.SIN); supported H in {16, 32, 64} (one thread per
 *                point) and {128, 256, 336} (register-blocked GEMM over 64-point sub-tiles, L <= 32).
 *                Tolerance vs the oracle: 1e-4 max-abs (BASELINE.json north_star).
 *   SAND_BF16  : tcgen05 tensor cores, BF16 operands, FP32 accumulate in TMEM; layer 1 (K = 3) as a
 *                split-BF16 MMA (x = x_hi + x_lo, relative error ~2^-16) or FP32 SIMT, all tails and
 *                the sine in FP32; supported H in {64, 128, 256, 336}; the per-column tables stay on
 *                chip, which bounds L (e.g. L <= 24 at H = 256; larger -> SAND_ERR_UNSUPPORTED).
 *                Tolerance 5e-3.
 *   SAND_TF32X3: reserved (returns SAND_ERR_UNSUPPORTED in this build): 3xTF32 operands take 4 bytes
 *                per element, so a 256-row tile's split A operand (hi + lo) would not fit in shared memory.
 *   SAND_F16X3 : FP32-accurate tensor-core path (tmlp_x3.cu): every H x H layer as three tcgen05 kind::f16
 *                products of split operands, v = v_hi + v_lo (FP16 each, 22 significant bits):
 *                A_hi W_hi + A_lo W_hi + A_hi W_lo, FP32 accumulate in TMEM; layer 1 in FP32 SIMT; sine with
 *                a Cody-Waite reduction (~5e-7).  H in {64, 128, 256}.  Tolerance 1e-4 like SAND_FP32.
 *                The same kernel evaluates the Eq. 5 population calls below whatever ctx's precision
 *                (SAND_OPT_FP32_TENSOR).                                                            */
typedef enum { SAND_FP32 = 0, SAND_TF32X3 = 1, SAND_BF16 = 2, SAND_F16X3 = 3 } sand_precision;

/* Tail form: LINEAR t_i = a_i . h_i + c_i for every layer (BASELINE.json configs);
 * MULT t_1 linear, t_i = (a_i0 . h_i + c_i0) * (a_i1 . h_i + c_i1) for i >= 2 (Eq. 3).        */
typedef enum { SAND_TAIL_LINEAR = 0, SAND_TAIL_MULT = 1 } sand_tail_mode;

typedef struct {
  int L;                 /* hidden layers, 1..SAND_MAX_L                                       */
  int H;                 /* hidden width                                                        */
  float omega0;          /* SIREN frequency: h_i = sin(omega0 * (W_i h_{i-1} + b_i)), > 0       */
  sand_precision prec;
  sand_tail_mode tail;
  int device;            /* CUDA device ordinal the context binds to                            */
} sand_config;

typedef struct sand_ctx sand_ctx;   /* opaque */

/* Create a context on cfg->device.  Validates L in [1, 32], omega0 > 0 and that (prec, H) is a
 * supported pair.  *out is set only on success.  Errors: SAND_ERR_ARG, SAND_ERR_UNSUPPORTED,
 * SAND_ERR_CUDA. */
int sand_create(const sand_config* cfg, sand_ctx** out);

/* Release every device resource of ctx.  NULL-safe.  Synchronizes ctx's stream first. */
int sand_destroy(sand_ctx* ctx);

/* Load the T-MLP parameters (Eq. 2/3) from a HOST FP32 blob in canonical order:
 *   for i = 1..L: W_i [H][fan_in] row-major (fan_in = 3 if i == 1 else H), b_i [H];
 *   LINEAR tails: for i = 1..L: a_i [H], c_i;
 *   MULT tails  : a_1 [H], c_1, then for i = 2..L: a_i0 [H], c_i0, a_i1 [H], c_i1.
 * n_floats must match exactly (else SAND_ERR_SIZE).  The blob is copied, converted on the device
 * (BF16 round-to-nearest-even for the H x H matrices in SAND_BF16 mode, laid out in the tcgen05
 * shared-memory image) and never referenced again.  Synchronous w.r.t. the host blob. */
int sand_load_weights(sand_ctx* ctx, const float* host_blob, size_t n_floats);

/* Volumetric network-depth map (Sec. 3.2; Eq. 7).  Domain [-1,1]^3; cell membership half-open
 * [lo, hi) per axis with the global upper face closed; points outside the domain clamp to the
 * boundary cell (their network input stays unclamped).  Cell arithmetic (float32, exact except
 * one rounding): u = x + 1; v = u * 2^(level-1); v = min(max(v, 0), 2^level - 1); c = floor(v).  */
typedef struct {
  int kind;                 /* 0 = dense voxel grid, 1 = octree                                 */
  int level;                /* voxel: G = 2^level cells per axis (1..10); octree: max level (0..20) */
  const uint8_t* depth;     /* HOST. voxel: G^3 depths, index i + G*(j + G*k) (x fastest);
                               octree: per-leaf depth.  0 = far (cached SDF), 1..L = exit depth  */
  const float* far_sdf;     /* HOST, optional (NULL if no depth-0 entry): cached SDF per cell/leaf */
  const uint32_t* nodes;    /* HOST, octree only: node i: bit31 = 1 -> leaf, low 31 bits = leaf
                               index; bit31 = 0 -> index of the first of 8 contiguous children,
                               octant = xbit | ybit<<1 | zbit<<2.  Node 0 is the root.           */
  int64_t n_nodes, n_leaves;
} sand_depthmap;

/* Copy a depth map to the device.  Validates depth <= L, child/leaf indices in range, descent
 * terminates within `level` steps; octrees with level <= 8 are baked on the device into a dense
 * 2^level grid (one load per query).  Errors: SAND_ERR_ARG, SAND_ERR_DEPTHMAP, SAND_ERR_OOM.     */
int sand_load_depthmap(sand_ctx* ctx, const sand_depthmap* dm);

/* Stream on which every subsequent kernel of ctx is enqueued (a cudaStream_t; NULL = legacy 0). */
int sand_set_stream(sand_ctx* ctx, void* cuda_stream);

/* Explicit execution options.  libsand reads no environment variable; every choice of kernel or
 * schedule is made here (defaults in brackets).
 *   SAND_OPT_PAIR_KERNEL  [2] SAND_BF16: 2 = the slot-team CTA-pair (cta_group::2) kernel (one N = H MMA
 *                         chain per layer, one epilogue team per tile slot; H in {64, 128, 256}, its tables
 *                         must fit shared memory), 1 = the two-pass CTA-pair kernels (H in {64, 128, 256,
 *                         336}), 0 = the 1-CTA kernel.  The default is 2 where usable, else 1, else 0; a value
 *                         without a kernel for the configuration -> SAND_ERR_UNSUPPORTED.  All compute the
 *                         same Eq. 2 / 3 arithmetic (BF16 operands, FP32 accumulation, sines and tails).
 *   SAND_OPT_DYN_SCHEDULE [0] sand_query_dynamic: 0 = a 64-point tile stops when all its points have
 *                         stopped; 1 = pools of 512 points re-compacted after every layer (both FP32 SIMT);
 *                         2 = every layer on the split-FP16 tensor-core kernel (SAND_F16X3 arithmetic),
 *                         the exit layer selected per point afterwards (H in {64, 128, 256}, else
 *                         SAND_ERR_UNSUPPORTED at the call).
 *   SAND_OPT_KPROF        [0] diagnostic, -DSAND_DIAG=1 builds only (ignored otherwise): 1 = per-role
 *                         clock64 wait / busy counters of the CTA-pair kernels printed to stderr after every
 *                         launch (adds a stream synchronisation); 2, 3 = timing-only modes that skip epilogue
 *                         math / weight streaming (wrong results).
 *   SAND_OPT_FP32_TENSOR  [1] sand_required_depth / sand_populate_leaf_depths at H in {64, 128, 256}: 1 = the
 *                         split-FP16 tensor-core kernel (SAND_F16X3 arithmetic), 0 = the FP32 SIMT kernel.
 * Errors: SAND_ERR_ARG (unknown option or value), SAND_ERR_UNSUPPORTED.                          */
typedef enum { SAND_OPT_PAIR_KERNEL = 1, SAND_OPT_DYN_SCHEDULE = 2, SAND_OPT_KPROF = 3, SAND_OPT_FP32_TENSOR = 4 } sand_option;
int sand_set_option(sand_ctx* ctx, int option, int64_t value);
int sand_get_option(const sand_ctx* ctx, int option, int64_t* value);

/* Level-of-detail cap (Sec. 3.4; Fig. 4): evaluated depth = min(d, cap) for d >= 1;
 * depth-0 (far) entries are unaffected.  cap in 1..L (default L).  Error: SAND_ERR_ARG.          */
int sand_set_lod_cap(sand_ctx* ctx, int cap);

/* Optional: pre-size the workspace for queries of up to n_max points (avoids allocation inside
 * sand_query, required before CUDA-graph capture). */
int sand_reserve(sand_ctx* ctx, int64_t n_max);

/* Adaptive SDF query (Sec. 3.4): for each of n points (d_points: n x 3 float32 AoS, device),
 *   d_out_exit_depth[i] = evaluated depth (0 = far/cached, 1..L, 255 = non-finite point);
 *   d_out_sdf[i]        = cached sdf (depth 0), y_d (Eq. 2), or NaN (non-finite point).
 * Asynchronous on ctx's stream; n == 0 is a no-op; outputs fully overwritten; inputs untouched.
 * d_points needs 4-byte alignment (16-byte alignment takes the vectorised path).
 * Errors: SAND_ERR_ARG, SAND_ERR_STATE, SAND_ERR_OOM, SAND_ERR_CUDA.                            */
int sand_query(sand_ctx* ctx, const float* d_points, int64_t n,
               float* d_out_sdf, uint8_t* d_out_exit_depth);

/* End-to-end variant with HOST buffers: copies points host->device, runs sand_query, copies the
 * results device->host, in chunks of at most chunk_points double-buffered over two streams, so the
 * copies of one chunk overlap the kernels of the next.  chunk_points = 0 lets the library choose:
 * n / 8 clamped to [2^21, 2^23] points (measured on B200: the pipeline fill / drain of a large first
 * and last chunk dominates otherwise; too small chunks under-fill the 148 SMs).  Host buffers should
 * be pinned for full bandwidth.  Returns after the results are in host memory (synchronous). */
int sand_query_host(sand_ctx* ctx, const float* h_points, int64_t n,
                    float* h_out_sdf, uint8_t* h_out_exit_depth, int64_t chunk_points);

typedef struct {
  int64_t n;                      /* points in the last query                                    */
  int64_t n_nonfinite;            /* points with a non-finite coordinate                         */
  int64_t per_depth[SAND_MAX_L + 1]; /* per evaluated depth 0..L (conservation: sum + nonfinite = n) */
  int64_t tiles;                  /* 128-row tiles the fused T-MLP kernel processed              */
  double flops_exec;              /* executed H x H FLOPs: sum_p (d_p - 1) * 2 H^2               */
  double flops_ns;                /* north-star formula: sum_p d_p * 2 H^2                        */
  float ms_lookup, ms_bin, ms_mlp, ms_total;  /* CUDA-event times of the last sand_query         */
  int64_t queries;                /* sand_query calls since the previous sand_get_stats (<= 1024) */
  double ms_lookup_sum, ms_bin_sum, ms_mlp_sum, ms_total_sum; /* summed over those queries       */
} sand_stats;

/* Statistics of the last sand_query on ctx (counts) and per-stage CUDA-event times of every query
 * since the previous sand_get_stats (sums), recorded on ctx's stream without synchronising inside
 * sand_query.  Resets the time sums.  Synchronizes ctx's stream. */
int sand_get_stats(sand_ctx* ctx, sand_stats* out);

/* Diagnostic: copy the depth-binning permutation of the last query to host_perm[0 .. min(cap,
 * n_binned)): indices of the points with evaluated depth 1..L, grouped by depth (deepest first) and
 * in ascending point order within a depth.  *n_binned = number of such points.  host_perm may be
 * NULL to query the count only.  Synchronizes ctx's stream. */
int sand_debug_perm(sand_ctx* ctx, uint32_t* host_perm, int64_t cap, int64_t* n_binned);

/* ---------------------------------------------------------------------------------------------------
 * Volumetric network-depth map population (the step before the query path; Sec. 3.2).
 * Both calls evaluate the full L-layer T-MLP in FP32 accuracy (sine to ~5e-7: Cody-Waite reduction to [-pi, pi],
 * then MUFU.SIN) whatever ctx's precision -- on the tensor cores with split-FP16 operands (SAND_F16X3
 * arithmetic) for H in {64, 128, 256}, else FP32 SIMT (SAND_OPT_FP32_TENSOR) -- because
 * Eq. 5 compares cumulative outputs against r (1.5e-4 in the paper).  Only the weights must be
 * loaded.  Asynchronous on ctx's stream.  Errors: SAND_ERR_ARG, SAND_ERR_STATE, SAND_ERR_UNSUPPORTED
 * (H not in {16, 32, 64, 128, 256, 336}), SAND_ERR_CUDA, SAND_ERR_OOM.                              */

/* Required depth (Eq. 5) of each of n points (d_points: n x 3 float32 AoS, device):
 *   near != 0: d(x) = min{ i : |y_L(x) - y_i(x)| < r and sign(y_i(x)) = sign(y_L(x)) }  (delta = 1)
 *   near == 0: d(x) = min{ i : sign(y_i(x)) = sign(y_L(x)) }                             (delta = 0)
 * written to d_out_depth[n] (1..L; i = L always qualifies). */
int sand_required_depth(sand_ctx* ctx, const float* d_points, int64_t n, float r, int near,
                        uint8_t* d_out_depth);

/* Leaf depths (Eq. 6): d_samples holds n_leaves x samples_per_leaf points (leaf-major,
 * float32 AoS, device; the sample set is the caller's, e.g. corners + centre + seeded interior points);
 * d_leaf_depth[N] = max over leaf N's samples of the near-branch d(x).  Far leaves (Eq. 7) are not
 * passed: their payload is the cached SDF, not a depth. */
int sand_populate_leaf_depths(sand_ctx* ctx, const float* d_samples, int64_t n_leaves, int samples_per_leaf,
                              float r, uint8_t* d_leaf_depth);

/* ---------------------------------------------------------------------------------------------------
 * Dynamic-exit query without a depth map: the paper's 'SAND w/o Octree' alternative (Sec. 5, P:736-738,
 * Tab. octree).  Each point runs the T-MLP layer by layer and stops at the first
 * layer i >= 2 whose residual |t_i| < r (reading R23: t_1 = y_1 is the first prediction, not
 * a residual), else at L:
 *   d_out_exit_depth[p] = that layer (255 for a non-finite point),  d_out_sdf[p] = y_d (NaN if 255).
 * FP32 accuracy (sine to ~5e-7) like the population calls above.  Schedule: SAND_OPT_DYN_SCHEDULE (a 64-point
 * tile stops as soon as all of its points have stopped; pools of 512 points re-compacted after every
 * layer; or all layers on the tensor cores with the exit selected afterwards).  Only the weights must be loaded; the depth map
 * and LOD cap are ignored.  Asynchronous on ctx's stream.  Errors: SAND_ERR_ARG (n < 0, r < 0 or NaN,
 * NULL buffer), SAND_ERR_STATE, SAND_ERR_UNSUPPORTED (H as above), SAND_ERR_CUDA. */
int sand_query_dynamic(sand_ctx* ctx, const float* d_points, int64_t n, float r, float* d_out_sdf,
                       uint8_t* d_out_exit_depth);

/* ---------------------------------------------------------------------------------------------------
 * Marching cubes on the R x R x R query grid (the paper's mesh extraction; SURVEY.md 8(f)
 * NEXT #2; triangulation rule: DESIGN.md reading R24 -- a corner is inside iff sdf < 0, at most 5
 * triangles per cube, normals toward sdf > 0, watertight).  Grid vertex (i, j, k) is at
 * (x_i, x_j, x_k), x_i = fl32(2 i / (R - 1) - 1); its sdf is element i + R (j + R k).
 * Output: triangle soup d_tris[9 t + 3 m + c] = coordinate c of vertex m of triangle t (float32,
 * device, caller-owned, room for cap triangles).  *n_tris (host) receives the number of triangles of
 * the surface; only the first min(n, cap) are written, so a call with cap = 0 sizes the buffer.  The
 * order of triangles is not deterministic (the set is).  Synchronous (returns after the count is
 * read back).  2 <= R <= 65535.  The context keeps R / 8 bytes per grid vertex row of scratch (vertex sign
 * words of the planes one call covers).  A vertex on a crossing edge is the edge's lower corner moved by
 * t = s0 / (s0 - s1) along the edge's axis (t by the fast divide: within 2 ulp; the two cubes sharing an
 * edge evaluate the same expression, so shared vertices are bit-identical).
 * Errors: SAND_ERR_ARG (R < 2 or R > 65535, cap < 0, NULL argument), SAND_ERR_STATE, SAND_ERR_CUDA,
 * SAND_ERR_OOM. */

/* Marching cubes on a caller-provided sdf grid (R^3 float32, device). */
int sand_marching_cubes(sand_ctx* ctx, const float* d_sdf, int R, float* d_tris, int64_t cap, int64_t* n_tris);

/* Fused extraction: evaluates the adaptive query path (sand_query with the loaded weights, depth map and
 * LOD cap) slab by slab -- slab planes of cubes at a time (0 = 64), the slab's grid planes of points
 * generated on the device (the shared boundary plane's sdf carried over, not re-queried) -- and meshes
 * each slab as soon as its sdf exists, so the R^3 sdf grid is never materialised (R = 512, slab 64:
 * 290 MB of slab buffers instead of the 1.6 GB of points and 537 MB of sdf of the whole grid). */
int sand_mesh_grid(sand_ctx* ctx, int R, int slab, float* d_tris, int64_t cap, int64_t* n_tris);

/* Message for the last error on ctx (or of the last failed sand_create if ctx is NULL).
 * Valid until the next call on ctx.  Never NULL. */
const char* sand_last_error(const sand_ctx* ctx);

/* ABI version (SAND_ABI_VERSION) of the loaded library. */
int sand_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SAND_H_ */
