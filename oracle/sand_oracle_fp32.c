/*
 * sand_oracle_fp32.c -- plain, slow FP32 C oracle of SAND's adaptive query path.
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs; the product (paper_2604_25936_b200/) never links it.
 * It shares no header, table or helper with csrc/: everything below is restated from the paper.
 *
 * This is the oracle BASELINE.json's north star names ("a plain, slow FP32 C++ CPU implementation"):
 * IEEE binary32 arithmetic, every sum sequential in index order, no FMA contraction (built with
 * -ffp-contract=off), glibc sinf, one OpenMP thread per point range.  Its float64 twin
 * (oracle/sand_oracle.py) pins it (tests/test_oracle_fp32.py).
 *
 * Per point x (Sec. 3.4):
 *   1. cell of x in the depth map (reading R1, float32): per axis u = x + 1,
 *      v = u * 2^(level-1) (exact), v = min(max(v, 0), 2^level - 1), c = floor(v);
 *      voxel: payload at c_x + G (c_y + G c_z); octree: root-to-leaf descent, child octant at step k =
 *      bit (level-1-k) of (c_x, c_y, c_z) as xbit | ybit<<1 | zbit<<2 (Sec. 3.2; sand.h).
 *   2. d = payload; d = min(d, cap) for d >= 1 (LOD cap; reading R16).
 *   3. d = 0: sdf = cached far SDF of the cell / leaf (Eq. 7).
 *   4. d >= 1: h_0 = x; for i = 1..d: z_j = b_ij + sum_k W_ijk h_k; h_ij = sinf(omega0 * z_j) (Eq. 2,
 *      P:176-182; reading R4); t_i = c_i + sum_j a_ij h_ij (LINEAR) or, for i >= 2 with MULT tails,
 *      (c_i + sum_j a_ij h_ij) * (c1_i + sum_j a1_ij h_ij) (Eq. 3); y += t_i.  sdf = y_d.
 *   Non-finite x: depth 255, sdf NaN (include/sand.h convention, reading R19).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_NONFINITE 255

/* Cell coordinate of one axis (reading R1). */
static int64_t cell_axis(float x, int level) {
  const float G1 = (float)((1 << level) - 1);
  float u = x + 1.0f;
  float v = u * ldexpf(1.0f, level - 1);
  if (v < 0.0f) v = 0.0f;
  if (v > G1) v = G1;
  return (int64_t)floorf(v);
}

/* Returns the payload index (voxel cell or octree leaf), or -1 if the octree is deeper than level. */
static int64_t locate(int kind, int level, const uint32_t* nodes, float x, float y, float z) {
  const int64_t cx = cell_axis(x, level), cy = cell_axis(y, level), cz = cell_axis(z, level);
  if (kind == 0) {
    const int64_t G = (int64_t)1 << level;
    return cx + G * (cy + G * cz);
  }
  int64_t node = 0;
  for (int k = 0; k <= level; ++k) {
    const uint32_t payload = nodes[node];
    if (payload >> 31) return (int64_t)(payload & 0x7FFFFFFFu);
    const int bit = level - 1 - k;
    const int64_t oct = ((cx >> bit) & 1) | (((cy >> bit) & 1) << 1) | (((cz >> bit) & 1) << 2);
    node = (int64_t)payload + oct;
  }
  return -1;
}

/*
 * Parameters (canonical blob of include/sand.h, parsed here independently):
 *   W1 [H][3], Wh [L-1][H][H] (row j = output unit), b [L][H], a [L][H], c [L],
 *   a1 [L-1][H], c1 [L-1] (MULT only; NULL otherwise).
 * Depth map: kind 0 = voxel (depth [G^3], far [G^3] or NULL), 1 = octree (nodes, depth/far per leaf).
 * cap <= 0: no LOD cap.  nthreads <= 0: OpenMP default.
 * Returns 0, or -1 if some octree descent did not reach a leaf within `level` steps.
 */
int oracle_query_fp32(int L, int H, float omega0, int tail, const float* W1, const float* Wh, const float* b,
                      const float* a, const float* c, const float* a1, const float* c1, int kind, int level,
                      const uint8_t* depth, const float* far_sdf, const uint32_t* nodes, int cap,
                      const float* pts, int64_t n, float* out_sdf, uint8_t* out_depth, int nthreads) {
  int bad = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel reduction(| : bad)
  {
    float* hprev = (float*)malloc(sizeof(float) * (size_t)(H > 3 ? H : 3));
    float* hcur = (float*)malloc(sizeof(float) * (size_t)H);
#pragma omp for schedule(static)
    for (int64_t p = 0; p < n; ++p) {
      const float x = pts[3 * p], y = pts[3 * p + 1], z = pts[3 * p + 2];
      if (!isfinite(x) || !isfinite(y) || !isfinite(z)) {
        out_depth[p] = ORACLE_NONFINITE;
        out_sdf[p] = NAN;
        continue;
      }
      const int64_t cell = locate(kind, level, nodes, x, y, z);
      if (cell < 0) {
        bad = 1;
        out_depth[p] = 0;
        out_sdf[p] = NAN;
        continue;
      }
      int d = depth[cell];
      if (d > 0 && cap > 0 && d > cap) d = cap;
      out_depth[p] = (uint8_t)d;
      if (d == 0) {
        out_sdf[p] = far_sdf ? far_sdf[cell] : 0.0f;
        continue;
      }
      hprev[0] = x;
      hprev[1] = y;
      hprev[2] = z;
      int fan_in = 3;
      float yout = 0.0f;
      for (int i = 1; i <= d; ++i) {
        const float* W = i == 1 ? W1 : Wh + (size_t)(i - 2) * H * H;
        const float* bi = b + (size_t)(i - 1) * H;
        for (int j = 0; j < H; ++j) {
          float acc = bi[j];
          const float* wr = W + (size_t)j * fan_in;
          for (int k = 0; k < fan_in; ++k) {
            const float prod = wr[k] * hprev[k];
            acc = acc + prod;
          }
          const float arg = omega0 * acc;
          hcur[j] = sinf(arg);
        }
        const float* ai = a + (size_t)(i - 1) * H;
        float t0 = c[i - 1];
        for (int j = 0; j < H; ++j) {
          const float prod = ai[j] * hcur[j];
          t0 = t0 + prod;
        }
        float t = t0;
        if (tail == 1 && i >= 2) {
          const float* a1i = a1 + (size_t)(i - 2) * H;
          float t1 = c1[i - 2];
          for (int j = 0; j < H; ++j) {
            const float prod = a1i[j] * hcur[j];
            t1 = t1 + prod;
          }
          t = t0 * t1;
        }
        yout = yout + t;
        for (int j = 0; j < H; ++j) hprev[j] = hcur[j];
        fan_in = H;
      }
      out_sdf[p] = yout;
    }
    free(hprev);
    free(hcur);
  }
  return bad ? -1 : 0;
}

/* Exit depths only (steps 1-2 above): out_depth[p] = min(payload, cap) for payload >= 1, 0 for far cells,
 * 255 for non-finite points.  Returns 0, or -1 on a too-deep octree. */
int oracle_lookup_fp32(int kind, int level, const uint8_t* depth, const uint32_t* nodes, int cap, const float* pts,
                       int64_t n, uint8_t* out_depth, int nthreads) {
  int bad = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t p = 0; p < n; ++p) {
    const float x = pts[3 * p], y = pts[3 * p + 1], z = pts[3 * p + 2];
    if (!isfinite(x) || !isfinite(y) || !isfinite(z)) {
      out_depth[p] = ORACLE_NONFINITE;
      continue;
    }
    const int64_t cell = locate(kind, level, nodes, x, y, z);
    if (cell < 0) {
      bad = 1;
      out_depth[p] = 0;
      continue;
    }
    int d = depth[cell];
    if (d > 0 && cap > 0 && d > cap) d = cap;
    out_depth[p] = (uint8_t)d;
  }
  return bad ? -1 : 0;
}

/* Threads the OpenMP runtime will use (reported as the CPU baseline's core count). */
int oracle_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
  return omp_get_max_threads();
#else
  (void)nthreads;
  return 1;
#endif
}
