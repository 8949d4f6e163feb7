// lookup.cu -- K1 depth-map lookup, K2a scan, K2b stable binning scatter, octree baking.
//
// K1 (Sec. 3.4, "we first query the volumetric network-depth map for all points";
// Eq. 7 P:237-246 far leaves return the cached SDF; LOD cap P:370): one pass over the n x 3 float32
// points (float4-vectorised, 12 B/pt) -> exit depth (1 B/pt), cached SDF for depth-0 points, and a
// per-block depth histogram.  K2a scans the histograms (deepest depth first) and K2b scatters point
// indices into perm[] so that every 128-row tile of the T-MLP kernel has one uniform depth (SPEC
// S:412 "depth-bucketed batching").  All three are HBM/L2-bound streaming kernels.
#include <cstdint>
#include <cuda_runtime.h>

#include "sand_internal.h"

namespace sand {

// Cell index along one axis; float32, no contraction: u = x + 1 (one rounding), v = u * 2^(l-1)
// (exact), clamp in float, floor.  Identical arithmetic to the oracle (reading R1).
__device__ __forceinline__ uint32_t cell_of(float x, float scale, float maxc) {
  float u = __fadd_rn(x, 1.0f);
  float v = __fmul_rn(u, scale);
  v = fminf(fmaxf(v, 0.0f), maxc);
  return (uint32_t)v;  // v >= 0 : truncation == floor (an FADD.RZ + 2^23 variant measured 4% slower)
}

struct LookupResult {
  uint32_t d;   // 0..L, or 255
  float far;
};

// KIND (compile time): 0 dense map without cached SDF, 1 dense with cached SDF, 2 octree descent.  Branch-free
// for the common finite case: the clamp in cell_of maps NaN / Inf to a valid boundary cell, and the non-finite
// decision is a select after the lookup.
template <int KIND>
__device__ __forceinline__ LookupResult lookup_one(float x, float y, float z, const LookupParams& lp,
                                                   float scale, float maxc) {
  LookupResult r;
  const bool fin = isfinite(x) && isfinite(y) && isfinite(z);
  const uint32_t cx = cell_of(x, scale, maxc), cy = cell_of(y, scale, maxc), cz = cell_of(z, scale, maxc);
  uint32_t d;
  float far = 0.0f;
  if (KIND < 2) {
    const uint64_t lin = (uint64_t)cx + ((uint64_t)cy << lp.level) + ((uint64_t)cz << (2 * lp.level));
    d = __ldg(lp.grid + lin);
    if (KIND == 1 && d == 0) far = __ldg(lp.grid_far + lin);
  } else {
    uint32_t node = 0, v;
    int bit = lp.level - 1;
    if (lp.top) {
      // resume the descent at level top_level from the dense start table (one L2-resident load
      // replaces the top_level pointer-chasing steps; entries may already be leaves)
      const int sh = lp.level - lp.top_level;
      const uint64_t t = (uint64_t)(cx >> sh) + ((uint64_t)(cy >> sh) << lp.top_level) +
                         ((uint64_t)(cz >> sh) << (2 * lp.top_level));
      v = __ldg(lp.top + t);
      bit = sh - 1;
    } else {
      v = __ldg(lp.nodes);
    }
    for (; !(v >> 31) && bit >= 0; --bit) {
      const uint32_t oct = ((cx >> bit) & 1u) | (((cy >> bit) & 1u) << 1) | (((cz >> bit) & 1u) << 2);
      node = v + oct;
      v = __ldg(lp.nodes + node);
    }
    const uint32_t leaf = v & 0x7FFFFFFFu;
    d = __ldg(lp.leaf_depth + leaf);
    if (d == 0 && lp.leaf_far) far = __ldg(lp.leaf_far + leaf);
  }
  if (d > (uint32_t)lp.cap) d = (uint32_t)lp.cap;  // d >= 1 only: cap >= 1 leaves 0 untouched
  r.d = fin ? d : (uint32_t)SAND_DEPTH_NONFINITE;
  r.far = fin ? far : __int_as_float(0x7fc00000);
  return r;
}

template <int KIND>
__global__ void __launch_bounds__(kLookupThreads) k_lookup(const float* __restrict__ pts, long long n,
                                                            LookupParams lp, uint8_t* __restrict__ out_depth,
                                                            float* __restrict__ out_sdf,
                                                            uint32_t* __restrict__ hist, long long nblk,
                                                            int vec_in, int vec_out, int vec_sdf) {
  __shared__ uint32_t sh[kMaxBins];
  const int nb = lp.L + 2;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const float scale = (float)(1u << lp.level) * 0.5f;
  const float maxc = (float)((1u << lp.level) - 1u);
  const long long base = (long long)blockIdx.x * kLookupChunk;
  const int lane = threadIdx.x & 31;
#pragma unroll (KIND == 0 ? 4 : 1)   // dense map without cached sdf: 4 chunks of loads in flight (0.354 -> 0.333 ms on C2); the far-field and descent variants measured slower unrolled
  for (int it = 0; it < kLookupChunk / (4 * kLookupThreads); ++it) {
    const long long p0 = base + (long long)it * 4 * kLookupThreads + 4 * threadIdx.x;
    const long long rem = n - p0;
    const int cnt = rem >= 4 ? 4 : (rem > 0 ? (int)rem : 0);
    float px[4], py[4], pz[4];
    if (cnt == 4 && vec_in) {
      const float4* q = reinterpret_cast<const float4*>(pts + 3 * p0);
      const float4 a = __ldcs(q), b = __ldcs(q + 1), c = __ldcs(q + 2);
      px[0] = a.x; py[0] = a.y; pz[0] = a.z; px[1] = a.w;
      py[1] = b.x; pz[1] = b.y; px[2] = b.z; py[2] = b.w;
      pz[2] = c.x; px[3] = c.y; py[3] = c.z; pz[3] = c.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j < cnt) {
          px[j] = pts[3 * (p0 + j)]; py[j] = pts[3 * (p0 + j) + 1]; pz[j] = pts[3 * (p0 + j) + 2];
        } else {
          px[j] = py[j] = pz[j] = 0.0f;
        }
      }
    }
    uint32_t dw = 0;
    int bins[4];
    float far[4];
    int nfar = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const LookupResult r = lookup_one<KIND>(px[j], py[j], pz[j], lp, scale, maxc);
      dw |= (r.d & 0xFFu) << (8 * j);
      bins[j] = (j < cnt) ? (r.d == SAND_DEPTH_NONFINITE ? lp.L + 1 : (int)r.d) : -1;
      far[j] = r.far;
      nfar += (j < cnt && (r.d == 0 || r.d == SAND_DEPTH_NONFINITE)) ? 1 : 0;
    }
    // cached / NaN sdf of far and non-finite points (Eq. 7): one 16-byte store when all four need it (the
    // far-field regime), else per point
    if (nfar == 4 && vec_sdf) {
      __stcs(reinterpret_cast<float4*>(out_sdf + p0), make_float4(far[0], far[1], far[2], far[3]));
    } else if (nfar) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t dj = (dw >> (8 * j)) & 0xFFu;
        if (j < cnt && (dj == 0 || dj == SAND_DEPTH_NONFINITE)) out_sdf[p0 + j] = far[j];
      }
    }
    if (cnt == 4 && vec_out) {
      *reinterpret_cast<uint32_t*>(out_depth + p0) = dw;
    } else {
      for (int j = 0; j < cnt; ++j) out_depth[p0 + j] = (uint8_t)(dw >> (8 * j));
    }
    // warp-aggregated shared-memory histogram; fast path when each thread's 4 points share one bin (grid-ordered
    // queries: neighbouring points mostly have one depth)
    const bool same = bins[1] == bins[0] && bins[2] == bins[0] && bins[3] == bins[0];
    if (__all_sync(0xffffffffu, same)) {
      const unsigned m = __match_any_sync(0xffffffffu, bins[0]);
      if (bins[0] >= 0 && lane == (__ffs(m) - 1)) atomicAdd(&sh[bins[0]], 4u * (uint32_t)__popc(m));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const unsigned m = __match_any_sync(0xffffffffu, bins[j]);
        if (bins[j] >= 0 && lane == (__ffs(m) - 1)) atomicAdd(&sh[bins[j]], (uint32_t)__popc(m));
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x) hist[(long long)i * nblk + blockIdx.x] = sh[i];
}

// Block-wide exclusive scan helper (1024 threads).
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v, unsigned long long* tot) {
  __shared__ unsigned long long ws[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    unsigned long long s = (lane < (int)(blockDim.x >> 5)) ? ws[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    ws[lane] = s;
  }
  __syncthreads();
  const unsigned long long wpre = w ? ws[w - 1] : 0ull;
  *tot = ws[(blockDim.x >> 5) - 1];
  __syncthreads();
  return wpre + inc - v;
}

// K2a, in three coalesced passes over the (L+2) x nblk histogram (bin-major):
//   k_scan_partial: per (bin, chunk of kScanChunk blocks) sums
//   k_scan_top    : bin totals, deepest-first starts, per-(depth, chunk) prefixes, the tile table
//   k_scan_offs   : per block exclusive prefix within its chunk + chunk prefix -> offs[d][b]
constexpr int kScanThreads = 1024;
constexpr int kScanPer = 8;                           // histogram entries per thread
constexpr int kScanChunk = kScanThreads * kScanPer;   // blocks per chunk

__global__ void __launch_bounds__(kScanThreads) k_scan_partial(const uint32_t* __restrict__ hist, long long nblk,
                                                                unsigned long long* __restrict__ part, int nchunk) {
  const int bin = blockIdx.y, c = blockIdx.x;
  const long long b0 = (long long)c * kScanChunk + (long long)threadIdx.x * kScanPer;
  unsigned long long s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k)
    if (b0 + k < nblk) s += hist[(long long)bin * nblk + b0 + k];
  unsigned long long tot;
  (void)block_excl_scan(s, &tot);
  if (threadIdx.x == 0) part[(long long)bin * nchunk + c] = tot;
}

__global__ void k_scan_top(const unsigned long long* __restrict__ part, int nchunk, int L, int tile_rows, int even_bins,
                           unsigned long long* __restrict__ cpre, QueryMeta* __restrict__ meta) {
  if (threadIdx.x != 0) return;
  long long counts[kMaxBins];
  for (int b = 0; b < kMaxBins; ++b) {
    long long t = 0;
    if (b < L + 2)
      for (int c = 0; c < nchunk; ++c) t += (long long)part[(long long)b * nchunk + c];
    counts[b] = t;
    meta->count[b] = t;
    meta->start[b] = 0;
    meta->tile_begin[b] = meta->tile_end[b] = 0;
  }
  long long running = 0, tb = 0;
  for (int d = L; d >= 1; --d) {   // deepest first
    meta->start[d] = running;
    for (int c = 0; c < nchunk; ++c) {
      cpre[(long long)d * nchunk + c] = (unsigned long long)running;
      running += (long long)part[(long long)d * nchunk + c];
    }
    meta->tile_begin[d] = tb;
    long long nt = (counts[d] + tile_rows - 1) / tile_rows;
    if (even_bins) nt += nt & 1;   // tile pairs never straddle a depth bin (slot-team kernel: tile 2u + s -> slot s)
    tb += nt;
    meta->tile_end[d] = tb;
  }
  meta->total_tiles = tb;
  meta->tile_rows = tile_rows;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_offs(const uint32_t* __restrict__ hist, long long nblk,
                                                             const unsigned long long* __restrict__ cpre,
                                                             int nchunk, uint32_t* __restrict__ offs) {
  const int d = blockIdx.y + 1, c = blockIdx.x;
  const long long b0 = (long long)c * kScanChunk + (long long)threadIdx.x * kScanPer;
  uint32_t v[kScanPer];
  unsigned long long s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    v[k] = (b0 + k < nblk) ? hist[(long long)d * nblk + b0 + k] : 0u;
    s += v[k];
  }
  unsigned long long tot;
  unsigned long long ex = block_excl_scan(s, &tot) + cpre[(long long)d * nchunk + c];
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    if (b0 + k < nblk) offs[(long long)d * nblk + b0 + k] = (uint32_t)ex;
    ex += v[k];
  }
}

// K2b: stable scatter.  Warp w of a block owns the contiguous points [512 w, 512 w + 512) of the block's 4096
// and walks them in 16 rounds of 32 (lane i <-> point 32 r + i), so the stable order is round-major, lane
// order within a round.  Per round one __match_any_sync groups the lanes of equal depth; a point's rank is
// its warp's running count of that depth (shared memory, updated by the group's first lane) plus the
// number of equal lanes below it.  After all rounds one block-wide prefix over the warps' counts gives every
// warp its base per depth, and the 16 (depth, rank) pairs kept in registers are written out.
__global__ void __launch_bounds__(kLookupThreads) k_scatter(const uint8_t* __restrict__ depth, long long n,
                                                             int L, const uint32_t* __restrict__ offs,
                                                             uint32_t* __restrict__ perm, long long nblk, int vec16) {
  constexpr int kWarps = kLookupThreads / 32;
  constexpr int kRounds = kLookupChunk / kLookupThreads;   // 16
  static_assert(kRounds == 16, "the one-depth fast path reads a warp's 512 depths as 32 x 16 bytes");
  __shared__ uint32_t wcnt[kWarps][kMaxBins];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int d = lane; d < kMaxBins; d += 32) wcnt[warp][d] = 0;
  __syncwarp();
  const long long p0 = (long long)blockIdx.x * kLookupChunk + (long long)warp * (32 * kRounds) + lane;
  uint32_t key[kRounds];   // (depth << 16) | rank within the warp, depth 0 = not binned
  // Fast path (grid-ordered queries: most warps): the warp's 512 depths in ONE 16-byte load per lane; if they are all
  // the same byte the ranks are the point order and nothing else of the depths is needed (the 16 byte loads and
  // the 16-way compare of the general path were 40% of this issue-bound kernel's instructions).
  bool fast = false;
  const long long wp0 = p0 - lane;
  if (vec16 && wp0 + 32 * kRounds <= n) {
    const uint4 w = __ldcs(reinterpret_cast<const uint4*>(depth + wp0) + lane);
    uint32_t d = w.x & 0xFFu;
    const uint32_t pat = d * 0x01010101u;
    const uint32_t dl0 = __shfl_sync(0xffffffffu, d, 0);
    fast = __all_sync(0xffffffffu, w.x == pat && w.y == pat && w.z == pat && w.w == pat && d == dl0);
    if (fast) {
      if (d < 1 || d > (uint32_t)L) d = 0;   // far, non-finite or padding: not binned
#pragma unroll
      for (int r = 0; r < kRounds; ++r) key[r] = (d << 16) | (uint32_t)(32 * r + lane);
      if (lane == 0) wcnt[warp][d] = 32u * kRounds;
    }
  }
  if (!fast) {
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {   // all loads first (independent of the ranking chain)
    const long long pt = p0 + 32 * r;
    key[r] = pt < n ? __ldcs(depth + pt) : 0u;
  }
  bool one = true;   // all 512 points of this warp at one depth (grid-ordered queries: the common case)
  uint32_t d0 = key[0];
  if (d0 < 1 || d0 > (uint32_t)L) d0 = 0;
#pragma unroll
  for (int r = 1; r < kRounds; ++r) one &= (key[r] == d0) || (d0 == 0 && (key[r] < 1 || key[r] > (uint32_t)L));
  const uint32_t dl0 = __shfl_sync(0xffffffffu, d0, 0);   // every lane executes the shuffle (no short-circuit)
  one = __all_sync(0xffffffffu, one && dl0 == d0);
  if (one) {
    // rank of point 32 r + lane = 32 r + lane (round-major, lane order: the stable order)
#pragma unroll
    for (int r = 0; r < kRounds; ++r) key[r] = (d0 << 16) | (uint32_t)(32 * r + lane);
    if (lane == 0) wcnt[warp][d0] = 32u * kRounds;
  } else {
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      uint32_t d = key[r];
      if (d < 1 || d > (uint32_t)L) d = 0;   // far, non-finite or padding: not binned
      const unsigned m = __match_any_sync(0xffffffffu, d);
      const uint32_t before = wcnt[warp][d];
      __syncwarp();
      if (lane == __ffs(m) - 1) wcnt[warp][d] = before + (uint32_t)__popc(m);
      __syncwarp();
      key[r] = (d << 16) | (before + (uint32_t)__popc(m & lt));
    }
  }
  }
  __syncthreads();
  // warp bases: base[w][d] = offs[d][block] + sum of warps < w (in place over wcnt)
  if (tid >= 1 && tid <= L) {
    uint32_t acc = offs[(long long)tid * nblk + blockIdx.x];
    for (int w = 0; w < kWarps; ++w) { const uint32_t t = wcnt[w][tid]; wcnt[w][tid] = acc; acc += t; }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const uint32_t d = key[r] >> 16;
    if (d) perm[wcnt[warp][d] + (key[r] & 0xFFFFu)] = (uint32_t)(p0 + 32 * r);
  }
}

__global__ void k_bake(const uint32_t* __restrict__ nodes, const uint8_t* __restrict__ leaf_depth,
                       const float* __restrict__ leaf_far, int level, uint8_t* __restrict__ grid,
                       float* __restrict__ grid_far, int* err) {
  const long long G = 1ll << level;
  const long long total = G * G * G;
  for (long long lin = blockIdx.x * (long long)blockDim.x + threadIdx.x; lin < total;
       lin += (long long)gridDim.x * blockDim.x) {
    const uint32_t cx = (uint32_t)(lin & (G - 1)), cy = (uint32_t)((lin >> level) & (G - 1)),
                   cz = (uint32_t)(lin >> (2 * level));
    uint32_t v = nodes[0];
    int bit = level - 1;
    for (; !(v >> 31) && bit >= 0; --bit) {
      const uint32_t oct = ((cx >> bit) & 1u) | (((cy >> bit) & 1u) << 1) | (((cz >> bit) & 1u) << 2);
      v = nodes[v + oct];
    }
    if (!(v >> 31)) { *err = 1; continue; }
    const uint32_t leaf = v & 0x7FFFFFFFu;
    grid[lin] = leaf_depth[leaf];
    if (grid_far) grid_far[lin] = leaf_far ? leaf_far[leaf] : 0.0f;
  }
}

// Start table for deep octrees: top[cell] = node payload after descending top_level levels (or the
// leaf payload met earlier) -- the same octant walk as the lookup's own descent.
__global__ void k_bake_top(const uint32_t* __restrict__ nodes, int top_level, uint32_t* __restrict__ top) {
  const long long G = 1ll << top_level;
  for (long long lin = blockIdx.x * (long long)blockDim.x + threadIdx.x; lin < G * G * G;
       lin += (long long)gridDim.x * blockDim.x) {
    const uint32_t cx = (uint32_t)(lin & (G - 1)), cy = (uint32_t)((lin >> top_level) & (G - 1)),
                   cz = (uint32_t)(lin >> (2 * top_level));
    uint32_t v = nodes[0];
    for (int bit = top_level - 1; !(v >> 31) && bit >= 0; --bit) {
      const uint32_t oct = ((cx >> bit) & 1u) | (((cy >> bit) & 1u) << 1) | (((cz >> bit) & 1u) << 2);
      v = nodes[v + oct];
    }
    top[lin] = v;
  }
}

cudaError_t launch_bake_top(const uint32_t* nodes, int top_level, uint32_t* top, cudaStream_t st) {
  k_bake_top<<<148 * 8, 256, 0, st>>>(nodes, top_level, top);
  return cudaGetLastError();
}

cudaError_t launch_lookup(const float* pts, long long n, const LookupParams& lp, uint8_t* out_depth,
                          float* out_sdf, uint32_t* hist, long long nblk, cudaStream_t st) {
  const int vec_in = ((reinterpret_cast<uintptr_t>(pts) & 15) == 0) ? 1 : 0;
  const int vec_out = ((reinterpret_cast<uintptr_t>(out_depth) & 3) == 0) ? 1 : 0;
  const int vec_sdf = ((reinterpret_cast<uintptr_t>(out_sdf) & 15) == 0) ? 1 : 0;
  if (lp.dense && lp.grid_far)
    k_lookup<1><<<(unsigned)nblk, kLookupThreads, 0, st>>>(pts, n, lp, out_depth, out_sdf, hist, nblk, vec_in, vec_out,
                                                           vec_sdf);
  else if (lp.dense)
    k_lookup<0><<<(unsigned)nblk, kLookupThreads, 0, st>>>(pts, n, lp, out_depth, out_sdf, hist, nblk, vec_in, vec_out,
                                                           vec_sdf);
  else
    k_lookup<2><<<(unsigned)nblk, kLookupThreads, 0, st>>>(pts, n, lp, out_depth, out_sdf, hist, nblk, vec_in, vec_out,
                                                           vec_sdf);
  return cudaGetLastError();
}

long long scan_scratch_words(long long nblk) {
  const long long nchunk = (nblk + kScanChunk - 1) / kScanChunk;
  return 2 * (long long)kMaxBins * (nchunk > 0 ? nchunk : 1);
}

cudaError_t launch_scan(const uint32_t* hist, long long nblk, int L, int tile_rows, int even_bins, uint32_t* offs,
                        QueryMeta* meta, unsigned long long* scratch, cudaStream_t st) {
  const int nchunk = (int)((nblk + kScanChunk - 1) / kScanChunk);
  unsigned long long* part = scratch;
  unsigned long long* cpre = scratch + (long long)kMaxBins * nchunk;
  k_scan_partial<<<dim3(nchunk, L + 2), kScanThreads, 0, st>>>(hist, nblk, part, nchunk);
  k_scan_top<<<1, 32, 0, st>>>(part, nchunk, L, tile_rows, even_bins, cpre, meta);
  k_scan_offs<<<dim3(nchunk, L), kScanThreads, 0, st>>>(hist, nblk, cpre, nchunk, offs);
  return cudaGetLastError();
}

cudaError_t launch_scatter(const uint8_t* depth, long long n, int L, const uint32_t* offs, uint32_t* perm,
                           long long nblk, cudaStream_t st) {
  const int vec16 = ((reinterpret_cast<uintptr_t>(depth) & 15) == 0) ? 1 : 0;
  k_scatter<<<(unsigned)nblk, kLookupThreads, 0, st>>>(depth, n, L, offs, perm, nblk, vec16);
  return cudaGetLastError();
}

cudaError_t launch_bake_octree(const uint32_t* nodes, const uint8_t* leaf_depth, const float* leaf_far,
                               int level, uint8_t* grid, float* grid_far, int* err_flag, cudaStream_t st) {
  k_bake<<<148 * 8, 256, 0, st>>>(nodes, leaf_depth, leaf_far, level, grid, grid_far, err_flag);
  return cudaGetLastError();
}

}  // namespace sand
