// depthpop.cu -- volumetric network-depth map population on the GPU.
//
// PAPER.md Sec. 3.2: the required network depth of a point (Eq. 5)
//     d(x) = min{ i : |y_L(x) - y_i(x)| < r  and  sign(y_i(x)) = sign(y_L(x)) }      (near, delta = 1)
//     d(x) = min{ i : sign(y_i(x)) = sign(y_L(x)) }                                   (far,  delta = 0)
// and the leaf depth (Eq. 6) d(N) = max over the leaf's sample points of d(x).
//
// Eq. 5 compares cumulative outputs against r (1.5e-4 in the paper), far below the BF16 path's
// error, so the full-depth evaluation here is FP32 (sine to ~5e-7, dp_sin), whatever the context's precision.
// k_required_depth: persistent blocks of 256 threads over tiles of 64 points; every layer is a register-
// blocked FP32 GEMM (thread = 8 points x ceil(H/32) units, W^T double-buffered in shared memory by cp.async, 16 rows at a
// time, activations transposed [unit][point] in shared memory) with the sine, tail and running y_i
// fused; after layer L each point's d(x) is decided from its y_1..y_L.  k_leaf_max: Eq. 6 pooling.
#include <cstdint>
#include <cuda_runtime.h>

#include "sand_internal.h"

namespace sand {

constexpr int kDpP = 64;          // points per tile
constexpr int kDpS = 68;          // row stride of the [unit][point] activations: 16-byte rows, 4-way (not
                                  // 32-way) bank conflicts when the 32 lanes of a warp touch 32 units
constexpr int kDpThreads = 256;   // 8 point groups (warps) x 32 unit lanes (512 measured slower: more loads per FMA)
constexpr int kDpPPW = kDpP / (kDpThreads / 32);   // points per warp
constexpr int kDpKC = 32;         // W^T rows staged per step (16: 2.6% slower)

template <int H>
struct DpShape {
  static constexpr int U = (H + 31) / 32;                    // units per thread
  static constexpr int HP = U * 32;                          // padded unit count
  static constexpr int KC = H > 256 ? 8 : kDpKC;             // W^T rows per stage (H = 336: fit 227 KB)
  static constexpr size_t SMEM = (size_t)2 * HP * kDpS * 4   // h ping-pong, [unit][point]
                                 + (size_t)2 * KC * HP * 4;  // W^T stages, double-buffered
};

// 16-byte global -> shared async copy (no register staging), completion by commit / wait groups
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// sin(x) to ~4e-7 absolute: two-constant Cody-Waite reduction to [-pi, pi] (k = rint(x / 2pi),
// 2pi = hi + lo with hi = fl32(2pi)), then MUFU.SIN, whose error on [-pi, pi] is ~2^-21.4 -- FP32-grade
// for the |x| <~ 100 of a SIREN layer, at a quarter of the instructions of the libm sinf path.
__device__ __forceinline__ float dp_sin(float x) {
  const float k = rintf(x * 0.159154943091895f);
  float r = fmaf(-k, 6.28318548202514648f, x);
  r = fmaf(-k, -1.7484555314695172e-7f, r);
  return __sinf(r);
}

// ---- building blocks shared by the kernels below (one 64-point tile, activations [unit][point])
// W^T rows [k0, k0 + KC) of a layer -> stage buffer b (H % 16 == 0: rows are whole float4s)
template <int H>
__device__ __forceinline__ void dp_stage(float* ws, const float* W, int k0, int b, int tid) {
  using C = DpShape<H>;
  constexpr int RV = H / 4;
  for (int i = tid; i < C::KC * RV; i += kDpThreads) {
    const int kk = i / RV, j4 = i % RV;
    cp_async16(ws + (b * C::KC + kk) * C::HP + 4 * j4, W + (size_t)(k0 + kk) * H + 4 * j4);
  }
  cp_async_commit();
}

// hout[j][p] = sin(w0 (W h_in)[j][p] + w0 b[j]) for a hidden layer (W^T given, [k][j]); register-blocked
// FP32 GEMM, W^T streamed through two cp.async stages.  Ends with the block synchronised.
template <int H>
__device__ __forceinline__ void dp_hidden(const float* W, const float* bias, float w0, const float* hin, float* hout,
                                          float* ws, int tid) {
  using C = DpShape<H>;
  const int tj = tid & 31, tp = tid >> 5;
  // accumulators for point pairs: one FFMA2 does two points' FMA of the same weight (half the issue slots
  // of scalar FFMA for the same FMA-pipe work)
  float2 acc[kDpPPW / 2][C::U];
#pragma unroll
  for (int a = 0; a < kDpPPW / 2; ++a)
#pragma unroll
    for (int u = 0; u < C::U; ++u) acc[a][u] = make_float2(0.f, 0.f);
  __syncthreads();   // previous users of both stage buffers are done
  dp_stage<H>(ws, W, 0, 0, tid);
  for (int k0 = 0, b = 0; k0 < H; k0 += C::KC, b ^= 1) {
    if (k0 + C::KC < H) {
      dp_stage<H>(ws, W, k0 + C::KC, b ^ 1, tid);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* wsb = ws + b * C::KC * C::HP;
#pragma unroll 4
    for (int kk = 0; kk < C::KC; ++kk) {
      float2 hv[kDpPPW / 2];
#pragma unroll
      for (int q4 = 0; q4 < kDpPPW / 4; ++q4) {
        const float4 hq = *reinterpret_cast<const float4*>(hin + (k0 + kk) * kDpS + tp * kDpPPW + 4 * q4);
        hv[2 * q4] = make_float2(hq.x, hq.y);
        hv[2 * q4 + 1] = make_float2(hq.z, hq.w);
      }
#pragma unroll
      for (int u = 0; u < C::U; ++u) {
        const float w = wsb[kk * C::HP + tj + 32 * u];
        const float2 w2 = make_float2(w, w);
#pragma unroll
        for (int a = 0; a < kDpPPW / 2; ++a) acc[a][u] = __ffma2_rn(w2, hv[a], acc[a][u]);
      }
    }
    __syncthreads();   // stage b is overwritten by the copy issued next iteration
  }
#pragma unroll
  for (int u = 0; u < C::U; ++u) {
    const int j = tj + 32 * u;
    const float bb = j < H ? bias[j] : 0.f;
#pragma unroll
    for (int a = 0; a < kDpPPW / 2; ++a) {
      hout[j * kDpS + tp * kDpPPW + 2 * a] = j < H ? dp_sin(fmaf(acc[a][u].x, w0, bb)) : 0.f;
      hout[j * kDpS + tp * kDpPPW + 2 * a + 1] = j < H ? dp_sin(fmaf(acc[a][u].y, w0, bb)) : 0.f;
    }
  }
  __syncthreads();
}

// t_l of every tile point (LINEAR: a . h + c;  MULT, l >= 2: (a . h + c)(a1 . h + c1)) -> tl[p]
template <int H, int TAIL>
__device__ __forceinline__ void dp_tails(const MlpDev& m, int l, const float* hcur, float* tl, int tid) {
  const int tj = tid & 31, tp = tid >> 5;
  const float* a_t = m.tables + m.off_a;
  const float* a1_t = m.tables + m.off_a1;
  const float* c_t = m.tables + m.off_c;
  const float* c1_t = m.tables + m.off_c1;
  for (int pp = 0; pp < kDpPPW; ++pp) {
    const int p = tp * kDpPPW + pp;
    float s0 = 0.f, s1 = 0.f;
    for (int j = tj; j < H; j += 32) {
      const float h = hcur[j * kDpS + p];
      s0 = fmaf(a_t[(l - 1) * H + j], h, s0);
      if (TAIL == SAND_TAIL_MULT && l >= 2) s1 = fmaf(a1_t[(l - 2) * H + j], h, s1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (tj == 0) {
      float t = s0 + c_t[l - 1];
      if (TAIL == SAND_TAIL_MULT && l >= 2) t *= s1 + c1_t[l - 2];
      tl[p] = t;
    }
  }
}

// Dynamic exit with re-compaction (SURVEY 8(f) NEXT #3 as the north star states it): a block owns pools
// of kDynPool points and runs them layer-synchronously -- every layer over the pool's still-running
// points only, packed into full 64-point tiles (the survivors' slots are compacted after each layer),
// with their activations parked in a per-block global scratch hbuf[slot][HP] between layers (L2-
// resident).  The work is the sum of the exit layers, not a tile's slowest point.
constexpr int kDynPool = 512;
#ifndef SAND_DYN_ABL
#define SAND_DYN_ABL 0   // timing ablation (wrong results): 1 = no activation gather / park
#endif

template <int H, int TAIL>
__global__ void __launch_bounds__(kDpThreads, 1) k_dynamic_pool(MlpDev m, const float* __restrict__ w_t,
                                                                const float* __restrict__ pts, long long n, float r,
                                                                float* __restrict__ out_sdf,
                                                                uint8_t* __restrict__ out_dep,
                                                                float* __restrict__ hbuf_all) {
  using C = DpShape<H>;
  extern __shared__ __align__(16) float sm[];
  float* hA = sm;                               // [HP][kDpS]: this tile's h_{l-1}
  float* hB = hA + C::HP * kDpS;                // [HP][kDpS]: this tile's h_l
  float* ws = hB + C::HP * kDpS;                // [2][KC][HP]
  __shared__ float px[3][kDpP];
  __shared__ float tl[kDpP];
  __shared__ int act[kDynPool];                 // running slots, packed
  __shared__ float ybuf[kDynPool];              // y_l per slot
  __shared__ int keep[kDynPool];                // scan scratch for the compaction
  __shared__ int s_nact;
  const int L = m.L;
  const float w0 = m.omega0;
  const int tid = threadIdx.x;
  const float4* w1 = reinterpret_cast<const float4*>(m.tables + m.off_w1);
  const float* bias_t = m.tables + m.off_bias;
  float* hbuf = hbuf_all + (size_t)blockIdx.x * kDynPool * C::HP;
  for (int i = tid; i < 2 * C::KC * C::HP; i += kDpThreads) ws[i] = 0.f;
  const long long npool = (n + kDynPool - 1) / kDynPool;
  for (long long pool = blockIdx.x; pool < npool; pool += gridDim.x) {
    const long long base = pool * kDynPool;
    const int cnt = (int)min((long long)kDynPool, n - base);
    __syncthreads();
    // non-finite points leave at once; the others start running
    if (tid == 0) s_nact = 0;
    __syncthreads();
    for (int q = tid; q < kDynPool; q += kDpThreads) {
      int run = 0;
      if (q < cnt) {
        const float x = pts[3 * (base + q)], y = pts[3 * (base + q) + 1], z = pts[3 * (base + q) + 2];
        run = isfinite(x) && isfinite(y) && isfinite(z);
        if (!run) { out_dep[base + q] = 255; out_sdf[base + q] = __int_as_float(0x7fc00000); }
      }
      keep[q] = run;
      ybuf[q] = 0.f;
    }
    __syncthreads();
    if (tid == 0) {   // serial stable compaction (kDynPool entries; negligible against a layer's GEMM)
      int k = 0;
      for (int q = 0; q < cnt; ++q) if (keep[q]) act[k++] = q;
      s_nact = k;
    }
    __syncthreads();
    for (int l = 1; l <= L && s_nact > 0; ++l) {
      const int nact = s_nact;
      for (int t0 = 0; t0 < nact; t0 += kDpP) {
        const int np = min(kDpP, nact - t0);
        if (l == 1) {
          for (int i = tid; i < 3 * kDpP; i += kDpThreads) {
            const int p = i / 3, c = i % 3;
            px[c][p] = p < np ? pts[3 * (base + act[t0 + p]) + c] : 0.f;
          }
          __syncthreads();
          for (int i = tid; i < C::HP * kDpP; i += kDpThreads) {
            const int j = i / kDpP, p = i % kDpP;
            float h = 0.f;
            if (j < H) {
              const float4 w = w1[j];
              h = dp_sin(fmaf(w.z, px[2][p], fmaf(w.y, px[1][p], fmaf(w.x, px[0][p], w.w))));
            }
            hB[j * kDpS + p] = h;
          }
          __syncthreads();
        } else {
          // gather h_{l-1} of the tile's slots: float4 loads, all of a thread's loads in flight at once
          constexpr int NV = kDpP * C::HP / 4 / kDpThreads;   // float4 per thread
          float4 v[NV];
#pragma unroll
          for (int u = 0; u < NV; ++u) {
            const int i = tid + u * kDpThreads, p = i / (C::HP / 4), j4 = i % (C::HP / 4);
            v[u] = (p < np && SAND_DYN_ABL != 1)
                       ? *reinterpret_cast<const float4*>(hbuf + (size_t)act[t0 + p] * C::HP + 4 * j4)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < NV; ++u) {
            const int i = tid + u * kDpThreads, p = i / (C::HP / 4), j = 4 * (i % (C::HP / 4));
            hA[j * kDpS + p] = v[u].x;
            hA[(j + 1) * kDpS + p] = v[u].y;
            hA[(j + 2) * kDpS + p] = v[u].z;
            hA[(j + 3) * kDpS + p] = v[u].w;
          }
          dp_hidden<H>(w_t + (size_t)(l - 2) * H * H, bias_t + (size_t)(l - 2) * H, w0, hA, hB, ws, tid);
        }
        dp_tails<H, TAIL>(m, l, hB, tl, tid);
        __syncthreads();
        if (tid < np) {
          const int q = act[t0 + tid];
          const float y = ybuf[q] + tl[tid];
          ybuf[q] = y;
          const bool stop = l == L || (l >= 2 && fabsf(tl[tid]) < r);
          if (stop) { out_sdf[base + q] = y; out_dep[base + q] = (uint8_t)l; }
          keep[t0 + tid] = !stop;
        }
        if (l < L && SAND_DYN_ABL != 1)   // park h_l of the tile's slots for the next layer (float4 stores)
          for (int i = tid; i < kDpP * C::HP / 4; i += kDpThreads) {
            const int p = i / (C::HP / 4), j = 4 * (i % (C::HP / 4));
            if (p < np)
              *reinterpret_cast<float4*>(hbuf + (size_t)act[t0 + p] * C::HP + j) =
                  make_float4(hB[j * kDpS + p], hB[(j + 1) * kDpS + p], hB[(j + 2) * kDpS + p], hB[(j + 3) * kDpS + p]);
          }
        __syncthreads();
      }
      if (tid == 0) {
        int k = 0;
        for (int q = 0; q < nact; ++q) if (keep[q]) act[k++] = act[q];
        s_nact = k;
      }
      __syncthreads();
    }
  }
}

// FP32 adaptive query for wide nets (SAND_FP32 contexts with H >= 128; the one-thread-per-point SIMT
// kernel keeps H <= 64): the binned 128-row tiles of uniform depth d (K2), each as two 64-point
// sub-tiles evaluated to layer d with the register-blocked FP32 GEMM above; y_d -> out[perm[row]].
template <int H, int TAIL>
__global__ void __launch_bounds__(kDpThreads, 1) k_query_fp32(MlpDev m, const float* __restrict__ w_t,
                                                              const float* __restrict__ pts,
                                                              const uint32_t* __restrict__ perm,
                                                              const QueryMeta* __restrict__ meta,
                                                              float* __restrict__ out) {
  using C = DpShape<H>;
  extern __shared__ __align__(16) float sm[];
  float* hA = sm;
  float* hB = hA + C::HP * kDpS;
  float* ws = hB + C::HP * kDpS;
  __shared__ float px[3][kDpP];
  __shared__ float tl[kDpP];
  __shared__ float yv[kDpP];
  __shared__ uint32_t idx[kDpP];
  __shared__ long long s_tile_end[kMaxBins], s_tile_begin[kMaxBins], s_start[kMaxBins], s_count[kMaxBins];
  const int L = m.L, tid = threadIdx.x;
  const float w0 = m.omega0;
  const float4* w1 = reinterpret_cast<const float4*>(m.tables + m.off_w1);
  const float* bias_t = m.tables + m.off_bias;
  for (int i = tid; i < 2 * C::KC * C::HP; i += kDpThreads) ws[i] = 0.f;
  if (tid < kMaxBins) {
    s_tile_end[tid] = meta->tile_end[tid];
    s_tile_begin[tid] = meta->tile_begin[tid];
    s_start[tid] = meta->start[tid];
    s_count[tid] = meta->count[tid];
  }
  __syncthreads();
  const long long T = meta->total_tiles;
  for (long long t = blockIdx.x; t < T; t += gridDim.x) {
    int d = 0;
    for (int dd = L; dd >= 1; --dd)
      if (t < s_tile_end[dd]) { d = dd; break; }
    const long long rend = s_start[d] + s_count[d];
    for (int sub = 0; sub < kTileM / kDpP; ++sub) {
      const long long r0 = s_start[d] + (t - s_tile_begin[d]) * kTileM + (long long)sub * kDpP;
      const int np = (int)min((long long)kDpP, rend - r0);
      if (np <= 0) break;
      __syncthreads();
      if (tid < kDpP) {
        idx[tid] = tid < np ? perm[r0 + tid] : 0u;
        yv[tid] = 0.f;
      }
      __syncthreads();
      for (int i = tid; i < 3 * kDpP; i += kDpThreads) {
        const int p = i / 3, c = i % 3;
        px[c][p] = p < np ? pts[3ll * idx[p] + c] : 0.f;
      }
      __syncthreads();
      for (int i = tid; i < C::HP * kDpP; i += kDpThreads) {   // layer 1 (K = 3)
        const int j = i / kDpP, p = i % kDpP;
        float h = 0.f;
        if (j < H) {
          const float4 w = w1[j];
          h = dp_sin(fmaf(w.z, px[2][p], fmaf(w.y, px[1][p], fmaf(w.x, px[0][p], w.w))));
        }
        hA[j * kDpS + p] = h;
      }
      __syncthreads();
      dp_tails<H, TAIL>(m, 1, hA, tl, tid);
      __syncthreads();
      if (tid < kDpP) yv[tid] += tl[tid];
      float* hin = hA;
      float* hout = hB;
      for (int l = 2; l <= d; ++l) {
        dp_hidden<H>(w_t + (size_t)(l - 2) * H * H, bias_t + (size_t)(l - 2) * H, w0, hin, hout, ws, tid);
        dp_tails<H, TAIL>(m, l, hout, tl, tid);
        __syncthreads();
        if (tid < kDpP) yv[tid] += tl[tid];
        float* x = hin; hin = hout; hout = x;
      }
      __syncthreads();
      if (tid < np) out[idx[tid]] = yv[tid];
    }
  }
}

// MODE 0: Eq. 5 required depth of every point (full-depth evaluation, decision after layer L).
// MODE 1: dynamic exit without a depth map ('SAND w/o Octree'; R23): a point stops at
//   the first layer i >= 2 with |t_i| < r (else L) and returns y_i; a tile stops computing as soon as all
//   of its points have stopped (tile-level early exit; no re-compaction across tiles).
template <int H, int TAIL, int MODE>
__global__ void __launch_bounds__(kDpThreads, 1) k_required_depth(MlpDev m, const float* __restrict__ w_t,
                                                                  const float* __restrict__ pts, long long n,
                                                                  float r, int near, uint8_t* __restrict__ out,
                                                                  float* __restrict__ out_sdf) {
  using C = DpShape<H>;
  extern __shared__ __align__(16) float sm[];
  float* hA = sm;                               // [HP][kDpS]
  float* hB = hA + C::HP * kDpS;
  float* ws = hB + C::HP * kDpS;                // [2][C::KC][HP] (columns >= H stay zero)
  __shared__ float ys[32][kDpP];                // y_i per point (L <= 32)
  __shared__ float px[3][kDpP];
  __shared__ float tl[kDpP];                    // MODE 1: t_l of the current layer
  __shared__ int xit[kDpP];                     // MODE 1: 0 running, l = stopped after layer l, 255 none
  const int L = m.L;
  const float w0 = m.omega0;
  const int tid = threadIdx.x, tj = tid & 31, tp = tid >> 5;   // warp = point group
  const float4* w1 = reinterpret_cast<const float4*>(m.tables + m.off_w1);
  const float* bias_t = m.tables + m.off_bias;   // [L-1][H], w0 * b_i
  const float* a_t = m.tables + m.off_a;         // [L][H]
  const float* a1_t = m.tables + m.off_a1;       // [L-1][H] (MULT)
  const float* c_t = m.tables + m.off_c;         // [L]
  const float* c1_t = m.tables + m.off_c1;       // [L-1] (MULT)
  const long long ntiles = (n + kDpP - 1) / kDpP;
  for (int i = tid; i < 2 * C::KC * C::HP; i += kDpThreads) ws[i] = 0.f;
  __syncthreads();
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long p0 = tile * kDpP;
    for (int i = tid; i < 3 * kDpP; i += kDpThreads) {
      const int p = i / 3, c = i % 3;
      px[c][p] = (p0 + p < n) ? pts[3 * (p0 + p) + c] : 0.f;
    }
    __syncthreads();
    if (MODE == 1 && tid < kDpP)
      xit[tid] = (p0 + tid < n && isfinite(px[0][tid]) && isfinite(px[1][tid]) && isfinite(px[2][tid])) ? 0 : 255;
    // ---- layer 1 (K = 3) + tail 1
    for (int i = tid; i < C::HP * kDpP; i += kDpThreads) {
      const int j = i / kDpP, p = i % kDpP;
      float h = 0.f;
      if (j < H) {
        const float4 w = w1[j];
        h = dp_sin(fmaf(w.z, px[2][p], fmaf(w.y, px[1][p], fmaf(w.x, px[0][p], w.w))));
      }
      hA[j * kDpS + p] = h;
    }
    __syncthreads();
    auto tails = [&](int l, const float* hcur) {
      // t_l per point: warp tp reduces its kDpPPW points over all H units (lane = unit residue)
      for (int pp = 0; pp < kDpPPW; ++pp) {
        const int p = tp * kDpPPW + pp;
        float s0 = 0.f, s1 = 0.f;
        for (int j = tj; j < H; j += 32) {
          const float h = hcur[j * kDpS + p];
          s0 = fmaf(a_t[(l - 1) * H + j], h, s0);
          if (TAIL == SAND_TAIL_MULT && l >= 2) s1 = fmaf(a1_t[(l - 2) * H + j], h, s1);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          s0 += __shfl_xor_sync(0xffffffffu, s0, o);
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        }
        if (tj == 0) {
          float t = s0 + c_t[l - 1];
          if (TAIL == SAND_TAIL_MULT && l >= 2) t *= s1 + c1_t[l - 2];
          ys[l - 1][p] = (l == 1 ? 0.f : ys[l - 2][p]) + t;
          if (MODE == 1) tl[p] = t;
        }
      }
    };
    tails(1, hA);
    // ---- hidden layers: h_out[j][p] = sin(w0 * (W_l h_in)[j][p] + w0 b_l[j])
    float* hin = hA;
    float* hout = hB;
    for (int l = 2; l <= L; ++l) {
      dp_hidden<H>(w_t + (size_t)(l - 2) * H * H, bias_t + (size_t)(l - 2) * H, w0, hin, hout, ws, tid);
      tails(l, hout);
      float* t = hin; hin = hout; hout = t;
      if (MODE == 1 && l < L) {
        __syncthreads();
        int run = 0;
        if (tid < kDpP) {
          if (xit[tid] == 0 && fabsf(tl[tid]) < r) xit[tid] = l;
          run = xit[tid] == 0;
        }
        if (!__syncthreads_or(run)) break;   // every point of the tile has stopped
      }
    }
    __syncthreads();
    if (MODE == 1) {
      if (tid < kDpP && p0 + tid < n) {
        const int x = xit[tid];
        const int d = x == 0 ? L : x;
        out[p0 + tid] = (uint8_t)d;
        out_sdf[p0 + tid] = d == 255 ? __int_as_float(0x7fc00000) : ys[d - 1][tid];
      }
      __syncthreads();
      continue;
    }
    // ---- Eq. 5 decision per point
    if (tid < kDpP && p0 + tid < n) {
      const float yL = ys[L - 1][tid];
      const float sL = (yL > 0.f) - (yL < 0.f);
      int d = L;
      for (int i = 1; i < L; ++i) {
        const float yi = ys[i - 1][tid];
        const float si = (yi > 0.f) - (yi < 0.f);
        if (si == sL && (!near || fabsf(yL - yi) < r)) { d = i; break; }
      }
      out[p0 + tid] = (uint8_t)d;
    }
    __syncthreads();
  }
}

__global__ void k_leaf_max(const uint8_t* __restrict__ d, long long n_leaves, int spl, uint8_t* __restrict__ out) {
  const long long leaf = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (leaf >= n_leaves) return;
  uint32_t mx = 0;
  for (int s = 0; s < spl; ++s) mx = max(mx, (uint32_t)d[leaf * spl + s]);
  out[leaf] = (uint8_t)mx;
}

template <int H, int TAIL, int MODE>
static cudaError_t launch_rd_t(const MlpDev& m, const float* w_t, const float* pts, long long n, float r, int near,
                               uint8_t* out, float* out_sdf, int num_sms, cudaStream_t st) {
  const size_t sm = DpShape<H>::SMEM;
  cudaError_t e = cudaFuncSetAttribute(k_required_depth<H, TAIL, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const long long ntiles = (n + kDpP - 1) / kDpP;
  const int grid = (int)(ntiles < num_sms ? ntiles : num_sms);
  k_required_depth<H, TAIL, MODE><<<grid, kDpThreads, sm, st>>>(m, w_t, pts, n, r, near, out, out_sdf);
  return cudaGetLastError();
}

bool depthpop_supported(int H) {
  return H == 16 || H == 32 || H == 64 || H == 128 || H == 256 || H == 336;
}

static cudaError_t launch_dp(const MlpDev& m, const float* w_t, const float* pts, long long n, float r, int near,
                             uint8_t* out, float* out_sdf, int mode, int num_sms, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const bool mult = m.tail == SAND_TAIL_MULT;
#define SAND_DP_CASE(HH)                                                                                   \
  case HH:                                                                                                 \
    if (mode == 1)                                                                                         \
      return mult ? launch_rd_t<HH, 1, 1>(m, w_t, pts, n, r, near, out, out_sdf, num_sms, st)              \
                  : launch_rd_t<HH, 0, 1>(m, w_t, pts, n, r, near, out, out_sdf, num_sms, st);             \
    return mult ? launch_rd_t<HH, 1, 0>(m, w_t, pts, n, r, near, out, out_sdf, num_sms, st)                \
                : launch_rd_t<HH, 0, 0>(m, w_t, pts, n, r, near, out, out_sdf, num_sms, st);
  switch (m.H) {
    SAND_DP_CASE(16)
    SAND_DP_CASE(32)
    SAND_DP_CASE(64)
    SAND_DP_CASE(128)
    SAND_DP_CASE(256)
    SAND_DP_CASE(336)
    default: return cudaErrorInvalidValue;
  }
#undef SAND_DP_CASE
}

cudaError_t launch_required_depth(const MlpDev& m, const float* w_t, const float* pts, long long n, float r,
                                  int near, uint8_t* out, int num_sms, cudaStream_t st) {
  return launch_dp(m, w_t, pts, n, r, near, out, nullptr, 0, num_sms, st);
}

template <int H, int TAIL>
static cudaError_t launch_pool_t(const MlpDev& m, const float* w_t, const float* pts, long long n, float r,
                                 float* out_sdf, uint8_t* out_depth, float* hbuf, int grid, cudaStream_t st) {
  const size_t sm = DpShape<H>::SMEM;
  cudaError_t e = cudaFuncSetAttribute(k_dynamic_pool<H, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k_dynamic_pool<H, TAIL><<<grid, kDpThreads, sm, st>>>(m, w_t, pts, n, r, out_sdf, out_depth, hbuf);
  return cudaGetLastError();
}

template <int H, int TAIL>
static cudaError_t launch_qf_t(const MlpDev& m, const float* w_t, const float* pts, const uint32_t* perm,
                               const QueryMeta* meta, float* out, int num_sms, cudaStream_t st) {
  const size_t sm = DpShape<H>::SMEM;
  cudaError_t e = cudaFuncSetAttribute(k_query_fp32<H, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k_query_fp32<H, TAIL><<<num_sms, kDpThreads, sm, st>>>(m, w_t, pts, perm, meta, out);
  return cudaGetLastError();
}

bool query_fp32_supported(int H) { return H == 128 || H == 256 || H == 336; }

cudaError_t launch_query_fp32(const MlpDev& m, const float* w_t, const float* pts, const uint32_t* perm,
                              const QueryMeta* meta, float* out, int num_sms, cudaStream_t st) {
  const bool mult = m.tail == SAND_TAIL_MULT;
  switch (m.H) {
    case 128: return mult ? launch_qf_t<128, 1>(m, w_t, pts, perm, meta, out, num_sms, st)
                          : launch_qf_t<128, 0>(m, w_t, pts, perm, meta, out, num_sms, st);
    case 256: return mult ? launch_qf_t<256, 1>(m, w_t, pts, perm, meta, out, num_sms, st)
                          : launch_qf_t<256, 0>(m, w_t, pts, perm, meta, out, num_sms, st);
    case 336: return mult ? launch_qf_t<336, 1>(m, w_t, pts, perm, meta, out, num_sms, st)
                          : launch_qf_t<336, 0>(m, w_t, pts, perm, meta, out, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

size_t dynamic_scratch_floats(int H, int num_sms) {
  return (size_t)num_sms * kDynPool * (size_t)((H + 31) / 32 * 32);
}

cudaError_t launch_query_dynamic(const MlpDev& m, const float* w_t, const float* pts, long long n, float r,
                                 float* out_sdf, uint8_t* out_depth, float* hbuf, int num_sms, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (!hbuf)   // tile-level early exit (no scratch): MODE 1 of the population kernel
    return launch_dp(m, w_t, pts, n, r, 1, out_depth, out_sdf, 1, num_sms, st);
  const long long npool = (n + kDynPool - 1) / kDynPool;
  const int grid = (int)(npool < num_sms ? npool : num_sms);
  const bool mult = m.tail == SAND_TAIL_MULT;
#define SAND_DYN_CASE(HH)                                                                              \
  case HH:                                                                                             \
    return mult ? launch_pool_t<HH, 1>(m, w_t, pts, n, r, out_sdf, out_depth, hbuf, grid, st)          \
                : launch_pool_t<HH, 0>(m, w_t, pts, n, r, out_sdf, out_depth, hbuf, grid, st);
  switch (m.H) {
    SAND_DYN_CASE(16)
    SAND_DYN_CASE(32)
    SAND_DYN_CASE(64)
    SAND_DYN_CASE(128)
    SAND_DYN_CASE(256)
    SAND_DYN_CASE(336)
    default: return cudaErrorInvalidValue;
  }
#undef SAND_DYN_CASE
}

cudaError_t launch_leaf_max(const uint8_t* d, long long n_leaves, int spl, uint8_t* out, cudaStream_t st) {
  if (n_leaves <= 0) return cudaSuccess;
  k_leaf_max<<<(unsigned)((n_leaves + 255) / 256), 256, 0, st>>>(d, n_leaves, spl, out);
  return cudaGetLastError();
}

}  // namespace sand
