// tmlp_x3.cu -- FP32-accurate T-MLP on the tensor cores (SAND_F16X3), CTA pair (cta_group::2), H in {64, 128, 256}.
//
// The H x H layers of Eq. 2 in FP32 accuracy on tcgen05: every operand is split into two
// FP16 values, v = v_hi + v_lo (v_hi = fp16(v), v_lo = fp16(v - v_hi): 22 significant bits), and a layer is
// the three products
//     Z = A_hi W_hi^T + A_lo W_hi^T + A_hi W_lo^T        (the dropped A_lo W_lo^T is ~2^-22 relative)
// accumulated in FP32 in TMEM, after a K = 16 MMA that puts the split bias (1, 1) x (b_hi, b_lo) in the
// accumulator.  w0 is folded into W and b on the host.  Layer 1 (K = 3) is evaluated in FP32 SIMT in the
// epilogue.  The sine is a Cody-Waite reduction to [-pi, pi] (two FMAs) followed by MUFU.SIN (|err| ~ 5e-7).
// FP16 keeps the split operands at 2 bytes (TF32 operands would need 4), so A_hi + A_lo of a 256-row tile
// fit in shared memory like the BF16 kernel's two tile slots.  One tile is in flight per CTA pair.
//
// Three modes on the same machinery:
//   query (POP = 0; Sec. 3.4): binned 256-row tiles of uniform exit depth d, y_d -> sdf[perm[row]];
//   population (POP = 1; Eq. 5): 256 consecutive samples per tile, all L layers, every y_i kept, and
//     the required depth d(x) = min{ i : sign(y_i) = sign(y_L) [and |y_L - y_i| < r] } -> depth[sample];
//   dynamic exit (POP = 2; "SAND w/o Octree", R23): as population, every t_i kept, and
//     the exit layer d = min{ i >= 2 : |t_i| < r } (else L), y_d -> sdf, d -> depth (255 / NaN for
//     non-finite points).  All L layers are evaluated (no tile-level early stop), the selection is exact.
//
// Warp roles per CTA ("leader" = even CTA):
//   warp 0   producer (lane 0): this CTA's half of a hidden layer's operands through an NST-stage ring:
//            stage 0 = [split bias operand | K-chunk 0 of W_hi], then the other W_hi chunks, then W_lo chunks
//   warp 1   TMEM allocator; leader: the MMA issuer; odd CTA: relays "my half landed" (w_peer)
//   warp 2   IO: tile rows' points -> x buffer (double-buffered by tile), per-layer reduction of the tail
//            partials -> t_i, y_i, and the tile's outputs (sdf, or the Eq. 5 depth)
//   warps 3..18  16 epilogue warps = 4 TMEM lane quadrants x 4 column groups (tmlp_tc2.cu's 16x256b scheme)
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "sand_internal.h"

namespace sand {

template <int H>
struct X3Shape {
  static constexpr int KC = H / 64;                // 64-wide K chunks (128-byte swizzle atoms of fp16)
  static constexpr int A_CHUNK = 128 * 128;        // one K-chunk of this CTA's 128 rows (bytes)
  static constexpr int A_BYTES = KC * A_CHUNK;     // A_hi or A_lo
  static constexpr int WH_CHUNK = (H / 2) * 128;   // this CTA's half (H/2 rows) of one K-chunk
  static constexpr int SMALL = (H / 2) * 32 < 1024 ? 1024 : (H / 2) * 32;   // split-bias operand (padded)
  static constexpr int STAGE = SMALL + WH_CHUNK;   // ring slot: [bias operand (stage 0 of a layer only)][1 chunk]
  static constexpr int NSJ = 2 * KC;               // ring stages per hidden layer (W_hi chunks, then W_lo)
  static constexpr int ONES_BYTES = 128 * 32;      // bias MMA A operand: rows (1, 1, 0, ...) in fp16
  static constexpr int XB = 128 * 16;              // x of one tile: float4 per row
  static constexpr int CQ = H / 4;                 // columns per epilogue column group
  static constexpr int TMEM_COLS = H;              // one FP32 accumulator (64, 128 or 256: powers of two)
  static constexpr int THREADS = 96 + 512;
  static constexpr int TILE = 256;
  static_assert(H == 64 || H == 128 || H == 256, "split-FP16 kernel: H in {64, 128, 256}");
};

struct X3Params {
  MlpDev m;
  const float* pts;          // query: n x 3 (gathered through perm); population: the samples
  const uint32_t* perm;      // query only
  const QueryMeta* meta;     // query only
  float* out_sdf;            // query
  uint8_t* out_depth;        // population
  long long n;               // population: number of samples
  float r;                   // population: Eq. 5 threshold
  int near;                  // population: Eq. 5 branch (1: sign and |y_L - y_i| < r; 0: sign only)
  int nst;
};

// f16 pair from two floats (cvt.rn.f16x2.f32: round to nearest even), and back
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float2 unpack_f16x2(uint32_t v) {
  float a, b;
  asm("{\n.reg .f16 l, h;\nmov.b32 {l, h}, %2;\ncvt.f32.f16 %0, l;\ncvt.f32.f16 %1, h;\n}\n" : "=f"(a), "=f"(b) : "r"(v));
  return make_float2(a, b);
}

// sin z to ~5e-7 absolute: k = rint(z / 2 pi), r = z - k C1 - k C2 (C1 + C2 = 2 pi, C1 exact in 12 bits),
// then MUFU.SIN on |r| <= pi.
__device__ __forceinline__ float2 sin_precise2(float2 z) {
  const float2 t = __ffma2_rn(z, make_float2(0.15915494309189535f, 0.15915494309189535f),
                              make_float2(12582912.0f, 12582912.0f));
  const float2 k = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  float2 r = __ffma2_rn(k, make_float2(-6.28125f, -6.28125f), z);
  r = __ffma2_rn(k, make_float2(-1.9353071795864769e-3f, -1.9353071795864769e-3f), r);
  return make_float2(__sinf(r.x), __sinf(r.y));
}

__device__ __forceinline__ uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);   // D f32, A = B = f16
}

// Walk over this pair's tiles (tile i = pair + npairs * i), steps l = 1..d (population: d = L).
struct X3Walk {
  long long t;
  int d, l, ti;
  bool done;
};

template <int H, int TAIL, int POP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(X3Shape<H>::THREADS, 1)
    k_tmlp_x3(const X3Params p) {
  using C = X3Shape<H>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = smem_u32(smem_raw);
  if (base & 1023u) __trap();
  uint8_t* gbase = smem_raw;
  const int nst = p.nst;
  const int L = p.m.L;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // ---- shared memory (identical offsets in both CTAs)
  const uint32_t sAh = base;                                      // A_hi, SW128 K-major fp16
  const uint32_t sAl = sAh + C::A_BYTES;                          // A_lo
  const uint32_t sW = sAl + C::A_BYTES;                           // weight ring, nst x STAGE
  const uint32_t sOnes = sW + nst * C::STAGE;                     // bias-MMA A operand (constant)
  const uint32_t sX = sOnes + C::ONES_BYTES;                      // [2] x buffers (float4 per row)
  float* tab = reinterpret_cast<float*>(gbase + (sX + 2 * C::XB - base));
  const long long ntab = p.m.x3_floats;
  constexpr int NPL = TAIL == SAND_TAIL_MULT ? 8 : 4;             // partial planes per layer
  float* part = tab + ((ntab + 3) & ~3ll);                        // [2 parities][NPL][128]
  float* ybuf = part + 2 * NPL * 128;                             // population: [L][128] cumulative y_i
  const int ybuf_floats = POP == 2 ? 2 * L * 128 : POP ? L * 128 : 0;   // y_i (and t_i for POP = 2)
  const int nb = L + 2;
  long long* meta_s = reinterpret_cast<long long*>(ybuf + ybuf_floats);
  long long* s_tile_end = meta_s;
  long long* s_tile_begin = meta_s + nb;
  long long* s_start = meta_s + 2 * nb;
  long long* s_count = meta_s + 3 * nb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta_s + 4 * nb);
  const uint32_t b_wfull = smem_u32(bars);
  const uint32_t b_wempty = b_wfull + 8 * nst;
  const uint32_t b_wpeer = b_wempty + 8 * nst;
  const uint32_t b_afull = b_wpeer + 8 * nst;     // epilogue wrote the next A (both CTAs' 16 warps)
  const uint32_t b_accfull = b_afull + 8;         // MMA done (multicast commit)
  const uint32_t b_xfull = b_accfull + 8;         // [2] x of a tile written (IO warp)
  const uint32_t b_xfree = b_xfull + 16;          // [2] x read by the 16 epilogue warps (layer 1)
  const uint32_t b_pfull = b_xfree + 16;          // [2] partial planes of a layer written (16 warps)
  const uint32_t b_pfree = b_pfull + 16;          // [2] partial planes read (IO warp)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * nst + 10);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const float4* src = reinterpret_cast<const float4*>(p.m.x3_tables);
    float4* dst = reinterpret_cast<float4*>(tab);
    for (long long i = tid; i < (ntab + 3) / 4; i += blockDim.x) dst[i] = src[i];
    uint32_t* ones = reinterpret_cast<uint32_t*>(gbase + (sOnes - base));
    for (int i = tid; i < C::ONES_BYTES / 4; i += blockDim.x) ones[i] = 0u;
    if (!POP && tid < nb) {
      s_tile_end[tid] = p.meta->tile_end[tid];
      s_tile_begin[tid] = p.meta->tile_begin[tid];
      s_start[tid] = p.meta->start[tid];
      s_count[tid] = p.meta->count[tid];
    }
    __syncthreads();
    for (int r = tid; r < 128; r += blockDim.x) ones[l1_off((uint32_t)r, 0) / 4] = 0x3C003C00u;   // fp16 (1, 1)
    fence_proxy_async_smem();
  }
  if (tid == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(b_wfull + 8 * i, 1);
      mbar_init(b_wempty + 8 * i, 1);
      mbar_init(b_wpeer + 8 * i, 1);
    }
    mbar_init(b_afull, 32);
    mbar_init(b_accfull, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(b_xfull + 8 * i, 1);
      mbar_init(b_xfree + 8 * i, 16);
      mbar_init(b_pfull + 8 * i, 16);
      mbar_init(b_pfree + 8 * i, 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_cg2(smem_u32(tmem_slot), C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const long long T = POP ? (p.n + C::TILE - 1) / C::TILE : p.meta->total_tiles;

  auto tile_depth = [&](long long t) {
    if (POP) return L;
    for (int d = L; d >= 1; --d)
      if (t < s_tile_end[d]) return d;
    return 0;
  };
  auto wstart = [&](X3Walk& w) {
    w.ti = 0;
    w.t = pair;
    w.done = w.t >= T;
    w.l = 1;
    w.d = w.done ? 0 : tile_depth(w.t);
  };
  auto wadvance = [&](X3Walk& w) {
    if (w.l == w.d) {
      ++w.ti;
      w.t += npairs;
      w.done = w.t >= T;
      w.l = 1;
      w.d = w.done ? 0 : tile_depth(w.t);
    } else {
      ++w.l;
    }
  };

  if ((warp == 0 && lane == 0) || warp == 1) {
    // ======== producer (warp 0 lane 0) / MMA issuer (leader warp 1) / relay (odd warp 1): hidden layers only
    constexpr size_t LCTA = (size_t)C::SMALL + 2 * (size_t)C::KC * C::WH_CHUNK;   // one CTA's half of a layer
    const uint8_t* img = reinterpret_cast<const uint8_t*>(p.m.x3_image) + (size_t)rank * LCTA;
    const uint32_t peer_wpeer = mapa_shared(b_wpeer, 0);
    const uint32_t idesc = idesc_f16(256, H);
    uint32_t pa = 0;
    int st = 0;
    uint32_t ph = 0;
    X3Walk w;
    wstart(w);
#pragma unroll 1
    while (!w.done) {
      const int l = w.l;
      if (l >= 2) {
        const uint8_t* src = img + (size_t)(l - 2) * 2 * LCTA;
        if (warp == 0) {
#pragma unroll 1
          for (int j = 0; j < C::NSJ; ++j) {
            mbar_wait_lazy(b_wempty + 8 * st, ph ^ 1u);
            const uint32_t slot = sW + st * C::STAGE;
            // stage j: j == 0 -> [bias | W_hi chunk 0]; 0 < j < KC -> W_hi chunk j; KC <= j -> W_lo chunk j - KC
            const uint32_t bytes = j == 0 ? C::STAGE : C::WH_CHUNK;
            const size_t off = j == 0 ? 0 : (size_t)C::SMALL + (size_t)j * C::WH_CHUNK;
            mbar_arrive_expect_tx(b_wfull + 8 * st, bytes);
            bulk_g2s(j == 0 ? slot : slot + C::SMALL, src + off, bytes, b_wfull + 8 * st);
            if (++st == nst) { st = 0; ph ^= 1u; }
          }
        } else if (rank == 0) {
          mbar_wait_cluster(b_afull, pa);   // the epilogue wrote A (hi, lo) of layer l - 1 and read the accumulator
          pa ^= 1u;
          tc_fence_after();
#pragma unroll 1
          for (int j = 0; j < C::NSJ; ++j) {
            mbar_wait(b_wfull + 8 * st, ph);
            mbar_wait_cluster(b_wpeer + 8 * st, ph);
            tc_fence_after();
            const uint32_t slot = sW + st * C::STAGE;
            if (j == 0) mma_bf16_cg2_w(tmem_base, desc_nosw(sOnes, 128, 256), desc_nosw(slot, 128, 256), idesc, 0u);
            const uint64_t w_d = desc_sw128(slot + C::SMALL);
            const int kc = j < C::KC ? j : j - C::KC;
            const uint64_t ah = desc_sw128(sAh) + (uint64_t)(kc * (C::A_CHUNK >> 4));
            mma4_bf16_cg2_w(tmem_base, ah, w_d, idesc, 1u);                      // A_hi W_hi  or  A_hi W_lo
            if (j < C::KC)
              mma4_bf16_cg2_w(tmem_base, desc_sw128(sAl) + (uint64_t)(kc * (C::A_CHUNK >> 4)), w_d, idesc, 1u);   // A_lo W_hi
            mma_commit_cg2_mc_w(b_wempty + 8 * st, 0x3);
            if (++st == nst) { st = 0; ph ^= 1u; }
          }
          mma_commit_cg2_mc_w(b_accfull, 0x3);
        } else {
#pragma unroll 1
          for (int j = 0; j < C::NSJ; ++j) {
            mbar_wait(b_wfull + 8 * st, ph);
            if (lane == 0) mbar_arrive_remote(peer_wpeer + 8 * st);
            __syncwarp();
            if (++st == nst) { st = 0; ph ^= 1u; }
          }
        }
      }
      wadvance(w);
    }
  } else if (warp == 2) {
    // ======== IO warp: x of the tile rows, per-layer tail reduction, outputs
    const float* tc0 = tab + p.m.x3_off_c;     // [L] tail biases (MULT: c_i0)
    const float* tc1 = tab + p.m.x3_off_c1;    // [L] (MULT: c_i1 at index i-1)
    auto rows_of = [&](long long t, uint32_t (&ix)[4], int& d) {
      d = tile_depth(t);
      if (POP) {
        const long long r0 = t * C::TILE + (long long)rank * 128;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const long long r = r0 + lane + 32 * k;
          ix[k] = r < p.n ? (uint32_t)r : 0xFFFFFFFFu;
        }
      } else {
        const long long r0 = s_start[d] + (t - s_tile_begin[d]) * C::TILE + (long long)rank * 128;
        const long long rend = s_start[d] + s_count[d];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const long long r = r0 + lane + 32 * k;
          ix[k] = r < rend ? __ldg(p.perm + r) : 0xFFFFFFFFu;
        }
      }
    };
    auto fill = [&](int buf, const uint32_t (&ix)[4]) {
      float4* xb = reinterpret_cast<float4*>(gbase + (sX + buf * C::XB - base));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool v = ix[k] != 0xFFFFFFFFu;
        const size_t i = v ? ix[k] : 0;
        xb[lane + 32 * k] = v ? make_float4(__ldg(p.pts + 3 * i), __ldg(p.pts + 3 * i + 1), __ldg(p.pts + 3 * i + 2), 0.f)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(b_xfull + 8 * buf);
    };
    X3Walk w;
    wstart(w);
    uint32_t cur[4], nxt[4];
    int dcur = 0, dnxt = 0;
    if (!w.done) { rows_of(w.t, cur, dcur); fill(0, cur); }
    if (w.t + npairs < T) rows_of(w.t + npairs, nxt, dnxt);
    float y[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t par = 0, pfpar[2] = {0, 0};
#pragma unroll 1
    while (!w.done) {
      const int l = w.l;
      if (l == 1 && w.t + npairs < T) {
        // prefetch the next tile's x into the other buffer once its previous user (two tiles back) read it
        const int nb_ = (w.ti + 1) & 1;
        if (w.ti >= 1) mbar_wait_lazy(b_xfree + 8 * nb_, (uint32_t)(((w.ti - 1) >> 1) & 1));
        fill(nb_, nxt);
      }
      // this layer's tail partials
      mbar_wait_lazy(b_pfull + 8 * par, pfpar[par]);
      pfpar[par] ^= 1u;
      const float* pl = part + par * NPL * 128;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int rr = lane + 32 * k;
        float s0 = tc0[l - 1], s1 = 0.f;
#pragma unroll
        for (int g = 0; g < 4; ++g) s0 += pl[128 * g + rr];
        float t = s0;
        if (TAIL == SAND_TAIL_MULT && l >= 2) {
          s1 = tc1[l - 1];
#pragma unroll
          for (int g = 4; g < 8; ++g) s1 += pl[128 * g + rr];
          t = s0 * s1;
        }
        y[k] += t;
        if (POP) ybuf[(l - 1) * 128 + rr] = y[k];
        if (POP == 2) ybuf[(L + l - 1) * 128 + rr] = t;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(b_pfree + 8 * par);
      par ^= 1u;
      if (l == w.d) {
        if (POP == 2) {
          // R23: exit at the first layer i >= 2 whose residual |t_i| < r, else at L
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (cur[k] == 0xFFFFFFFFu) continue;
            const int rr = lane + 32 * k;
            const size_t gi = cur[k];
            const bool fin = isfinite(__ldg(p.pts + 3 * gi)) && isfinite(__ldg(p.pts + 3 * gi + 1)) &&
                             isfinite(__ldg(p.pts + 3 * gi + 2));
            int dd = L;
            for (int i = 2; i < L; ++i)
              if (fabsf(ybuf[(L + i - 1) * 128 + rr]) < p.r) { dd = i; break; }
            p.out_sdf[gi] = fin ? ybuf[(dd - 1) * 128 + rr] : __int_as_float(0x7fc00000);
            p.out_depth[gi] = fin ? (uint8_t)dd : (uint8_t)SAND_DEPTH_NONFINITE;
          }
        } else if (POP) {
          // Eq. 5: d(x) = min{ i : sign(y_i) = sign(y_L) [and |y_L - y_i| < r] }; i = L always qualifies
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (cur[k] == 0xFFFFFFFFu) continue;
            const int rr = lane + 32 * k;
            const float yL = y[k];
            int dd = L;
            for (int i = 1; i < L; ++i) {
              const float yi = ybuf[(i - 1) * 128 + rr];
              const bool same = (yi > 0.f) == (yL > 0.f) && (yi < 0.f) == (yL < 0.f);
              if (same && (!p.near || fabsf(yL - yi) < p.r)) { dd = i; break; }
            }
            p.out_depth[cur[k]] = (uint8_t)dd;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (cur[k] != 0xFFFFFFFFu) p.out_sdf[cur[k]] = y[k];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) { y[k] = 0.f; cur[k] = nxt[k]; }
        dcur = dnxt;
        if (w.t + 2ll * npairs < T) rows_of(w.t + 2ll * npairs, nxt, dnxt);
      }
      wadvance(w);
    }
    (void)dcur;
  } else if (warp >= 3) {
    // ======== epilogue (16 warps): thread (quad, tq) owns rows 32q + quad + 8k and columns 2tq, 2tq+1 of each
    // 8-column chunk of its group (the 16x256b TMEM shape)
    const int ew = warp - 3;
    const int q = warp & 3;
    const int cq = ew >> 2;
    const int quad = lane >> 2, tq = lane & 3;
    const int c0 = cq * C::CQ;
    constexpr int NCH = C::CQ / 8;
    constexpr int CB = NCH >= 2 ? 2 : 1;         // 8-column chunks per TMEM load batch
    const uint32_t tm_q = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
    const uint32_t a_off = (uint32_t)(4 * q + (lane >> 3)) * 1024 + (uint32_t)(lane & 7) * 128;
    const float4* tw1 = reinterpret_cast<const float4*>(tab + p.m.x3_off_w1);   // [H] (w0 W1 x y z, w0 b1)
    const float* tta = tab + p.m.x3_off_a;     // [L][H]
    const float* ta1 = tab + p.m.x3_off_a1;    // [L-1][H] (MULT)
    const uint32_t afull_dst = rank == 0 ? b_afull : mapa_shared(b_afull, 0);
    X3Walk w;
    wstart(w);
    uint32_t pacc = 0, par = 0, pfpar[2] = {1, 1};
    float4 xr[4];
#pragma unroll 1
    while (!w.done) {
      const int l = w.l, d = w.d;
      const bool store = l != d;
      float2 yv[4], yv1[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) { yv[k] = make_float2(0.f, 0.f); yv1[k] = make_float2(0.f, 0.f); }
      if (l == 1) {
        const int xb = w.ti & 1;
        mbar_wait(b_xfull + 8 * xb, (uint32_t)((w.ti >> 1) & 1));
        const float4* xs = reinterpret_cast<const float4*>(gbase + (sX + xb * C::XB - base));
#pragma unroll
        for (int k = 0; k < 4; ++k) xr[k] = xs[32 * q + quad + 8 * k];
        __syncwarp();
        if (lane == 0) mbar_arrive(b_xfree + 8 * xb);
      } else {
        mbar_wait(b_accfull, pacc);
        pacc ^= 1u;
        tc_fence_after();
      }
      const float* ta = tta + (l - 1) * H + c0 + 2 * tq;
      const float* a1p = ta1 + (l - 2) * H + c0 + 2 * tq;
      auto chunk = [&](const uint32_t* ra, const uint32_t* rb, const int jc) {
        const float2 a2 = *reinterpret_cast<const float2*>(ta + jc);
        float2 c2 = make_float2(0.f, 0.f);
        if (TAIL == SAND_TAIL_MULT && l >= 2) c2 = *reinterpret_cast<const float2*>(a1p + jc);
        float4 wa, wb;
        if (l == 1) { wa = tw1[c0 + jc + 2 * tq]; wb = tw1[c0 + jc + 2 * tq + 1]; }
        uint32_t phi[4], plo[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float2 z;
          if (l == 1) {
            // layer 1 in FP32: z = w0 (W1 x + b1), sequential over x, y, z
            const float4 x = xr[k];
            z = make_float2(wa.w, wb.w);
            z = __ffma2_rn(make_float2(wa.x, wb.x), make_float2(x.x, x.x), z);
            z = __ffma2_rn(make_float2(wa.y, wb.y), make_float2(x.y, x.y), z);
            z = __ffma2_rn(make_float2(wa.z, wb.z), make_float2(x.z, x.z), z);
          } else {
            const uint32_t* r = k < 2 ? ra : rb;
            const int o = 2 * (k & 1);
            z = make_float2(__uint_as_float(r[o]), __uint_as_float(r[o + 1]));
          }
          const float2 h = sin_precise2(z);
          yv[k] = __ffma2_rn(a2, h, yv[k]);
          if (TAIL == SAND_TAIL_MULT) yv1[k] = __ffma2_rn(c2, h, yv1[k]);
          phi[k] = pack_f16x2(h.x, h.y);
          const float2 hb = unpack_f16x2(phi[k]);
          plo[k] = pack_f16x2(h.x - hb.x, h.y - hb.y);
        }
        if (store) {
          const uint32_t u = (uint32_t)((c0 + jc) >> 3);
          const uint32_t o = (u >> 3) * C::A_CHUNK + (((u & 7u) ^ (uint32_t)(lane & 7)) << 4) + a_off;
          stmatrix_x4(sAh + o, phi);
          stmatrix_x4(sAl + o, plo);
        }
      };
#pragma unroll
      for (int bb = 0; bb < NCH / CB; ++bb) {
        uint32_t r0[4 * CB], r1[4 * CB];
        if (l >= 2) {
          tmem_ld_16x256b<CB>(tm_q + bb * 8 * CB, r0);
          tmem_ld_16x256b<CB>(tm_q + (16u << 16) + bb * 8 * CB, r1);
          tmem_wait_ld_dep(r0);
          tmem_wait_ld_dep(r1);
        }
#pragma unroll
        for (int i = 0; i < CB; ++i) chunk(r0 + 4 * i, r1 + 4 * i, bb * 8 * CB + 8 * i);
      }
      // publish the next layer's A (and that the accumulator has been read)
      if (store) {
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(afull_dst);
          else mbar_arrive_remote(afull_dst);
        }
      } else {
        tc_fence_before();
      }
      // tail partials of this layer: quad sums, one value per row per column group (plane)
      mbar_wait(b_pfree + 8 * par, pfpar[par]);
      pfpar[par] ^= 1u;
      float* pl = part + par * NPL * 128;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float v = yv[k].x + yv[k].y;
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (tq == 0) pl[cq * 128 + 32 * q + quad + 8 * k] = v;
        if (TAIL == SAND_TAIL_MULT) {
          float v1 = yv1[k].x + yv1[k].y;
          v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
          v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
          if (tq == 0) pl[(4 + cq) * 128 + 32 * q + quad + 8 * k] = v1;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(b_pfull + 8 * par);
      par ^= 1u;
      wadvance(w);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_cg2(tmem_base, C::TMEM_COLS);
}

// ------------------------------------------------------------------------------------ host side
static constexpr size_t kSmemMaxX3 = 232448;

template <int H>
static size_t smem_x3(long long tab_floats, int L, int tail, int pop, int nst) {
  using C = X3Shape<H>;
  const size_t npl = tail == SAND_TAIL_MULT ? 8 : 4;
  return 2 * (size_t)C::A_BYTES + (size_t)nst * C::STAGE + C::ONES_BYTES + 2 * (size_t)C::XB +
         (size_t)((tab_floats + 3) & ~3ll) * 4 + 2 * npl * 128 * 4 + (size_t)(pop == 2 ? 2 : pop ? 1 : 0) * L * 128 * 4 +
         4 * (size_t)(L + 2) * 8 + (3 * (size_t)nst + 10) * 8 + 16;
}

template <int H>
static int pick_nst_x3(long long tab_floats, int L, int tail, int pop) {
  int best = 0;
  for (int nst = 1; nst <= 8; ++nst)
    if (smem_x3<H>(tab_floats, L, tail, pop, nst) <= kSmemMaxX3) best = nst;
  return best;
}

bool x3_available(int H) { return H == 64 || H == 128 || H == 256; }

static void x3_layout(int L, int H, int tail, MlpDev* m) {
  auto al4 = [](long long v) { return (v + 3) & ~3ll; };
  m->x3_off_w1 = 0;                                   // float4 [H]
  m->x3_off_a = al4(4ll * H);                         // [L][H]
  m->x3_off_a1 = al4(m->x3_off_a + (long long)L * H);  // [L-1][H]
  m->x3_off_c = al4(m->x3_off_a1 + (tail == SAND_TAIL_MULT ? (long long)(L - 1) * H : 0));
  m->x3_off_c1 = al4(m->x3_off_c + L);
  m->x3_floats = al4(m->x3_off_c1 + L);
}

bool x3_usable(int L, int H, int tail, int pop) {
  if (!x3_available(H)) return false;
  MlpDev m{};
  x3_layout(L, H, tail, &m);
  switch (H) {
    case 64: return pick_nst_x3<64>(m.x3_floats, L, tail, pop) >= 2;
    case 128: return pick_nst_x3<128>(m.x3_floats, L, tail, pop) >= 2;
    case 256: return pick_nst_x3<256>(m.x3_floats, L, tail, pop) >= 2;
    default: return false;
  }
}

static inline uint16_t f16_rne(float f) {
  // IEEE binary16 round-to-nearest-even (normal and subnormal results; |f| < 65504 here)
  uint32_t u;
  std::memcpy(&u, &f, 4);
  const uint32_t sign = (u >> 16) & 0x8000u;
  const uint32_t absu = u & 0x7FFFFFFFu;
  if (absu >= 0x477FF000u) return (uint16_t)(sign | 0x7C00u);           // overflow -> inf (not reached)
  if (absu < 0x38800000u) {                                            // subnormal half: value = m * 2^-24
    float a;
    std::memcpy(&a, &absu, 4);
    const float m = a * 16777216.0f;                                   // exact (power of two)
    float r = std::nearbyint(m);                                       // current rounding mode: nearest-even
    return (uint16_t)(sign | (uint32_t)r);
  }
  const uint32_t e = ((absu >> 23) - 112u) << 10;
  uint32_t mant = absu & 0x7FFFFFu;
  uint32_t hv = e | (mant >> 13);
  const uint32_t rest = mant & 0x1FFFu;
  if (rest > 0x1000u || (rest == 0x1000u && (hv & 1u))) ++hv;
  return (uint16_t)(sign | hv);
}
static inline float f16_to_f32(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
  float v;
  if (e == 0) {
    v = (float)m * 5.9604644775390625e-8f;
  } else {
    const uint32_t u = ((e + 112u) << 23) | (m << 13);
    std::memcpy(&v, &u, 4);
  }
  uint32_t u;
  std::memcpy(&u, &v, 4);
  u |= sign;
  std::memcpy(&v, &u, 4);
  return v;
}
static inline void f16_split(float v, uint16_t* hi, uint16_t* lo) {
  *hi = f16_rne(v);
  *lo = f16_rne(v - f16_to_f32(*hi));
}

void x3_build_host(int L, int H, int tail, float w0, const float* const* W, const float* const* b,
                   const float* const* a, const float* const* a1, const float* c, const float* c1, MlpDev* m,
                   std::vector<float>* tables, std::vector<uint8_t>* img) {
  x3_layout(L, H, tail, m);
  std::vector<float>& t = *tables;
  t.assign((size_t)m->x3_floats, 0.f);
  for (int j = 0; j < H; ++j) {
    t[m->x3_off_w1 + 4 * j + 0] = w0 * W[0][3 * j + 0];
    t[m->x3_off_w1 + 4 * j + 1] = w0 * W[0][3 * j + 1];
    t[m->x3_off_w1 + 4 * j + 2] = w0 * W[0][3 * j + 2];
    t[m->x3_off_w1 + 4 * j + 3] = w0 * b[0][j];
  }
  for (int i = 0; i < L; ++i) {
    std::memcpy(&t[m->x3_off_a + (size_t)i * H], a[i], sizeof(float) * H);
    t[m->x3_off_c + i] = c[i];
    t[m->x3_off_c1 + i] = c1[i];
  }
  if (tail == SAND_TAIL_MULT)
    for (int i = 1; i < L; ++i) std::memcpy(&t[m->x3_off_a1 + (size_t)(i - 1) * H], a1[i], sizeof(float) * H);
  // per (layer, CTA r): [split bias: H/2 rows x 16 fp16, (b_hi, b_lo) at k = 0, 1, l1_off layout, padded]
  //                     [KC chunks of W_hi: H/2 rows x 128 B, SW128 K-major][KC chunks of W_lo]
  // CTA r holds output rows r H/2 + [0, H/2) (cta_group::2 splits an instruction's N rows in halves).
  const int KC = H / 64, Hh = H / 2;
  const size_t small = Hh * 32 < 1024 ? 1024 : (size_t)Hh * 32, chunk = (size_t)Hh * 128;
  const size_t lcta = small + 2 * KC * chunk;
  img->assign(L >= 2 ? (size_t)(L - 1) * 2 * lcta : 0, 0);
  for (int i = 1; i < L; ++i)
    for (int n = 0; n < H; ++n) {
      const int r = n / Hh, row = n % Hh;
      uint8_t* bp = img->data() + ((size_t)(i - 1) * 2 + r) * lcta;
      uint16_t hi, lo;
      f16_split(w0 * b[i][n], &hi, &lo);
      std::memcpy(bp + l1_off((uint32_t)row, 0), &hi, 2);
      std::memcpy(bp + l1_off((uint32_t)row, 1), &lo, 2);
      for (int k = 0; k < H; ++k) {
        const int kc = k / 64, kk = k % 64;
        const size_t within = (size_t)(row / 8) * 1024 + (row % 8) * 128 + (size_t)(((kk / 8) ^ (row % 8)) * 16) + (kk % 8) * 2;
        f16_split(w0 * W[i][(size_t)n * H + k], &hi, &lo);
        std::memcpy(bp + small + kc * chunk + within, &hi, 2);
        std::memcpy(bp + small + (KC + kc) * chunk + within, &lo, 2);
      }
    }
}

template <int H, int TAIL, int POP>
static cudaError_t launch_x3_t(const X3Params& p0, int num_sms, cudaStream_t st) {
  X3Params p = p0;
  p.nst = pick_nst_x3<H>(p.m.x3_floats, p.m.L, TAIL, POP);
  if (p.nst < 2) return cudaErrorInvalidConfiguration;
  const size_t sm = smem_x3<H>(p.m.x3_floats, p.m.L, TAIL, POP, p.nst);
  static bool attr = false;   // per instantiation
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(k_tmlp_x3<H, TAIL, POP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)kSmemMaxX3);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_tmlp_x3<H, TAIL, POP><<<num_sms & ~1, X3Shape<H>::THREADS, sm, st>>>(p);
  return cudaGetLastError();
}

template <int POP>
static cudaError_t launch_x3_any(const X3Params& p, int num_sms, cudaStream_t st) {
  const bool mult = p.m.tail == SAND_TAIL_MULT;
  switch (p.m.H) {
    case 64: return mult ? launch_x3_t<64, 1, POP>(p, num_sms, st) : launch_x3_t<64, 0, POP>(p, num_sms, st);
    case 128: return mult ? launch_x3_t<128, 1, POP>(p, num_sms, st) : launch_x3_t<128, 0, POP>(p, num_sms, st);
    case 256: return mult ? launch_x3_t<256, 1, POP>(p, num_sms, st) : launch_x3_t<256, 0, POP>(p, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_tmlp_x3(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta, float* out,
                           int num_sms, cudaStream_t st) {
  X3Params p{};
  p.m = m; p.pts = pts; p.perm = perm; p.meta = meta; p.out_sdf = out;
  return launch_x3_any<0>(p, num_sms, st);
}

cudaError_t launch_required_depth_x3(const MlpDev& m, const float* pts, long long n, float r, int near, uint8_t* out,
                                     int num_sms, cudaStream_t st) {
  X3Params p{};
  p.m = m; p.pts = pts; p.n = n; p.r = r; p.near = near; p.out_depth = out;
  return launch_x3_any<1>(p, num_sms, st);
}

cudaError_t launch_query_dynamic_x3(const MlpDev& m, const float* pts, long long n, float r, float* out_sdf,
                                    uint8_t* out_depth, int num_sms, cudaStream_t st) {
  X3Params p{};
  p.m = m; p.pts = pts; p.n = n; p.r = r; p.out_sdf = out_sdf; p.out_depth = out_depth;
  return launch_x3_any<2>(p, num_sms, st);
}

}  // namespace sand
