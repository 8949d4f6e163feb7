// tmlp_tc4.cu -- CTA-pair (cta_group::2) persistent fused T-MLP kernel with one epilogue team per tile slot
// (SAND_BF16, H in {64, 128, 256}).
//
// Computes, per binned 256-row tile of uniform exit depth d (Sec. 3.4), exactly what
// tmlp_tc2.cu computes (same operands, same BF16 roundings, R20 / R26):
//   layer 1   : Z_1 = w0 (x W_1^T + b_1), one K = 16 split-BF16 MMA (x_hi W_hi + x_hi W_lo + x_lo W_hi + b)
//   layer 2..d: Z_l = [1 1 0..][w0 b_hi, w0 b_lo, 0..]^T + H_{l-1} bf16(w0 W_l)^T   (FP32 in TMEM)
//   every l   : h_l = sin(Z_l) (Eq. 2), tail t_l (Eq. 2 linear / Eq. 3 product), bf16(h_l) -> next A operand
//   output    : sdf[perm[row]] = y_d = sum_{l <= d} t_l
//
// What differs from tmlp_tc2.cu:
//   * Each layer is ONE N = H MMA chain per slot (no N-half passes): the A operand is read from shared memory
//     once per layer instead of twice.
//   * Two epilogue TEAMS, one per tile slot (warps 4-7 serve slot 0, warps 8-11 slot 1), each thread owning one
//     row (TMEM lane) and all H columns: the tail dot products are per-thread register sums (no shuffles, no
//     cross-warp Eq. 3 reduction), h goes to the SW128 A operand as 16-byte row segments, and the teams run
//     out of phase, so one team's waits (accumulator, publish, tile end) are covered by the other team's sines.
//   * The accumulator is read after the layer's whole MMA chain completed, so h is written in place (no pass-0
//     values held in registers).
//   * Weights stream as one bias operand + KC K-chunk stages per layer; when slot 1 runs the same hidden layer
//     right after slot 0 (the common case: both slots walk tiles of the same depth in lock step) it reuses
//     slot 0's stages, halving the L2 weight traffic.
//
// Warp roles (per CTA of the pair; "leader" = even CTA):
//   warp 0   weight producer (lane 0): bias operand + K-chunks of this CTA's N/2 B rows, bulk async copies
//   warp 1   TMEM allocator; leader: tcgen05.mma.cta_group::2 issuer (converged warp, elected lane);
//            odd CTA: relays "my half landed" to the leader (w_peer / b_peer)
//   warps 2, 3  IO of slot 0 / slot 1: perm rows, point gathers, the split-BF16 layer-1 operand, sdf[perm[row]]
//            stores
//   warps 4.. epilogue teams: team s = warps 4 + 4 NCG s .. ; thread = row 32 (warp % 4) + lane
// The producer, MMA issuer and relay walk one job order (slot 0, slot 1 alternating; a slot's jobs are its tiles'
// layers); each IO warp and each team walks its own slot's jobs.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include <type_traits>

#include "ptx.cuh"
#include "sand_internal.h"

#ifndef SAND_T4_NCG
#define SAND_T4_NCG 1     // column groups per team (1: a thread owns all H columns of its row)
#endif
#ifndef SAND_T4_PP
#define SAND_T4_PP 1      // LINEAR tails: all epilogue warps serve both slots step by step (ping-pong)
#endif
#ifndef SAND_T4_SHARE
#define SAND_T4_SHARE 1   // slot 1 reuses slot 0's weight stages when it runs the same layer right after it
#endif
#ifndef SAND_T4_PROF
#define SAND_T4_PROF 0    // 1: per-role clock64 wait / busy counters, dumped to stderr after every launch (synchronous)
#endif
#ifndef SAND_T4_TRACE
#define SAND_T4_TRACE 0   // 1: per-job clock64 timeline of CTA 0 (MMA issuer + epilogue warp 4), dumped by the host
#endif
#ifndef SAND_T4_ABL
#define SAND_T4_ABL 0     // ablation bitmask, timing only (wrong results): 1 no sine, 2 no A stores, 4 no TMEM loads, 8 no tail,
                          // 16 no tail-vector loads
#endif

namespace sand {

template <int H, bool PP>
struct Tc4Shape {
  static constexpr int KC = H / 64;                 // 64-wide K-chunks (128-byte swizzle atoms)
  static constexpr int NR = H / 2;                  // B rows (output features) per CTA (cta_group::2: half each)
  static constexpr int CHUNK = NR * 128;            // one K-chunk of this CTA's B rows (SW128)
  static constexpr int A_CHUNK = 128 * 128;         // one K-chunk of this CTA's 128 A rows
  static constexpr int A_BYTES = KC * A_CHUNK;
  static constexpr int BIAS_BYTES = NR * 32;        // K = 16 bias operand (l1_off layout, (b_hi, b_lo) at k = 9, 10)
  static constexpr int LAYER_BYTES = BIAS_BYTES + KC * CHUNK;   // one (layer, CTA) run of the image
  static constexpr int A1_BYTES = 128 * 32;
  static constexpr int W1_BYTES = NR * 32;
  // PP (ping-pong): all 16 epilogue warps serve both slots step by step (4 column groups); else two teams of
  // 4 NCG warps, one per slot
  static constexpr int NCG = PP ? 4 : SAND_T4_NCG;
  static constexpr int CW = H / NCG;                // columns per epilogue thread
  static constexpr int NB = CW / 32;                // 32-column TMEM load batches per thread
  static constexpr int TMEM_COLS = 2 * H <= 128 ? 128 : (2 * H <= 256 ? 256 : 512);
  static constexpr int NCTL = 4;
  static constexpr int TEAM_WARPS = 4 * NCG;        // epilogue warps serving one slot
  static constexpr int EPI_WARPS = PP ? TEAM_WARPS : 2 * TEAM_WARPS;
  static constexpr int THREADS = 32 * (NCTL + EPI_WARPS);
  static_assert(H % 64 == 0 && H <= 256, "team kernel: H in {64, 128, 192, 256}");
  static_assert(CW % 32 == 0, "whole 32-column batches per thread");
};

struct Tc4Params {
  MlpDev m;
  const float* pts;
  const uint32_t* perm;
  const QueryMeta* meta;
  float* out;
  int nst;
};

// Diagnostic counters (SAND_T4_PROF builds), per CTA: 0-3 team 0 wait_acc / busy / tile_end / steps, 4-7 team 1,
// 8 MMA wait a_full, 9 MMA wait a1_full, 10 MMA wait weights, 11 MMA loop, 12 producer wait empty,
// 13 IO0 wait a1_free, 14 IO0 wait io_done, 15 team 0 loop
constexpr int kT4Prof = 16;
__device__ unsigned long long g_t4prof[160][kT4Prof];
#define T4CLK() (SAND_T4_PROF ? clock64() : 0ll)
// Trace (SAND_T4_TRACE builds), CTA 0 only, per job j in MMA order: 0 MMA wait start, 1 a_full passed, 2 weights
// passed, 3 issue done (acc commit), 4 epilogue wait start, 5 accumulator ready, 6 published, 7 step end
constexpr int kT4Trace = 8192;
__device__ long long g_t4trace[kT4Trace][8];
// IO trace (slot 0 IO warp of CTA 0), per tile: 0 a1free wait start, 1 a1free ok, 2 fill+gather+perm done,
// 3 iodone wait start, 4 iodone ok, 5 partfree arrived, 6 end; team tile end: 7 partfree ok (epilogue warp 4)
__device__ long long g_t4iotr[kT4Trace][8];
#define T4IO(j, f) do { if (SAND_T4_TRACE && blockIdx.x == 0 && (j) < kT4Trace) g_t4iotr[(j)][(f)] = clock64(); } while (0)
#define T4TR(j, f) do { if (SAND_T4_TRACE && blockIdx.x == 0 && (j) < kT4Trace) g_t4trace[(j)][(f)] = clock64(); } while (0)

__device__ __forceinline__ int tile_depth4(long long t, const long long* te, int L) {
  for (int d = L; d >= 1; --d)
    if (t < te[d]) return d;
  return 0;
}

// Per-slot walk over this pair's tiles: tile i of slot s is 2 (pair + npairs i) + s -- the pair takes tile pairs
// (2u, 2u + 1), one tile per slot, and the scan pads every depth bin to an even tile count (launch_scan even_bins),
// so both slots always run tiles of the same depth in step and the same layer back to back (weight sharing);
// each tile yields jobs l = 1..d.
struct Walk4 {
  long long t;
  int d, l, ti;
  bool done;
  __device__ __forceinline__ void set(long long t_, long long T, const long long* te, int L) {
    t = t_;
    done = t >= T;
    l = 1;
    // tiles are ordered deepest depth first and a walk only moves forward: step the depth down from the last one
    if (!done)
      while (d > 1 && t >= te[d]) --d;
  }
  __device__ __forceinline__ void start(long long t0, long long T, const long long* te, int L) {
    ti = 0;
    d = L;
    set(t0, T, te, L);
  }
  __device__ __forceinline__ void advance(long long stride, long long T, const long long* te, int L) {
    if (l == d) { ++ti; set(t + stride, T, te, L); }
    else ++l;
  }
};

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
// bf16x2 pack without F2FP: F2FP.BF16.F32.PACK_AB issues to the same pipe as MUFU.SIN on sm_100a
// (scripts/micro/epi4.cu: sine + F2FP pack + store 10.4 clk per element-warp per SMSP, integer pack 9.0, MUFU
// floor 8).  Round to nearest, ties away from zero on the magnitude: bits + 0x8000, then the high halves of two
// words by one PRMT (IADD + PRMT on the ALU pipe).  h = sin(.) is finite, |h| <= 1, so no carry reaches the sign.
__device__ __forceinline__ uint32_t pack_bf16x2_int(float lo, float hi) {
  return __byte_perm(__float_as_uint(lo) + 0x8000u, __float_as_uint(hi) + 0x8000u, 0x7632);
}
#ifndef SAND_T4_NPOLY
#define SAND_T4_NPOLY 3   // sine pairs per 16 (per 32-column batch) evaluated by the FMA-pipe polynomial instead of MUFU
#endif
#ifndef SAND_T4_NPOLY_LAST
#define SAND_T4_NPOLY_LAST SAND_T4_NPOLY   // the share in a tile's last-layer steps (no A stores); 0-7 measured, 3 best
#endif
#ifndef SAND_T4_F2FP
#define SAND_T4_F2FP 1    // 1: pack with cvt.rn.bf16x2.f32 (F2FP); 0: integer pack
#endif
__device__ __forceinline__ uint32_t pack_h(float lo, float hi) {
  return SAND_T4_F2FP ? pack_bf16x2(lo, hi) : pack_bf16x2_int(lo, hi);
}
#ifndef SAND_T4_IPACK
#define SAND_T4_IPACK 0   // pairs (of the 4 in each 16-byte store) packed on the ALU instead of F2FP (1, 2 measured slower)
#endif
template <int J>
__device__ __forceinline__ uint32_t pack_k(float lo, float hi) {
  return J < SAND_T4_IPACK ? pack_bf16x2_int(lo, hi) : pack_h(lo, hi);
}
// Odd polynomial sine on the FMA pipe for two lanes at a time (shares the sine work with MUFU.SIN, which is the
// epilogue's binding pipe): k = rint(z / 2 pi) by the 1.5 2^23 magic add fused into the scaling FMA, r = z - 2 pi k
// in [-pi, pi], sin r = r P(r^2), odd minimax fit on [-pi, pi]: degree 9 (|err| < 6.2e-6, comparable to MUFU.SIN;
// degree 7 at 2.6e-4 compounds past the BF16 tolerance over 32 layers, tests/test_gpu_parity.py deep nets).
#ifndef SAND_T4_PDEG
#define SAND_T4_PDEG 9
#endif
__device__ __forceinline__ float2 sin_poly2(float2 z) {
#if SAND_T4_ABL & 1
  return z;
#else
  const float2 t = __ffma2_rn(z, make_float2(0.15915494309189535f, 0.15915494309189535f),
                              make_float2(12582912.0f, 12582912.0f));
  const float2 k = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 r = __ffma2_rn(k, make_float2(-6.283185307179586f, -6.283185307179586f), z);
  const float2 r2 = __fmul2_rn(r, r);
#if SAND_T4_PDEG == 9
  float2 q = __ffma2_rn(r2, make_float2(2.1478720100276405e-06f, 2.1478720100276405e-06f),
                        make_float2(-0.00019264993898104876f, -0.00019264993898104876f));
  q = __ffma2_rn(q, r2, make_float2(0.008308985270559788f, 0.008308985270559788f));
  q = __ffma2_rn(q, r2, make_float2(-0.16662438213825226f, -0.16662438213825226f));
  q = __ffma2_rn(q, r2, make_float2(0.9999793767929077f, 0.9999793767929077f));
#else
  float2 q = __ffma2_rn(r2, make_float2(-0.0001450767886126414f, -0.0001450767886126414f),
                        make_float2(0.007958059199154377f, 0.007958059199154377f));
  q = __ffma2_rn(q, r2, make_float2(-0.16566696763038635f, -0.16566696763038635f));
  q = __ffma2_rn(q, r2, make_float2(0.9992758631706238f, 0.9992758631706238f));
#endif
  return __fmul2_rn(q, r);
#endif
}
__device__ __forceinline__ float sin_mufu(float z) {
#if SAND_T4_ABL & 1
  return z;
#else
  return __sinf(z);
#endif
}

// ping-pong for LINEAR tails at H >= 128 (4 column groups of >= 32 columns); teams otherwise (Eq. 3 products need a
// row's two full dot products in one thread)
template <int H, int TAIL>
constexpr bool tc4_pp() { return SAND_T4_PP && TAIL == SAND_TAIL_LINEAR && H >= 128; }

template <int H, int TAIL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Tc4Shape<H, tc4_pp<H, TAIL>()>::THREADS, 1)
    k_tmlp_tc4(const Tc4Params p) {
  constexpr bool PP = tc4_pp<H, TAIL>();
  using C = Tc4Shape<H, PP>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = smem_u32(smem_raw);
  if (base & 1023u) __trap();
  const int nst = p.nst;
  const int L = p.m.L;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // ---- shared memory (identical offsets in both CTAs: the pair MMA relies on it)
  const uint32_t sA = base;                                  // [slot] KC x 16 KB, SW128 K-major
  const uint32_t sW = sA + 2 * C::A_BYTES;                   // chunk ring, nst x CHUNK
  const uint32_t sB = sW + nst * C::CHUNK;                   // bias ring, 2 x BIAS_BYTES
  // The bias MMA's A operand is the slot's layer-1 operand A1: its k = 9, 10 are 1 in every row and the bias
  // operand is zero outside k = 9, 10, so the product is b_hi + b_lo whichever tile's rows the IO warp is
  // writing into A1's other columns meanwhile (all finite).
  const uint32_t sW1 = sB + 2 * C::BIAS_BYTES;               // resident layer-1 B operand
  const uint32_t sA1 = sW1 + C::W1_BYTES;                    // [slot] layer-1 A operand
  const uint32_t sTab = sA1 + 2 * C::A1_BYTES;
  const long long ntab = (p.m.pt_floats + 3) & ~3ll;
  float* tab = reinterpret_cast<float*>(smem_raw + (sTab - base));
  float* part = tab + ntab;                                  // [slot][NCG][128] tile-end row sums
  const int nb = L + 2;
  long long* meta_s = reinterpret_cast<long long*>(part + 2 * C::NCG * 128);
  long long* s_tile_end = meta_s;
  long long* s_tile_begin = meta_s + nb;
  long long* s_start = meta_s + 2 * nb;
  long long* s_count = meta_s + 3 * nb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta_s + 4 * nb);
  const uint32_t b_wfull = smem_u32(bars);
  const uint32_t b_wempty = b_wfull + 8 * nst;
  const uint32_t b_wpeer = b_wempty + 8 * nst;
  const uint32_t b_bfull = b_wpeer + 8 * nst;     // [2] bias ring
  const uint32_t b_bempty = b_bfull + 16;
  const uint32_t b_bpeer = b_bempty + 16;
  const uint32_t b_afull = b_bpeer + 16;          // [slot] team step done (A written, accumulator read)
  const uint32_t b_accfull = b_afull + 16;        // [slot] the layer's MMA chain completed
  const uint32_t b_a1full = b_accfull + 16;       // [slot] layer-1 A written (leader: 2 arrivals)
  const uint32_t b_a1free = b_a1full + 16;        // [slot] layer-1 MMA done with A1
  const uint32_t b_iodone = b_a1free + 16;        // [slot] team wrote the tile's row sums
  const uint32_t b_partfree = b_iodone + 16;      // [slot] IO warp read them
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * nst + 6 + 12);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const float4* src = reinterpret_cast<const float4*>(p.m.pair_tables);
    float4* dst = reinterpret_cast<float4*>(tab);
    for (long long i = tid; i < ntab / 4; i += blockDim.x) dst[i] = src[i];
    const uint4* w1s = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(p.m.tc4_w1) + rank * C::W1_BYTES);
    uint4* w1d = reinterpret_cast<uint4*>(smem_raw + (sW1 - base));
    for (int i = tid; i < C::W1_BYTES / 16; i += blockDim.x) w1d[i] = w1s[i];
    if (tid < nb) {
      s_tile_end[tid] = p.meta->tile_end[tid];
      s_tile_begin[tid] = p.meta->tile_begin[tid];
      s_start[tid] = p.meta->start[tid];
      s_count[tid] = p.meta->count[tid];
    }
    fence_proxy_async_smem();   // W1 (generic stores) -> tensor core (async proxy)
  }
  if (tid == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(b_wfull + 8 * i, 1);
      mbar_init(b_wempty + 8 * i, 1);
      mbar_init(b_wpeer + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(b_bfull + 8 * i, 1);
      mbar_init(b_bempty + 8 * i, 1);
      mbar_init(b_bpeer + 8 * i, 1);
      mbar_init(b_afull + 8 * i, 2 * C::TEAM_WARPS);
      mbar_init(b_accfull + 8 * i, 1);
      mbar_init(b_a1full + 8 * i, 2);
      mbar_init(b_a1free + 8 * i, 1);
      mbar_init(b_iodone + 8 * i, C::TEAM_WARPS);
      mbar_init(b_partfree + 8 * i, 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_cg2(smem_u32(tmem_slot), C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const long long T = p.meta->total_tiles;
  const long long tstride = 2ll * npairs;
  const bool can_share = SAND_T4_SHARE && nst >= C::KC;

  if ((warp == 0 && lane == 0) || warp == 1) {
    // ================= warp 0 lane 0: weight producer; warp 1: MMA issuer (leader) / relay (odd CTA)
    // Weight sharing: a hidden-layer job of slot 1 that directly follows slot 0's job on the same layer is a
    // "sharer": it loads nothing and runs on the previous ("owner") job's bias + chunk stages, and it is the one
    // that releases them (its commits fire after both jobs' MMAs).  Every role derives the same decision.
    Walk4 w0, w1;
    w0.start(2ll * pair, T, s_tile_end, L);
    w1.start(2ll * pair + 1, T, s_tile_end, L);
    const uint8_t* img = reinterpret_cast<const uint8_t*>(p.m.tc4_image) + (size_t)rank * C::LAYER_BYTES;
    const uint32_t peer_wpeer = mapa_shared(b_wpeer, 0);
    const uint32_t peer_bpeer = mapa_shared(b_bpeer, 0);
    constexpr uint32_t ID = idesc_bf16(256, H);
    uint32_t pa[2] = {0, 0};
    int st = 0, bst = 0;          // next free chunk / bias stage (owner jobs)
    uint32_t ph = 0, bph = 0;
    int own_st = 0, own_bst = 0;  // stages of the last owner job (sharers reuse them)
    unsigned long long pc[5] = {0, 0, 0, 0, 0};   // SAND_T4_PROF: wait a_full, a1_full, weights, loop, empty
    const long long tl0 = T4CLK();
    int jc = 0;   // job counter (trace)
    auto job = [&](const Walk4& w, int s, bool share, bool next_shares) {
      const int l = w.l;
      const bool tr = SAND_T4_TRACE && warp == 1 && rank == 0 && lane == 0;
      if (tr) T4TR(jc, 0);
      if (l == 1) {
        if (warp == 1 && rank == 0) {
          long long c0 = T4CLK();
          if (w.ti != 0) { mbar_wait_cluster(b_afull + 8 * s, pa[s]); pa[s] ^= 1u; }
          long long c1 = T4CLK();
          if (tr) T4TR(jc, 1);
          mbar_wait_cluster(b_a1full + 8 * s, (uint32_t)(w.ti & 1));
          if (tr) T4TR(jc, 2);
          if (SAND_T4_PROF) { pc[0] += c1 - c0; pc[1] += T4CLK() - c1; }
          tc_fence_after();
          const uint32_t acc = tmem_base + (uint32_t)(s * H);
          mma_bf16_cg2_w(acc, desc_nosw(sA1 + s * C::A1_BYTES, 128, 256), desc_nosw(sW1, 128, 256), ID, 0u);
          mma_commit_cg2_mc_w(b_a1free + 8 * s, 0x3);
          mma_commit_cg2_mc_w(b_accfull + 8 * s, 0x3);
          if (tr) T4TR(jc, 3);
        }
        ++jc;
        return;
      }
      if (warp == 0) {
        if (share) return;
        const uint8_t* lb = img + (size_t)(l - 2) * 2 * C::LAYER_BYTES;
        long long c0 = T4CLK();
        mbar_wait(b_bempty + 8 * bst, bph ^ 1u);
        if (SAND_T4_PROF) pc[4] += T4CLK() - c0;
        mbar_arrive_expect_tx(b_bfull + 8 * bst, C::BIAS_BYTES);
        bulk_g2s(sB + bst * C::BIAS_BYTES, lb, C::BIAS_BYTES, b_bfull + 8 * bst);
        if (++bst == 2) { bst = 0; bph ^= 1u; }
        for (int kc = 0; kc < C::KC; ++kc) {
          c0 = T4CLK();
          mbar_wait(b_wempty + 8 * st, ph ^ 1u);
          if (SAND_T4_PROF) pc[4] += T4CLK() - c0;
          mbar_arrive_expect_tx(b_wfull + 8 * st, C::CHUNK);
          bulk_g2s(sW + st * C::CHUNK, lb + C::BIAS_BYTES + (size_t)kc * C::CHUNK, C::CHUNK, b_wfull + 8 * st);
          if (++st == nst) { st = 0; ph ^= 1u; }
        }
      } else if (rank == 0) {
        long long c0 = T4CLK();
        mbar_wait_cluster(b_afull + 8 * s, pa[s]);   // the slot's previous step (l - 1) is done
        pa[s] ^= 1u;
        if (SAND_T4_PROF) pc[0] += T4CLK() - c0;
        if (tr) T4TR(jc, 1);
        const uint32_t acc = tmem_base + (uint32_t)(s * H);
        const uint64_t a_d = desc_sw128(sA + s * C::A_BYTES);
        if (!share) {
          own_bst = bst;
          own_st = st;
          c0 = T4CLK();
          mbar_wait(b_bfull + 8 * bst, bph);
          mbar_wait_cluster(b_bpeer + 8 * bst, bph);
          if (SAND_T4_PROF) pc[2] += T4CLK() - c0;
          if (tr) T4TR(jc, 2);
          tc_fence_after();
          mma_bf16_cg2_w(acc, desc_nosw(sA1 + s * C::A1_BYTES, 128, 256), desc_nosw(sB + bst * C::BIAS_BYTES, 128, 256), ID, 0u);
#pragma unroll 1
          for (int kc = 0; kc < C::KC; ++kc) {
            c0 = T4CLK();
            mbar_wait(b_wfull + 8 * st, ph);
            mbar_wait_cluster(b_wpeer + 8 * st, ph);
            if (SAND_T4_PROF) pc[2] += T4CLK() - c0;
            tc_fence_after();
            mma4_bf16_cg2_w(acc, a_d + (uint64_t)(kc * (C::A_CHUNK >> 4)), desc_sw128(sW + st * C::CHUNK), ID, 1u);
            if (!next_shares) mma_commit_cg2_mc_w(b_wempty + 8 * st, 0x3);
            if (++st == nst) { st = 0; ph ^= 1u; }
          }
          if (!next_shares) mma_commit_cg2_mc_w(b_bempty + 8 * bst, 0x3);
          if (++bst == 2) { bst = 0; bph ^= 1u; }
        } else {
          if (tr) T4TR(jc, 2);
          tc_fence_after();
          mma_bf16_cg2_w(acc, desc_nosw(sA1 + s * C::A1_BYTES, 128, 256), desc_nosw(sB + own_bst * C::BIAS_BYTES, 128, 256),
                         ID, 0u);
          int cs = own_st;
#pragma unroll 1
          for (int kc = 0; kc < C::KC; ++kc) {
            mma4_bf16_cg2_w(acc, a_d + (uint64_t)(kc * (C::A_CHUNK >> 4)), desc_sw128(sW + cs * C::CHUNK), ID, 1u);
            mma_commit_cg2_mc_w(b_wempty + 8 * cs, 0x3);
            if (++cs == nst) cs = 0;
          }
          mma_commit_cg2_mc_w(b_bempty + 8 * own_bst, 0x3);
        }
        mma_commit_cg2_mc_w(b_accfull + 8 * s, 0x3);
        if (tr) T4TR(jc, 3);
      } else {
        if (share) { ++jc; return; }
        mbar_wait(b_bfull + 8 * bst, bph);
        if (lane == 0) mbar_arrive_remote(peer_bpeer + 8 * bst);
        __syncwarp();
        if (++bst == 2) { bst = 0; bph ^= 1u; }
        for (int kc = 0; kc < C::KC; ++kc) {
          mbar_wait(b_wfull + 8 * st, ph);
          if (lane == 0) mbar_arrive_remote(peer_wpeer + 8 * st);
          __syncwarp();
          if (++st == nst) { st = 0; ph ^= 1u; }
        }
      }
      ++jc;
    };
#pragma unroll 1
    while (!(w0.done && w1.done)) {
      bool s0_ran = false;
      int l0 = 0;
      if (!w0.done) {
        const bool nxt = can_share && !w1.done && w0.l >= 2 && w1.l == w0.l;
        job(w0, 0, false, nxt);
        s0_ran = true;
        l0 = w0.l;
        w0.advance(tstride, T, s_tile_end, L);
      }
      if (!w1.done) {
        const bool sh = can_share && s0_ran && w1.l >= 2 && w1.l == l0;
        job(w1, 1, sh, false);
        w1.advance(tstride, T, s_tile_end, L);
      }
    }
    if (SAND_T4_PROF) {
      pc[3] = T4CLK() - tl0;
      if (warp == 1 && rank == 0 && lane == 0)
        for (int k = 0; k < 4; ++k) g_t4prof[blockIdx.x][8 + k] = pc[k];
      if (warp == 0) g_t4prof[blockIdx.x][12] = pc[4];
    }
  } else if (warp == 2 || warp == 3) {
    // =========================== IO warps, one per tile slot (warp 2: slot 0, warp 3: slot 1): every global
    // access of the slot's tile rows.  At a tile's layer-1 job the warp waits until the layer-1 MMA consumed the
    // slot's A1 buffer and refills it with the slot's next tile (gathered one tile earlier); at a tile's last
    // job it waits for the team's row sums and stores sdf[perm[row]].  One warp per slot: a slot's next layer-1
    // operand never waits behind the other slot's tile end.
    const int s = warp - 2;
    const uint32_t a1full_dst = rank == 0 ? b_a1full : mapa_shared(b_a1full, 0);
    const float* tcs = tab + p.m.pt_off_csum;
    auto load_perm = [&](long long t, uint32_t (&ix)[4]) {
      const int d = tile_depth4(t, s_tile_end, L);
      const long long r0 = s_start[d] + (t - s_tile_begin[d]) * 256 + (long long)rank * 128;
      const long long rend = s_start[d] + s_count[d];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const long long r = r0 + lane + 32 * k;
        ix[k] = r < rend ? __ldg(p.perm + r) : 0xFFFFFFFFu;
      }
    };
    auto gather = [&](const uint32_t (&ix)[4], float (&x)[4], float (&y)[4], float (&z)[4]) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const size_t i = ix[k] == 0xFFFFFFFFu ? 0 : ix[k];
        x[k] = __ldg(p.pts + 3 * i); y[k] = __ldg(p.pts + 3 * i + 1); z[k] = __ldg(p.pts + 3 * i + 2);
      }
    };
    auto fill = [&](int s, const float (&x)[4], const float (&y)[4], const float (&z)[4]) {
      const uint32_t a1 = sA1 + s * C::A1_BYTES;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int row = lane + 32 * k;
        // split v = hi + lo (bf16 each).  A row, k = 0..15:
        //   x_hi y_hi z_hi | x_hi y_hi z_hi | x_lo y_lo z_lo | 1 1 | 0 0 0 0 0
        const uint32_t hxy = pack_bf16x2(x[k], y[k]);
        const uint32_t hz1 = pack_bf16x2(z[k], 1.0f);
        const float xh = __uint_as_float(hxy << 16), yh = __uint_as_float(hxy & 0xFFFF0000u);
        const float zh = __uint_as_float(hz1 << 16);
        const uint32_t lxy = pack_bf16x2(x[k] - xh, y[k] - yh);
        const uint32_t lz1 = pack_bf16x2(z[k] - zh, 1.0f);
        sts128(a1 + l1_off((uint32_t)row, 0), hxy, (hz1 & 0xFFFFu) | (hxy << 16), (hxy >> 16) | (hz1 << 16), lxy);
        sts128(a1 + l1_off((uint32_t)row, 8), lz1, 0x3F80u, 0u, 0u);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(a1full_dst + 8 * s);
        else mbar_arrive_remote(a1full_dst + 8 * s);
      }
    };
    // perm rows of tiles t (cur), t+S (p1), t+2S (p2), t+3S (p3; S = this slot's tile stride); the points of the
    // next tile to fill (px/py/pz) are gathered one whole tile ahead of their use
    uint32_t cur[4], p1[4], p2[4], p3[4];
    float px[4], py[4], pz[4];
    Walk4 w;
    w.start(2ll * pair + s, T, s_tile_end, L);
    {
      const long long t0 = 2ll * pair + s;
#pragma unroll
      for (int k = 0; k < 4; ++k) cur[k] = p1[k] = p2[k] = p3[k] = 0xFFFFFFFFu;
      if (t0 < T) {
        load_perm(t0, cur);
        gather(cur, px, py, pz);
        fill(s, px, py, pz);
      }
      if (t0 + tstride < T) { load_perm(t0 + tstride, p1); gather(p1, px, py, pz); }
      if (t0 + 2 * tstride < T) load_perm(t0 + 2 * tstride, p2);
    }
    unsigned long long io_w[2] = {0, 0};
    const bool iotr = SAND_T4_TRACE && s == 0 && lane == 0;
    auto io_step = [&]() {
      if (w.l == 1) {
        const long long t1 = w.t + tstride;
        if (iotr) T4IO(w.ti, 0);
        if (t1 < T) {
          const long long c0 = T4CLK();
          mbar_wait(b_a1free + 8 * s, (uint32_t)(w.ti & 1));   // this tile's layer-1 MMA has read A1
          if (iotr) T4IO(w.ti, 1);
          if (SAND_T4_PROF) io_w[0] += T4CLK() - c0;
          fill(s, px, py, pz);                                  // next tile's points (gathered a tile ago)
          if (t1 + tstride < T) gather(p2, px, py, pz);         // the tile after: in flight for a whole tile
          if (t1 + 2 * tstride < T) load_perm(t1 + 2 * tstride, p3);
        }
        if (iotr) T4IO(w.ti, 2);
      }
      if (w.l == w.d) {
        const long long c0 = T4CLK();
        if (iotr) T4IO(w.ti, 3);
        mbar_wait(b_iodone + 8 * s, (uint32_t)(w.ti & 1));
        if (iotr) T4IO(w.ti, 4);
        if (SAND_T4_PROF) io_w[1] += T4CLK() - c0;
        const float* pl = part + s * C::NCG * 128;
        const float cs = tcs[w.d];
        float y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float v = cs;
#pragma unroll
          for (int g = 0; g < C::NCG; ++g) v += pl[128 * g + lane + 32 * k];
          y[k] = v;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(b_partfree + 8 * s);
        if (iotr) T4IO(w.ti, 5);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (cur[k] != 0xFFFFFFFFu) p.out[cur[k]] = y[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) { cur[k] = p1[k]; p1[k] = p2[k]; p2[k] = p3[k]; }
        if (iotr) T4IO(w.ti, 6);
      }
    };
#pragma unroll 1
    while (!w.done) {
      io_step();
      w.advance(tstride, T, s_tile_end, L);
    }
    if (SAND_T4_PROF && s == 0 && lane == 0) { g_t4prof[blockIdx.x][13] = io_w[0]; g_t4prof[blockIdx.x][14] = io_w[1]; }
  } else if (warp >= C::NCTL) {
    // =========================== epilogue: one thread per row (TMEM lane), CW columns per thread.  Ping-pong:
    // all warps serve slot 0 and slot 1 step by step (the MMA of one slot overlaps the epilogue of the other);
    // teams: warps [TEAM_WARPS s, TEAM_WARPS (s + 1)) serve slot s only.
    const int ew = warp - C::NCTL;
    const int q = warp & 3;                      // TMEM lane quadrant
    const int cg = (ew % C::TEAM_WARPS) >> 2;    // column group
    const int row = 32 * q + lane;               // this CTA's tile row
    const int c0 = cg * C::CW;
    const uint32_t tm0 = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
    // A operand row segment: element (row, k) of K-chunk kc at kc * 16 KB + (row/8) 1024 + (row%8) 128 +
    // (((k%64)/8) ^ (row%8)) 16 + (k%8) 2
    const uint32_t a_row0 = sA + (uint32_t)(row >> 3) * 1024 + (uint32_t)(row & 7) * 128;
    const uint32_t rx = (uint32_t)(row & 7);
    const uint32_t tab_a = sTab + (uint32_t)p.m.pt_off_a * 4 + (uint32_t)c0 * 4;
    const uint32_t tab_a1 = sTab + (uint32_t)p.m.pt_off_a1 * 4 + (uint32_t)c0 * 4;
    const float* tc0 = tab + p.m.pt_off_c;
    const float* tc1 = tab + p.m.pt_off_c1;
    const uint32_t afull_dst = rank == 0 ? b_afull : mapa_shared(b_afull, 0);
    struct EState {
      Walk4 w;
      uint32_t pe;
      float ylin, yprod;
    };
    unsigned long long tp[4] = {0, 0, 0, 0};   // SAND_T4_PROF: wait_acc, busy, tile_end, steps
    const long long tt0 = T4CLK();

    // one 32-column batch at column offset cb (relative to c0) of layer l: sines, tail dot products, A stores
    auto batch = [&](const uint32_t (&r)[32], const int cb, const uint32_t a_row, const uint32_t ta, const uint32_t ta1,
                     float2 (&y0)[2], float2 (&y1)[2], auto st_c) {
      constexpr bool ST = decltype(st_c)::value;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float hv[8];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          if (4 * g + i / 2 < (ST ? SAND_T4_NPOLY : SAND_T4_NPOLY_LAST)) {
            const float2 hh = sin_poly2(make_float2(__uint_as_float(r[8 * g + i]), __uint_as_float(r[8 * g + i + 1])));
            hv[i] = hh.x;
            hv[i + 1] = hh.y;
          } else {
            hv[i] = sin_mufu(__uint_as_float(r[8 * g + i]));
            hv[i + 1] = sin_mufu(__uint_as_float(r[8 * g + i + 1]));
          }
        }
#if !(SAND_T4_ABL & 8)
#if SAND_T4_ABL & 16
        const float av = __uint_as_float((ta & 0xFFFFu) | 0x3c000000u);   // tail vectors not loaded (LDS cost probe)
        const float4 aa = make_float4(av, av, av, av), ab = aa;
#else
        const float4 aa = lds128f(ta + (uint32_t)(cb + 8 * g) * 4);
        const float4 ab = lds128f(ta + (uint32_t)(cb + 8 * g + 4) * 4);
#endif
        y0[0] = __ffma2_rn(make_float2(aa.x, aa.y), make_float2(hv[0], hv[1]), y0[0]);
        y0[1] = __ffma2_rn(make_float2(aa.z, aa.w), make_float2(hv[2], hv[3]), y0[1]);
        y0[0] = __ffma2_rn(make_float2(ab.x, ab.y), make_float2(hv[4], hv[5]), y0[0]);
        y0[1] = __ffma2_rn(make_float2(ab.z, ab.w), make_float2(hv[6], hv[7]), y0[1]);
        if (TAIL == SAND_TAIL_MULT) {
          const float4 ba = lds128f(ta1 + (uint32_t)(cb + 8 * g) * 4);
          const float4 bb = lds128f(ta1 + (uint32_t)(cb + 8 * g + 4) * 4);
          y1[0] = __ffma2_rn(make_float2(ba.x, ba.y), make_float2(hv[0], hv[1]), y1[0]);
          y1[1] = __ffma2_rn(make_float2(ba.z, ba.w), make_float2(hv[2], hv[3]), y1[1]);
          y1[0] = __ffma2_rn(make_float2(bb.x, bb.y), make_float2(hv[4], hv[5]), y1[0]);
          y1[1] = __ffma2_rn(make_float2(bb.z, bb.w), make_float2(hv[6], hv[7]), y1[1]);
        }
#endif
        if (ST) {
          const uint32_t k = (uint32_t)(c0 + cb + 8 * g);   // first column of this 8-column unit
          const uint32_t addr = a_row + (k >> 6) * C::A_CHUNK + ((((k & 63) >> 3) ^ rx) << 4);
#if SAND_T4_ABL & 2
          if (hv[0] == 1234.5f)
#endif
          sts128(addr, pack_k<0>(hv[0], hv[1]), pack_k<1>(hv[2], hv[3]), pack_k<2>(hv[4], hv[5]), pack_k<3>(hv[6], hv[7]));
        }
      }
    };

    // one step (layer l of the slot's current tile)
    int ec = 0;   // step counter (trace)
    const bool etr = SAND_T4_TRACE && ew == 0 && lane == 0;
    auto step = [&](EState& e, const int s) {
      const int l = e.w.l, d = e.w.d;
      if (etr) T4TR(ec, 4);
      const uint32_t tm = tm0 + (uint32_t)(s * H);
      const uint32_t a_row = a_row0 + (uint32_t)(s * C::A_BYTES);
      const long long c0 = T4CLK();
      mbar_wait(b_accfull + 8 * s, e.pe);
      const long long c1 = T4CLK();
      if (etr) T4TR(ec, 5);
      e.pe ^= 1u;
      tc_fence_after();
      const bool prod = TAIL == SAND_TAIL_MULT && l >= 2;
      const uint32_t ta = tab_a + (uint32_t)((l - 1) * H) * 4;
      const uint32_t ta1 = tab_a1 + (uint32_t)((l >= 2 ? l - 2 : 0) * H) * 4;
      float2 y0[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      float2 y1[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      auto run = [&](auto st_c) {
        uint32_t ra[32], rb[32];
#if SAND_T4_ABL & 4
#pragma unroll
        for (int i = 0; i < 32; ++i) { ra[i] = __float_as_uint(0.01f * (i + lane)); rb[i] = ra[i] ^ 1u; }
#else
        tmem_ld32(tm, ra);
#endif
#pragma unroll 1
        for (int b = 0; b < C::NB; b += 2) {
#if !(SAND_T4_ABL & 4)
          tmem_wait_ld_dep(ra);
          if (b + 1 < C::NB) tmem_ld32(tm + (uint32_t)(32 * (b + 1)), rb);
#endif
          batch(ra, 32 * b, a_row, ta, ta1, y0, y1, st_c);
          if (b + 1 < C::NB) {
#if !(SAND_T4_ABL & 4)
            tmem_wait_ld_dep(rb);
            if (b + 2 < C::NB) tmem_ld32(tm + (uint32_t)(32 * (b + 2)), ra);
#endif
            batch(rb, 32 * (b + 1), a_row, ta, ta1, y0, y1, st_c);
          }
        }
      };
      const bool store = l != d;
      if (store) run(std::true_type{});
      else run(std::false_type{});
      // publish: the accumulator has been read (all tcgen05.ld waited) and, unless this was the tile's last
      // layer, the next layer's A rows of this thread are written
      if (store) fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(afull_dst + 8 * s);
        else mbar_arrive_remote(afull_dst + 8 * s);
      }
      if (etr) T4TR(ec, 6);
      const float dot0 = (y0[0].x + y0[0].y) + (y0[1].x + y0[1].y);
      if (prod) {
        const float dot1 = (y1[0].x + y1[0].y) + (y1[1].x + y1[1].y);
        if (C::NCG == 1) e.yprod += (tc0[l - 1] + dot0) * (tc1[l - 1] + dot1);
      } else {
        e.ylin += dot0;
      }
      const long long c2 = T4CLK();
      if (SAND_T4_PROF) { tp[0] += c1 - c0; tp[1] += c2 - c1; tp[3] += 1; }
      if (l == d) {
        // tile end: hand this row's sum to the IO warp (which adds the tail-bias prefix sum csum[d])
        mbar_wait(b_partfree + 8 * s, (uint32_t)((e.w.ti & 1) ^ 1));
        if (etr && s == 0) T4IO(e.w.ti, 7);
        part[(s * C::NCG + cg) * 128 + row] = e.ylin + e.yprod;
        e.ylin = 0.f;
        e.yprod = 0.f;
        __syncwarp();
        if (lane == 0) mbar_arrive(b_iodone + 8 * s);
        if (SAND_T4_PROF) tp[2] += T4CLK() - c2;
      }
      e.w.advance(tstride, T, s_tile_end, L);
      if (etr) T4TR(ec, 7);
      ++ec;
    };
    int s_team = 0;
    if (PP) {
      EState e0, e1;
      e0.w.start(2ll * pair, T, s_tile_end, L);
      e1.w.start(2ll * pair + 1, T, s_tile_end, L);
      e0.pe = e1.pe = 0;
      e0.ylin = e0.yprod = e1.ylin = e1.yprod = 0.f;
#pragma unroll 1
      while (!(e0.w.done && e1.w.done)) {
        if (!e0.w.done) step(e0, 0);
        if (!e1.w.done) step(e1, 1);
      }
    } else {
      s_team = ew / C::TEAM_WARPS;
      EState e;
      e.w.start(2ll * pair + s_team, T, s_tile_end, L);
      e.pe = 0;
      e.ylin = e.yprod = 0.f;
#pragma unroll 1
      while (!e.w.done) step(e, s_team);
    }
    if (SAND_T4_PROF && q == 0 && cg == 0 && lane == 0) {
      for (int k = 0; k < 4; ++k) g_t4prof[blockIdx.x][4 * s_team + k] = tp[k];
      if (s_team == 0) g_t4prof[blockIdx.x][15] = T4CLK() - tt0;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_cg2(tmem_base, C::TMEM_COLS);
}

// ------------------------------------------------------------------------------------ host side
template <int H, int TAIL>
static size_t smem_for4(long long pt_floats, int L, int nst) {
  using C = Tc4Shape<H, tc4_pp<H, TAIL>()>;
  const size_t tab_bytes = (size_t)((pt_floats + 3) & ~3ll) * 4;
  return (size_t)2 * C::A_BYTES + (size_t)nst * C::CHUNK + 2 * C::BIAS_BYTES + C::W1_BYTES +
         2 * C::A1_BYTES + tab_bytes + (size_t)2 * C::NCG * 128 * 4 + 4 * (size_t)(L + 2) * sizeof(long long) +
         (3 * nst + 6 + 12) * 8 + 16;
}

static constexpr size_t kSmemMax4 = 232448;

template <int H, int TAIL>
static int pick_nst4(long long pt_floats, int L) {
  int best = 0;
  for (int nst = 2; nst <= 8; ++nst)
    if (smem_for4<H, TAIL>(pt_floats, L, nst) <= kSmemMax4) best = nst;
  return best;
}

bool tc4_available(int H, int tail) {
  // Eq. 3 products need both full dot products of a row in one thread
  return (H == 64 || H == 128 || H == 256) && (tail == SAND_TAIL_LINEAR || SAND_T4_NCG == 1);
}

bool tc4_runs(int L, int H, int tail, int prec, int pair_mode) {
  return prec == SAND_BF16 && pair_mode == 2 && tc4_usable(L, H, tail);
}

bool tc4_usable(int L, int H, int tail) {
  if (!tc4_available(H, tail)) return false;
  MlpDev m{};
  tc2_table_layout(L, H, tail, &m, false);
  const bool mult = tail == SAND_TAIL_MULT;
  switch (H) {
    case 64: return (mult ? pick_nst4<64, 1>(m.pt_floats, L) : pick_nst4<64, 0>(m.pt_floats, L)) > 0;
    case 128: return (mult ? pick_nst4<128, 1>(m.pt_floats, L) : pick_nst4<128, 0>(m.pt_floats, L)) > 0;
    case 256: return (mult ? pick_nst4<256, 1>(m.pt_floats, L) : pick_nst4<256, 0>(m.pt_floats, L)) > 0;
    default: return false;
  }
}

static inline uint16_t bf16_rne4(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)((u >> 16) | ((u & 0xFFFF) ? 0x40 : 0));  // inf/nan
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static inline void bf16_split4(float v, uint16_t* hi, uint16_t* lo) {
  *hi = bf16_rne4(v);
  uint32_t u = (uint32_t)*hi << 16;
  float h;
  std::memcpy(&h, &u, 4);
  *lo = bf16_rne4(v - h);
}

// Images of the team kernel.  Output feature n (= accumulator column n = K index n of the next layer) is B row
// n % (H/2) of CTA n / (H/2) (cta_group::2 takes an instruction's first N/2 B rows from the even CTA).
//   w1img : [2 CTAs][H/2 rows][16 bf16] (l1_off layout): (W_hi x y z | W_lo x y z | W_hi x y z | b_hi b_lo | 0)
//           of w0 W_1, w0 b_1 against the IO warp's A row (x_hi | x_hi | x_lo | 1 1 | 0)
//   img   : [L-1 layers][2 CTAs] runs of [bias operand: H/2 rows x 16 bf16, (w0 b_hi, w0 b_lo) at k = 9, 10, the
//           columns where the layer-1 A operand (the bias MMA's A) holds 1, 1]
//           [KC K-chunks of bf16(w0 W_l): H/2 rows x 128 B, SW128 K-major]
void tc4_build_host(int L, int H, float w0, const float* const* W, const float* const* b, std::vector<uint16_t>* w1img,
                    std::vector<uint8_t>* img) {
  const int NR = H / 2, KC = H / 64;
  const size_t bias_bytes = (size_t)NR * 32, chunk = (size_t)NR * 128, layer = bias_bytes + KC * chunk;
  w1img->assign((size_t)H * 16, 0);
  for (int n = 0; n < H; ++n) {
    const int cta = n / NR, r = n % NR;
    auto put = [&](int k, uint16_t v) { (*w1img)[((size_t)cta * NR * 32 + l1_off((uint32_t)r, (uint32_t)k)) / 2] = v; };
    for (int k = 0; k < 3; ++k) {
      uint16_t hi, lo;
      bf16_split4(w0 * W[0][3 * n + k], &hi, &lo);
      put(k, hi);
      put(3 + k, lo);
      put(6 + k, hi);
    }
    uint16_t bhi, blo;
    bf16_split4(w0 * b[0][n], &bhi, &blo);
    put(9, bhi);
    put(10, blo);
  }
  img->assign(L >= 2 ? (size_t)(L - 1) * 2 * layer : 0, 0);
  for (int i = 1; i < L; ++i)
    for (int n = 0; n < H; ++n) {
      const int cta = n / NR, r = n % NR;
      uint8_t* run = img->data() + ((size_t)(i - 1) * 2 + cta) * layer;
      uint16_t bhi, blo;
      bf16_split4(w0 * b[i][n], &bhi, &blo);
      std::memcpy(run + l1_off((uint32_t)r, 9), &bhi, 2);
      std::memcpy(run + l1_off((uint32_t)r, 10), &blo, 2);
      for (int k = 0; k < H; ++k) {
        const int kc = k / 64, kk = k % 64;
        const size_t byte = bias_bytes + kc * chunk + (size_t)(r / 8) * 1024 + (r % 8) * 128 +
                            (size_t)(((kk / 8) ^ (r % 8)) * 16) + (kk % 8) * 2;
        const uint16_t v = bf16_rne4(w0 * W[i][(size_t)n * H + k]);
        std::memcpy(run + byte, &v, 2);
      }
    }
}

template <int H, int TAIL>
static cudaError_t launch_tc4_t(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                                float* out, int num_sms, cudaStream_t st) {
  const int nst = pick_nst4<H, TAIL>(m.pt_floats, m.L);
  if (!nst) return cudaErrorInvalidConfiguration;
  const size_t sm = smem_for4<H, TAIL>(m.pt_floats, m.L, nst);
  Tc4Params p{m, pts, perm, meta, out, nst};
  const int grid = num_sms & ~1;
  k_tmlp_tc4<H, TAIL><<<grid, Tc4Shape<H, tc4_pp<H, TAIL>()>::THREADS, sm, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (SAND_T4_TRACE && e == cudaSuccess) {
    static long long tr[kT4Trace][8];
    e = cudaStreamSynchronize(st);
    for (int which = 0; which < 2 && e == cudaSuccess; ++which) {
      e = which ? cudaMemcpyFromSymbol(tr, g_t4iotr, sizeof tr) : cudaMemcpyFromSymbol(tr, g_t4trace, sizeof tr);
      FILE* f = e == cudaSuccess ? fopen(which ? "gpurun_out/t4iotrace.txt" : "gpurun_out/t4trace.txt", "w") : nullptr;
      if (f) {
        for (int j = 0; j < kT4Trace; ++j)
          fprintf(f, "%lld %lld %lld %lld %lld %lld %lld %lld\n", tr[j][0], tr[j][1], tr[j][2], tr[j][3], tr[j][4], tr[j][5],
                  tr[j][6], tr[j][7]);
        fclose(f);
      }
    }
  }
  if (SAND_T4_PROF && e == cudaSuccess) {
    // diagnostic build only: synchronous dump of the per-role counters (CTA averages; MMA over leaders)
    static unsigned long long h[160][kT4Prof];
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(h, g_t4prof, sizeof h);
    if (e == cudaSuccess) {
      double a[kT4Prof] = {0};
      for (int b = 0; b < grid; ++b)
        for (int k = 0; k < kT4Prof; ++k) a[k] += (double)h[b][k] / ((k >= 8 && k <= 11) ? grid / 2 : grid);
      for (int r = 0; r < 2; ++r) {   // even (leader) and odd CTAs separately: the odd CTA's arrivals are remote
        double q[kT4Prof] = {0};
        for (int b = r; b < grid; b += 2)
          for (int k = 0; k < kT4Prof; ++k) q[k] += (double)h[b][k] / (grid / 2);
        fprintf(stderr, "[t4prof] rank %d team0: loop %.0f wait_acc %.0f busy %.0f tile_end %.0f | IO0: wait_a1free %.0f wait_iodone %.0f\n",
                r, q[15], q[0], q[1], q[2], q[13], q[14]);
      }
      fprintf(stderr,
              "[t4prof] nst %d | team0: loop %.0f wait_acc %.0f busy %.0f tile_end %.0f steps %.0f | team1: wait_acc %.0f "
              "busy %.0f tile_end %.0f steps %.0f | MMA: loop %.0f wait_afull %.0f wait_a1full %.0f wait_w %.0f | "
              "producer wait_empty %.0f | IO0: wait_a1free %.0f wait_iodone %.0f\n",
              nst, a[15], a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[11], a[8], a[9], a[10], a[12], a[13], a[14]);
    }
  }
  return e;
}

template <int H, int TAIL>
static cudaError_t prep_tc4_t() {
  return cudaFuncSetAttribute(k_tmlp_tc4<H, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax4);
}

#define SAND_TC4_DISPATCH(FN, ...)                                                                    \
  do {                                                                                                \
    const bool mult = m_tail == SAND_TAIL_MULT;                                                       \
    switch (m_H) {                                                                                    \
      case 64: return mult ? FN<64, 1>(__VA_ARGS__) : FN<64, 0>(__VA_ARGS__);                         \
      case 128: return mult ? FN<128, 1>(__VA_ARGS__) : FN<128, 0>(__VA_ARGS__);                      \
      case 256: return mult ? FN<256, 1>(__VA_ARGS__) : FN<256, 0>(__VA_ARGS__);                      \
      default: return cudaErrorInvalidValue;                                                          \
    }                                                                                                 \
  } while (0)

cudaError_t launch_tmlp_tc4(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                            float* out, int num_sms, cudaStream_t st) {
  const int m_H = m.H, m_tail = m.tail;
  SAND_TC4_DISPATCH(launch_tc4_t, m, pts, perm, meta, out, num_sms, st);
}

cudaError_t prepare_tc4(int H, int tail) {
  const int m_H = H, m_tail = tail;
  SAND_TC4_DISPATCH(prep_tc4_t);
}

}  // namespace sand
