// tmlp_tc2.cu -- CTA-pair (cta_group::2) persistent fused T-MLP kernel (SAND_BF16, H in {64, 128, 256}).
//
// Computes, per binned 256-row tile of uniform exit depth d (Sec. 3.4):
//   layer 1   : Z_1 = x W_1^T + b_1 as ONE tcgen05 MMA with K = 16 in split-BF16 form (R20):
//               x = x_hi + x_lo, W_1 = W_hi + W_lo, b_1 = b_hi + b_lo (bf16 each), A row =
//               (x_hi, x_hi, x_lo, 1, 1, 0...), B row = (W_hi, W_lo, W_hi, b_hi, b_lo, 0...), so the FP32
//               accumulator holds x_hi W_hi + x_hi W_lo + x_lo W_hi + b (relative error ~2^-16)
//   layer 2..d: Z_l = [1 1 0..] [b_hi b_lo 0..]^T + H_{l-1} W_l^T: one K = 16 MMA puts the bias (split-BF16,
//               exact to ~2^-16) into the accumulator, then the K = H product (M = 256 over the CTA pair,
//               N = H, BF16 in, FP32 in TMEM).  w0 is folded into every weight and bias on the host, so the
//               accumulator holds w0 (W_l h + b_l) and the epilogue applies no scale and no bias.
//   every l   : epilogue h_l = sin(Z_l), t_l (Eq. 2 linear or Eq. 3 product), bf16(h_l) -> A
//   output    : sdf[perm[row]] = y_d = sum_{l <= d} t_l (Eq. 2).
//
// Warp roles (per CTA of the pair; "leader" = even CTA):
//   warp 0       weight producer (lane 0): this CTA's half (H/2 rows) of the job's B operands into an
//                NST-stage ring (w_full / w_empty mbarriers), one bulk async copy (TMA engine) per stage:
//                layer 1: the split-BF16 W_1 operand (K = 16); layer l >= 2: stage 0 = bias operand (K = 16)
//                + 2 K-chunks of W_l, later stages 2 K-chunks each
//   warp 1       TMEM allocator (2 accumulator slots x H columns); leader: the tcgen05.mma.cta_group::2
//                issuer (converged warp, one elected lane issues 4 K-steps per asm block); odd CTA: relays
//                "my half landed" (w_peer)
//   warp 2       IO: all global traffic of the tile rows -- gathers perm -> points, writes the split-BF16
//                layer-1 A operand (a1_full), drains finished tiles (partials + csum -> sdf[perm[row]])
//   warps 3..18  16 epilogue warps = 4 TMEM lane quadrants x 4 column quarters.  All of them work on one
//                tile slot at a time, alternating slot 0 / slot 1 step by step, so the MMA of one slot
//                overlaps the epilogue of the other (ping-pong).  A step = one layer of one slot.  They
//                issue no global memory operations (their proxy fence never waits on DRAM).
//                (Compile-time SAND_EPI5=1 at H = 256: 20 warps in 5 column groups of 7/7/6/6/6 8-column
//                chunks at 80 registers -- measured 3% slower.)
// Every role walks the same deterministic step sequence (rounds: slot 0 then slot 1; a slot's steps are
// its tiles' layers 1..d).  The MMA order equals the epilogue order, so the ping-pong cannot deadlock.
//
// Sine: MUFU.SIN (__sinf).  A compile-time share SAND_PP8 of every 8 element pairs can instead use an odd
// polynomial on the FMA pipe after a radian range reduction (measured slower on B200: FFMA2 retires one
// pair per 2 clk per SMSP, so a 8-instruction polynomial pair costs as much pipe time as two MUFU sines;
// DESIGN.md).
//
// Tails: LINEAR tails sum linearly over layers, so every thread keeps a running partial over its columns;
// the IO warp adds the four column quarters of a row and the tail-bias prefix sum csum[d] once per tile.
// MULT (Eq. 3) products need both full dot products per layer: reduced per step through SMEM.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include <type_traits>

#include "ptx.cuh"

#ifndef SAND_SPLIT_STORE
#define SAND_SPLIT_STORE 1   // separate store / exit-step code paths (no per-chunk store predicate; +1.3% C2)
#endif
#ifndef SAND_EPI5
#define SAND_EPI5 0
#endif
#ifndef SAND_PP8
#define SAND_PP8 0   // poly-sine pairs per 8 (radian reduction, any column); experiment
#endif
#ifndef SAND_W1RES
#define SAND_W1RES 1   // layer-1 B operand resident in shared memory (else streamed through the ring)
#endif
#ifndef SAND_ONES_A1
#define SAND_ONES_A1 0   // 1: bias MMA reads its (1, 1) A columns from the slot's layer-1 operand (k = 9, 10; same speed, saves 4 KB)
#endif
#ifndef SAND_SC
#define SAND_SC 2        // K-chunks per weight-ring stage
#endif
#ifndef SAND_SMR
#define SAND_SMR 0   // 1: 4 control warps (one warpgroup) shrink to SAND_SMR_CTL registers, the 16 epilogue warps grow to SAND_SMR_EPI
#endif
#ifndef SAND_SMR_CTL
#define SAND_SMR_CTL 64
#endif
#ifndef SAND_SMR_EPI
#define SAND_SMR_EPI 104
#endif
// setmaxnreg.inc only draws on registers the CTA released with .dec: the launch gives every one of the 640
// threads 96 registers (65536 / 640, rounded down to 8), so 16 epilogue warps may grow by at most what 4
// control warps give back, else the .inc waits forever.
static_assert(!SAND_SMR || 4 * (SAND_SMR_EPI - 96) <= 96 - SAND_SMR_CTL, "setmaxnreg budget");
#ifndef SAND_BW
#define SAND_BW 16   // accumulator columns per TMEM load batch (8, 16 or 32)
#endif
#ifndef SAND_EPI_BARWAIT
#define SAND_EPI_BARWAIT 1   // accumulator waits: one polling warp per column group + a named barrier
#endif
#ifndef SAND_HALFSTAGE
#define SAND_HALFSTAGE 0   // 1: ring stages of half a pass (KC/2 K-chunks; the first carries the bias), twice as many
#endif
#ifndef SAND_EARLY_LO
#define SAND_EARLY_LO 0   // 1: publish the first K-half of the next A as soon as it is stored (pass-1 start)
#endif
#ifndef SAND_DEFER_PUB
#define SAND_DEFER_PUB 0   // 1: publish a step's A after the first batch of the other slot's next step; 2: after its pass 0
#endif
#ifndef SAND_PDEG
#define SAND_PDEG 7
#endif
#ifndef SAND_DIAG
#define SAND_DIAG 0   // 1: diagnostic modes SAND_KPROF=2/3 (timing studies; build with SAND_BUILD_DEFS=-DSAND_DIAG=1)
#endif
#include "sand_internal.h"

#ifndef SAND_ABL
#define SAND_ABL 0   // ablation builds for timing studies (scripts/abl.sh); 0 = the product kernel
#endif

namespace sand {

template <int H>
struct Tc2Shape {
  static constexpr int KC = H / 64;                // 64-wide K chunks (128-byte swizzle atoms)
  static constexpr int A_CHUNK = 128 * 128;        // one K-chunk of this CTA's 128 rows (bytes)
  static constexpr int A_BYTES = KC * A_CHUNK;
  // Every layer's MMA runs as two N-half passes (N = H/2 each, committed separately), so the epilogue starts
  // on the first half while the tensor pipe computes the second.  cta_group::2 takes an instruction's N rows
  // of B half from each CTA: a CTA holds QR = H/4 rows per pass.
  static constexpr int HN = H / 2;                 // output columns per pass
  static constexpr int QR = H / 4;                 // B rows per CTA per pass
  static constexpr int QCHUNK = QR * 128;          // one K-chunk of a CTA's pass rows (SW128, bytes)
  static constexpr int QSMALL = QR * 32 < 1024 ? 1024 : QR * 32;   // K = 16 bias operand of a pass (padded so
                                                   // the SW128 chunks that follow stay 1024-aligned)
  static constexpr int PASS_BYTES = QSMALL + KC * QCHUNK;   // one pass in the image: [bias operand][KC K-chunks]
  static constexpr int SPP = (SAND_HALFSTAGE && KC >= 2) ? 2 : 1;   // ring stages per pass
  static constexpr int CPS = KC / SPP;                      // K-chunks per stage
  static constexpr int STAGE = QSMALL + CPS * QCHUNK;       // ring slot: [bias operand (first stage of a pass)][CPS chunks]
  static constexpr int A1_BYTES = 128 * 32;        // layer-1 A operand: 128 rows x 16 bf16
  static constexpr int W1_BYTES = 2 * QR * 32;     // resident layer-1 B operand: this CTA's 2 x QR rows
  static constexpr int ONES_BYTES = SAND_ONES_A1 ? 0 : 128 * 32;   // bias MMA A operand: 128 rows of (1, 1, 0, ...)
  static constexpr int BIAS_K = SAND_ONES_A1 ? 9 : 0;               // k of (b_hi, b_lo) in the bias operand
  static constexpr int NSLOT = 2;
  static constexpr int CQ = HN / 4;                // columns per epilogue column group per pass
  static constexpr int TMEM_COLS = 2 * H <= 128 ? 128 : (2 * H <= 256 ? 256 : 512);
  static constexpr int NGRP = 4;                   // epilogue column groups (x 4 TMEM lane quadrants = 16 warps)
  static constexpr int NCTL = SAND_SMR ? 4 : 3;    // control warps (a whole warpgroup when registers are rebalanced)
  static constexpr int THREADS = 32 * NCTL + 128 * NGRP;  // control warps + 16 epilogue warps
  static constexpr int TILE = 256;
  static_assert(H % 64 == 0 && H <= 256 && CQ % 8 == 0, "CTA-pair kernel: H in {64, 128, 192, 256}");
};

struct Tc2Params {
  MlpDev m;
  const float* pts;
  const uint32_t* perm;
  const QueryMeta* meta;
  float* out;
  int nst;
  int prof;   // diagnostic (SAND_OPT_KPROF, -DSAND_DIAG=1 builds only): per-role clock64 counters -> g_kprof
};

// Diagnostic counters (only written when Tc2Params::prof != 0), per CTA:
//  0 MMA wait A (a_full / a1_full)  1 MMA wait weights  2 MMA loop total  3 MMA jobs
//  4 producer wait w_empty  5 producer loads
//  6 epi wait acc_full  7 epi busy (steps excl. waits)  8 epi loop total  9 epi steps
//  10 IO wait  11 IO busy
constexpr int kProfSlots = 14;   // + 12 epi publish, 13 epi tile end
__device__ unsigned long long g_kprof[160][kProfSlots];

// ------------------------------------------------------------------------------ step sequence
__device__ __forceinline__ int tile_depth2(long long t, const long long* te, int L) {
  for (int d = L; d >= 1; --d)
    if (t < te[d]) return d;
  return 0;
}

// Per-slot walk over this pair's tiles: tile i of slot s is pair + npairs * (2 i + s); each tile yields
// steps l = 1..d.  Callers interleave slot 0 and slot 1 round by round.
struct SlotWalk {
  long long t;
  int d, l;
  int ti;   // index of the current tile among this slot's tiles (its IO / layer-1 buffer = ti & 1)
  bool done;
  __device__ __forceinline__ void set(long long t_, long long T, const long long* te, int L) {
    t = t_;
    done = t >= T;
    l = 1;
    d = done ? 0 : tile_depth2(t, te, L);
  }
  __device__ __forceinline__ void start(long long t0, long long T, const long long* te, int L) {
    ti = 0;
    set(t0, T, te, L);
  }
  __device__ __forceinline__ void advance(long long stride, long long T, const long long* te, int L) {
    if (l == d) { ++ti; set(t + stride, T, te, L); }
    else ++l;
  }
};

// ------------------------------------------------------------------------------ sine paths
// Radian-domain polynomial sine (FMA pipe only), any z: k = rint(z / 2 pi) by the 1.5 * 2^23 magic add
// fused into the scaling FMA, r = z - 2 pi k in [-pi, pi], sin r = r P(r^2), odd minimax fit on [-pi, pi]
// (degree 7: |err| < 2.6e-4; degree 9: < 6.2e-6, float32 Horner).
__device__ __forceinline__ float2 sin_poly_rad2(float2 z) {
  const float2 t = __ffma2_rn(z, make_float2(0.15915494309189535f, 0.15915494309189535f),
                              make_float2(12582912.0f, 12582912.0f));
  const float2 k = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 r = __ffma2_rn(k, make_float2(-6.283185307179586f, -6.283185307179586f), z);
  const float2 r2 = __fmul2_rn(r, r);
#if SAND_PDEG == 9
  float2 p = __ffma2_rn(r2, make_float2(2.1478720100276405e-06f, 2.1478720100276405e-06f),
                        make_float2(-0.00019264993898104876f, -0.00019264993898104876f));
  p = __ffma2_rn(p, r2, make_float2(0.008308985270559788f, 0.008308985270559788f));
  p = __ffma2_rn(p, r2, make_float2(-0.16662438213825226f, -0.16662438213825226f));
  p = __ffma2_rn(p, r2, make_float2(0.9999793767929077f, 0.9999793767929077f));
#else
  float2 p = __ffma2_rn(r2, make_float2(-0.0001450767886126414f, -0.0001450767886126414f),
                        make_float2(0.007958059199154377f, 0.007958059199154377f));
  p = __ffma2_rn(p, r2, make_float2(-0.16566696763038635f, -0.16566696763038635f));
  p = __ffma2_rn(p, r2, make_float2(0.9992758631706238f, 0.9992758631706238f));
#endif
  return __fmul2_rn(p, r);
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Per-slot epilogue state (kept in registers: two named instances, never indexed at run time).
struct EpiSlot {
  SlotWalk w;
  uint32_t pe;        // acc_full parity
  uint32_t kpar;      // MULT per-step reduction buffer parity
  float ylin[4];      // this thread's running partials of the linear tail terms (its 4 rows)
  float yprod;        // MULT: sum of the Eq. 3 products (column-quarter 0 warps, row 32 q + lane)
};

template <int H, int TAIL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Tc2Shape<H>::THREADS, 1)
    k_tmlp_tc2(const Tc2Params p) {
  using C = Tc2Shape<H>;
  constexpr int NSLOT = C::NSLOT;
  extern __shared__ uint8_t smem_raw[];
  // The dynamic window starts after the 1 KB reserved system area, i.e. 1024-aligned (required by the
  // SW128 operands; no slack is budgeted for re-alignment).
  const uint32_t base = smem_u32(smem_raw);
  if (base & 1023u) __trap();
  uint8_t* gbase = smem_raw;
  const int nst = p.nst;
  const int L = p.m.L;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // ---- shared memory carve-up (identical offsets in both CTAs: the pair MMA relies on it)
  const uint32_t sA = base;                                       // [slot] KC x 16 KB, SW128 K-major
  const uint32_t sW = sA + NSLOT * C::A_BYTES;                    // weight ring, nst x STAGE
  const uint32_t sOnes = sW + nst * C::STAGE;                     // bias-MMA A operand (constant; unless ONES_A1)
  const uint32_t sW1 = sOnes + C::ONES_BYTES;                     // resident layer-1 B operand (both passes)
  const uint32_t sA1 = sW1 + C::W1_BYTES;                         // [slot] layer-1 A operand
  float* tab = reinterpret_cast<float*>(gbase + ((sA1 + NSLOT * C::A1_BYTES) - base));
  const long long ntab = p.m.pt_floats;
  constexpr int NGRP = C::NGRP;
  constexpr int NPL = TAIL == SAND_TAIL_MULT ? NGRP + 1 : NGRP;   // partial planes: column groups (+ Eq. 3 products)
  float* part = tab + ((ntab + 3) & ~3ll);                        // [slot][plane][128] tile-end partials
  float2* red2 = reinterpret_cast<float2*>(part + NSLOT * NPL * 128);   // MULT: [slot][kpar][cq][128]
  const int red2_floats = (TAIL == SAND_TAIL_MULT) ? NSLOT * 2 * NGRP * 128 * 2 : 0;
  const int nb = L + 2;
  long long* meta_s = reinterpret_cast<long long*>(part + NSLOT * NPL * 128 + red2_floats);
  long long* s_tile_end = meta_s;
  long long* s_tile_begin = meta_s + nb;
  long long* s_start = meta_s + 2 * nb;
  long long* s_count = meta_s + 3 * nb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta_s + 4 * nb);
  const uint32_t b_wfull = smem_u32(bars);
  const uint32_t b_wempty = b_wfull + 8 * nst;
  const uint32_t b_wpeer = b_wempty + 8 * nst;
  const uint32_t b_afull = b_wpeer + 8 * nst;           // [slot][K-half] epilogue step: A K-chunks [0, KC/2) written +
                                                        // accumulator pass 0 read (lo); all A written + all read (hi)
  const uint32_t b_accfull = b_afull + 16 * NSLOT;      // [slot][pass]  accumulator half ready
  const uint32_t b_a1full = b_accfull + 16 * NSLOT;     // [slot]  layer-1 A written (leader: 2 arrivals)
  const uint32_t b_a1free = b_a1full + 8 * NSLOT;       // [slot]  layer-1 MMA done with the A1 buffer
  const uint32_t b_iodone = b_a1free + 8 * NSLOT;       // [slot]  all epilogue warps wrote their partials
  const uint32_t b_partfree = b_iodone + 8 * NSLOT;     // [slot]  IO warp has read the partials
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * nst + 9 * NSLOT);   // (3 nst + 9 NSLOT) barriers
#ifdef SAND_HANG_DEBUG
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("[bars] wfull 0x%x wempty 0x%x wpeer 0x%x afull 0x%x accfull 0x%x a1full 0x%x a1free 0x%x iodone 0x%x\n",
           b_wfull, b_wempty, b_wpeer, b_afull, b_accfull, b_a1full, b_a1free, b_iodone);
#endif

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const float4* src = reinterpret_cast<const float4*>(p.m.pair_tables);
    float4* dst = reinterpret_cast<float4*>(tab);
    for (long long i = tid; i < (ntab + 3) / 4; i += blockDim.x) dst[i] = src[i];
    // A rows (1, 1, 0, ..., 0) against the bias operand's (b_hi, b_lo, 0, ...): the K = 16 bias MMA
    if (!SAND_ONES_A1) {
      uint32_t* ones = reinterpret_cast<uint32_t*>(gbase + (sOnes - base));
      for (int i = tid; i < C::ONES_BYTES / 4; i += blockDim.x) ones[i] = 0u;
      __syncthreads();
      for (int r = tid; r < 128; r += blockDim.x) ones[l1_off((uint32_t)r, 0) / 4] = 0x3F803F80u;
    }
    {
      const uint4* w1s = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(p.m.w1_image) + rank * C::W1_BYTES);
      uint4* w1d = reinterpret_cast<uint4*>(gbase + (sW1 - base));
      for (int i = tid; i < C::W1_BYTES / 16; i += blockDim.x) w1d[i] = w1s[i];
    }
    if (tid < nb) {
      s_tile_end[tid] = p.meta->tile_end[tid];
      s_tile_begin[tid] = p.meta->tile_begin[tid];
      s_start[tid] = p.meta->start[tid];
      s_count[tid] = p.meta->count[tid];
    }
    fence_proxy_async_smem();   // ones operand (generic stores) -> tensor core (async proxy)
  }
  constexpr uint32_t kEpiWarps = 4 * NGRP;
  if (tid == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(b_wfull + 8 * i, 1);
      mbar_init(b_wempty + 8 * i, 1);
      mbar_init(b_wpeer + 8 * i, 1);
    }
    // a_full: one arrive per epilogue warp of both CTAs
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(b_afull + 16 * s, 2 * kEpiWarps);
      mbar_init(b_afull + 16 * s + 8, 2 * kEpiWarps);
      mbar_init(b_accfull + 16 * s, 1);
      mbar_init(b_accfull + 16 * s + 8, 1);
    }
    for (int s = 0; s < NSLOT; ++s) { mbar_init(b_a1full + 8 * s, 2); mbar_init(b_a1free + 8 * s, 1); }
    for (int s = 0; s < NSLOT; ++s) { mbar_init(b_iodone + 8 * s, kEpiWarps); mbar_init(b_partfree + 8 * s, 1); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_cg2(smem_u32(tmem_slot), C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();   // both CTAs' barriers initialised before any remote arrive / multicast commit
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const long long T = p.meta->total_tiles;
  const long long tstride = 2ll * npairs;

  // Register rebalancing (setmaxnreg is per warpgroup, issued by all its threads at the top of their role
  // branch so that ptxas applies the new limit to the whole role): the control warpgroup (warps 0-3) gives
  // registers back, the epilogue warpgroups take them (per SMSP: 1 control + 4 epilogue warps).
  if (warp < C::NCTL) {
  if (SAND_SMR) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(SAND_SMR_CTL));
  if ((warp == 0 && lane == 0) || warp == 1) {
    {
      // warp 0: producer (lane 0); warp 1: MMA issuer (leader CTA) / relay (odd CTA), all 32 lanes converged,
      // side effects by one elected lane
      // producer / MMA issuer / relay: one job per epilogue step, in the epilogue's order
      SlotWalk w0, w1;
      w0.start(pair, T, s_tile_end, L);
      w1.start(pair + npairs, T, s_tile_end, L);
      // hidden-layer image: [L-1][CTA][pass][STAGE]: one bulk copy per pass
      const uint8_t* img = reinterpret_cast<const uint8_t*>(p.m.w_image_pair) + (size_t)rank * 2 * C::PASS_BYTES;
      const uint32_t peer_wpeer = mapa_shared(b_wpeer, 0);
      constexpr uint32_t ID = idesc_bf16(256, C::HN);
      uint32_t pa[2][2] = {{0, 0}, {0, 0}};   // [slot][lo, hi] a_full parities
      int st = 0;
      uint32_t ph = 0;
      unsigned long long pc[6] = {0, 0, 0, 0, 0, 0};
      const long long t_start = (SAND_DIAG && p.prof) ? clock64() : 0;
      // a_full[s] completes once per epilogue step of slot s (all epilogue warps of both CTAs arrived:
      // A written for the next layer and accumulator read).  Every MMA job but the first of a slot waits
      // for the previous step of its slot, so the accumulator is never overwritten while read.
      auto wait_prev_half = [&](const SlotWalk& w, int s, int hi) {
        if (w.ti == 0 && w.l == 1) return;
        const long long c0_ = (SAND_DIAG && p.prof) ? clock64() : 0;
        mbar_wait_cluster(b_afull + 16 * s + 8 * hi, pa[s][hi]);
        if (SAND_DIAG && p.prof) { pc[0] += clock64() - c0_; pc[3] += hi; }
        pa[s][hi] ^= 1u;
      };
      auto wait_prev_step = [&](const SlotWalk& w, int s) { wait_prev_half(w, s, 0); wait_prev_half(w, s, 1); };
      auto job = [&](const SlotWalk& w, int s) {
        const int l = w.l;
        const int nsj = l == 1 ? 0 : 2 * C::SPP;   // ring stages of this job
        if (warp == 0) {
          for (int j = 0; j < nsj && !(SAND_DIAG && p.prof == 3); ++j) {
            const long long c0_ = (SAND_DIAG && p.prof) ? clock64() : 0;
            mbar_wait_lazy(b_wempty + 8 * st, ph ^ 1u);
            if (SAND_DIAG && p.prof) { pc[4] += clock64() - c0_; pc[5] += 1; }
            // stage j = pass j / SPP, part j % SPP: part 0 = [bias | CPS chunks], part 1 = the other CPS chunks
            const uint8_t* pb = img + ((size_t)(l - 2) * 4 + j / C::SPP) * C::PASS_BYTES;
            const bool first = (j % C::SPP) == 0;
            const uint32_t bytes = first ? C::STAGE : C::CPS * C::QCHUNK;
            mbar_arrive_expect_tx(b_wfull + 8 * st, bytes);
            bulk_g2s(first ? sW + st * C::STAGE : sW + st * C::STAGE + C::QSMALL,
                     first ? pb : pb + C::QSMALL + (size_t)C::CPS * C::QCHUNK, bytes, b_wfull + 8 * st);
            if (++st == nst) { st = 0; ph ^= 1u; }
          }
        } else if (rank == 0) {
          const bool early = SAND_EARLY_LO && l >= 2 && C::KC >= 2;
          if (early) wait_prev_half(w, s, 0);   // K-chunks [0, KC/2) of A and the pass-0 accumulator are free
          else wait_prev_step(w, s);
          const uint32_t acc = tmem_base + (uint32_t)(s * H);
          if (l == 1) {
            // ---- layer 1: per pass one K = 16 MMA on the split-BF16 operands (A written by the IO warps)
            const long long c0_ = (SAND_DIAG && p.prof) ? clock64() : 0;
            mbar_wait_cluster(b_a1full + 8 * s, (uint32_t)(w.ti & 1));
            if (SAND_DIAG && p.prof) { pc[0] += clock64() - c0_; }
            tc_fence_after();
            const uint64_t a1d = desc_nosw(sA1 + s * C::A1_BYTES, 128, 256);
            mma_bf16_cg2_w(acc, a1d, desc_nosw(sW1, 128, 256), ID, 0u);
            mma_commit_cg2_mc_w(b_accfull + 16 * s, 0x3);
            mma_bf16_cg2_w(acc + C::HN, a1d, desc_nosw(sW1 + C::QR * 32, 128, 256), ID, 0u);
            mma_commit_cg2_mc_w(b_a1free + 8 * s, 0x3);
            mma_commit_cg2_mc_w(b_accfull + 16 * s + 8, 0x3);
            return;
          }
          tc_fence_after();
          // descriptors precomputed once per job / stage: a K-step of 32 B is +2 in the address field.
          // (Computing them per MMA costs the single issuing thread more than the tensor pipe's time.)
          const uint64_t a_d = desc_sw128(sA + s * C::A_BYTES);
          // bias: (1, 1) x (b_hi, b_lo) initialises the accumulator half.  With SAND_ONES_A1 the A operand is
          // the slot's layer-1 operand, whose k = 9, 10 are always 1 (the IO warp may be rewriting its other
          // columns for the next tile meanwhile: they hold finite values and meet zeros in the bias operand,
          // so the product is b_hi + b_lo whichever version the tensor core reads)
          const uint64_t ones_d = desc_nosw(SAND_ONES_A1 ? sA1 + s * C::A1_BYTES : sOnes, 128, 256);
#pragma unroll 1
          for (int jj = 0; jj < 2 * C::SPP; ++jj) {
            const int j = jj / C::SPP, part = jj % C::SPP;   // pass, stage within the pass
            const long long c0_ = (SAND_DIAG && p.prof) ? clock64() : 0;
            if (!(SAND_DIAG && p.prof == 3)) { mbar_wait(b_wfull + 8 * st, ph);
            mbar_wait_cluster(b_wpeer + 8 * st, ph); }   // diagnostic 3: no weight streaming
            if (SAND_DIAG && p.prof) pc[1] += clock64() - c0_;
            tc_fence_after();
            const uint32_t slot = sW + st * C::STAGE;
            const uint32_t d = acc + (uint32_t)(j * C::HN);
            if (part == 0) mma_bf16_cg2_w(d, ones_d, desc_nosw(slot, 128, 256), ID, 0u);
            const uint64_t w_d = desc_sw128(slot + C::QSMALL);
#pragma unroll 1
            for (int c = 0; c < C::CPS; ++c) {
              const int kc = part * C::CPS + c;
              if (early && j == 0 && kc == C::KC / 2) { wait_prev_half(w, s, 1); tc_fence_after(); }
              mma4_bf16_cg2_w(d, a_d + (uint64_t)(kc * (C::A_CHUNK >> 4)), w_d + (uint64_t)(c * (C::QCHUNK >> 4)), ID, 1u);
            }
            mma_commit_cg2_mc_w(b_wempty + 8 * st, 0x3);
            if (part == C::SPP - 1) mma_commit_cg2_mc_w(b_accfull + 16 * s + 8 * j, 0x3);
            if (++st == nst) { st = 0; ph ^= 1u; }
          }
        } else {
          for (int j = 0; j < nsj && !(SAND_DIAG && p.prof == 3); ++j) {
            mbar_wait(b_wfull + 8 * st, ph);
            if (lane == 0) mbar_arrive_remote(peer_wpeer + 8 * st);
            __syncwarp();
            if (++st == nst) { st = 0; ph ^= 1u; }
          }
        }
      };
#pragma unroll 1
      while (!(w0.done && w1.done)) {
        if (!w0.done) { job(w0, 0); w0.advance(tstride, T, s_tile_end, L); }
        if (!w1.done) { job(w1, 1); w1.advance(tstride, T, s_tile_end, L); }
      }
      if (SAND_DIAG && p.prof) {
        pc[2] = clock64() - t_start;
        if (warp == 1 && rank == 0 && lane == 0)
          for (int k = 0; k < 4; ++k) g_kprof[blockIdx.x][k] = pc[k];
        if (warp == 0)
          for (int k = 4; k < 6; ++k) g_kprof[blockIdx.x][k] = pc[k];
      }
    }
  } else if (warp == 2) {
    // =========================== IO warp: every global access of the tile rows
    // Walks the epilogue's step order.  At a tile's layer-1 step it waits until the layer-1 MMA has
    // consumed the slot's A1 buffer (a1_free) and refills it with the slot's next tile (perm rows were
    // loaded one tile earlier, so only the point gather is on the critical path), then prefetches the
    // perm rows of the tile after.  At a tile's last step it waits for y_d (io_done) and stores
    // sdf[perm[row]].  Perm rows live in registers: cur (tile being computed), nxt (next tile, in A1
    // once filled), pre (the tile after).
    const uint32_t a1full_dst = rank == 0 ? b_a1full : mapa_shared(b_a1full, 0);
    const float* tcs = tab + p.m.pt_off_csum;
    unsigned long long io_wait = 0, io_busy = 0;
    auto load_perm = [&](long long t, uint32_t (&ix)[4]) {
      const int d = tile_depth2(t, s_tile_end, L);
      const long long r0 = s_start[d] + (t - s_tile_begin[d]) * C::TILE + (long long)rank * 128;
      const long long rend = s_start[d] + s_count[d];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const long long r = r0 + lane + 32 * k;
        ix[k] = r < rend ? __ldg(p.perm + r) : 0xFFFFFFFFu;
      }
    };
    // point gather of a tile's rows (issued a slot-step before the layer-1 operand is built from them, so the
    // DRAM latency of the 12-byte gathers is off the layer-1 critical path)
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
        const uint32_t hxy = pack_bf16x2(x[k], y[k]);                // lo half = x_hi, hi half = y_hi
        const uint32_t hz1 = pack_bf16x2(z[k], 1.0f);                // lo half = z_hi, hi half = 1
        const float xh = __uint_as_float(hxy << 16), yh = __uint_as_float(hxy & 0xFFFF0000u);
        const float zh = __uint_as_float(hz1 << 16);
        const uint32_t lxy = pack_bf16x2(x[k] - xh, y[k] - yh);      // x_lo, y_lo (exact residuals)
        const uint32_t lz1 = pack_bf16x2(z[k] - zh, 1.0f);           // z_lo, 1
        const uint32_t w0 = hxy;                                     // k 0,1: x_hi y_hi
        const uint32_t w1 = (hz1 & 0xFFFFu) | (hxy << 16);           // k 2,3: z_hi x_hi
        const uint32_t w2 = (hxy >> 16) | (hz1 << 16);               // k 4,5: y_hi z_hi
        const uint32_t w3 = lxy;                                     // k 6,7: x_lo y_lo
        const uint32_t w4 = lz1;                                     // k 8,9: z_lo 1
        const uint32_t w5 = 0x3F80u;                                 // k 10,11: 1 0
        st_shared_v4(a1 + l1_off((uint32_t)row, 0), w0, w1, w2, w3);
        st_shared_v4(a1 + l1_off((uint32_t)row, 8), w4, w5, 0u, 0u);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(a1full_dst + 8 * s);
        else mbar_arrive_remote(a1full_dst + 8 * s);
      }
    };
    struct IoSlot { uint32_t cur[4], nxt[4], pre[4]; float nx[4], ny[4], nz[4]; };
    SlotWalk w0, w1;
    w0.start(pair, T, s_tile_end, L);
    w1.start(pair + npairs, T, s_tile_end, L);
    IoSlot q0, q1;
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      IoSlot& q = s ? q1 : q0;
      const long long t0 = pair + (long long)npairs * s;
#pragma unroll
      for (int k = 0; k < 4; ++k) q.cur[k] = q.nxt[k] = q.pre[k] = 0xFFFFFFFFu;
      if (t0 < T) {
        load_perm(t0, q.cur);
        gather(q.cur, q.nx, q.ny, q.nz);
        fill(s, q.nx, q.ny, q.nz);
      }
      if (t0 + tstride < T) { load_perm(t0 + tstride, q.nxt); gather(q.nxt, q.nx, q.ny, q.nz); }
    }
    auto io_step = [&](const SlotWalk& w, int s, IoSlot& q) {
      const long long c0_ = (SAND_DIAG && p.prof) ? clock64() : 0;
      long long waited = 0;
      if (w.l == 1) {
        const long long t1 = w.t + tstride;
        if (t1 < T) {
          mbar_wait_lazy(b_a1free + 8 * s, (uint32_t)(w.ti & 1));   // this tile's layer-1 MMA read A1
          if (SAND_DIAG && p.prof) waited += clock64() - c0_;
          fill(s, q.nx, q.ny, q.nz);
          if (t1 + tstride < T) load_perm(t1 + tstride, q.pre);
        }
      }
      if (w.l == w.d) {
        const long long c1_ = (SAND_DIAG && p.prof) ? clock64() : 0;
        mbar_wait_lazy(b_iodone + 8 * s, (uint32_t)(w.ti & 1));
        if (SAND_DIAG && p.prof) waited += clock64() - c1_;
        const float* pl = part + s * NPL * 128;
        const float cs = tcs[w.d];
        float y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = lane + 32 * k;
          float v = cs;
#pragma unroll
          for (int g = 0; g < NPL; ++g) v += pl[128 * g + r];
          y[k] = v;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(b_partfree + 8 * s);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (q.cur[k] != 0xFFFFFFFFu) p.out[q.cur[k]] = y[k];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 4; ++k) { q.cur[k] = q.nxt[k]; q.nxt[k] = q.pre[k]; }
        if (w.t + 2 * tstride < T) gather(q.nxt, q.nx, q.ny, q.nz);   // the tile after next: its layer-1 operand
      }
      if (SAND_DIAG && p.prof) { io_wait += waited; io_busy += clock64() - c0_ - waited; }
    };
#pragma unroll 1
    while (!(w0.done && w1.done)) {
      if (!w0.done) { io_step(w0, 0, q0); w0.advance(tstride, T, s_tile_end, L); }
      if (!w1.done) { io_step(w1, 1, q1); w1.advance(tstride, T, s_tile_end, L); }
    }
    if (SAND_DIAG && p.prof && lane == 0) { g_kprof[blockIdx.x][10] = io_wait; g_kprof[blockIdx.x][11] = io_busy; }
  }
  } else {
    if (SAND_SMR) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(SAND_SMR_EPI));
    // =========================== epilogue (16 warps, both slots, step by step)
    const int ew = warp - C::NCTL;
    const int q = warp & 3;                  // TMEM lane quadrant = warp % 4
    const int cq = ew >> 2;                  // column group (quarter when NGRP = 4)
    // TMEM access in the 16x256b shape: thread (quad = lane / 4, tq = lane % 4) owns rows
    // R_k = 32q + quad + 8k (k = 0..3) and, in every 8-column chunk, columns 2 tq and 2 tq + 1.  Each
    // per-column table value it loads serves 4 rows (4x fewer shared-memory table reads than one row per
    // thread), at the price of 4-byte A-operand stores.
    // Columns: the group's CQ columns of each pass, c0 + pass * HN + [0, CQ).
    const int quad = lane >> 2, tq = lane & 3;
    constexpr int NCHP = C::CQ / 8;               // 8-column chunks per group per pass
    const int c0 = cq * C::CQ;
    constexpr int BW = NCHP * 8 >= SAND_BW ? SAND_BW : NCHP * 8;   // columns per TMEM load batch (2 x BW/2 registers)
    constexpr int CB = BW / 8;                    // 8-column chunks per batch
    static_assert(NCHP % CB == 0, "whole TMEM load batches per group");
    const uint32_t tm_q = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
    const uint32_t a_st = sA + (uint32_t)(4 * q + (lane >> 3)) * 1024 + (uint32_t)(lane & 7) * 128;
    const float* tta = tab + p.m.pt_off_a;     // [L][H] tail vectors (a_l or a_l0)
    const float* ta1 = tab + p.m.pt_off_a1;    // [L-1][H] (MULT)
    const float* tc0 = tab + p.m.pt_off_c;     // [L]
    const float* tc1 = tab + p.m.pt_off_c1;    // [L] (MULT, index l-1)
    const uint32_t bar_q = 1 + q;              // per-quadrant named barrier (tile-end / MULT reductions)
    const uint32_t afull_dst0 = rank == 0 ? b_afull : mapa_shared(b_afull, 0);
    unsigned long long ep_wait = 0, ep_busy = 0, ep_steps = 0, ep_pub = 0, ep_tend = 0;

    auto publish_half = [&](int s, bool wrote_a, int hi) {
      if (wrote_a) fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(afull_dst0 + 16 * s + 8 * hi);
        else mbar_arrive_remote(afull_dst0 + 16 * s + 8 * hi);
      }
    };
    // the lo half is published early (SAND_EARLY_LO, at the start of pass 1) or together with the hi half
    auto publish = [&](int s, bool wrote_a) {
      if (!SAND_EARLY_LO) publish_half(s, wrote_a, 0);
      publish_half(s, wrote_a, 1);
    };
    auto quad_sum = [](float v) {
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      return v;
    };

    // one epilogue step (layer l of the current tile) of slot s
    int pend = -1;          // slot whose publish is deferred into the other slot's step (SAND_DEFER_PUB)
    bool pend_store = false;
    auto flush_pend = [&]() {
      if (pend >= 0) { publish(pend, pend_store); pend = -1; }
    };
    auto step = [&](EpiSlot& e, const int s, const bool defer_ok) {
      const int d = e.w.d, l = e.w.l;
      const uint32_t aSt = a_st + s * C::A_BYTES;
      float2 yv[4], yv1[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) { yv[k] = make_float2(0.f, 0.f); yv1[k] = make_float2(0.f, 0.f); }
      long long wt = 0;
      const long long c0_ = (SAND_DIAG && p.prof) ? clock64() : 0;
      const bool store = l != d;
      const float* ta = tta + (l - 1) * H + c0 + 2 * tq;
      const float* a1 = ta1 + (l - 2) * H + c0 + 2 * tq;
      const bool prod = TAIL == SAND_TAIL_MULT && l >= 2;
      const uint32_t tm = tm_q + (uint32_t)(s * H);
      // one 8-column chunk at column offset jc of this group: ra = rows R0, R1; rb = rows R2, R3 (4 regs each)
      auto chunk = [&](const uint32_t* ra, const uint32_t* rb, const int jc, uint32_t (&pk)[4]) {
#if SAND_ABL == 2   // ablation build (timing only): no table loads
        const float2 a2 = make_float2(0.1f * jc, 0.2f);
#else
        const float2 a2 = *reinterpret_cast<const float2*>(ta + jc);
#endif
        float2 c2 = make_float2(0.f, 0.f);
        if (TAIL == SAND_TAIL_MULT && prod) c2 = *reinterpret_cast<const float2*>(a1 + jc);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t* r = k < 2 ? ra : rb;
          const int o = 2 * (k & 1);
          // z = w0 (W h + b) straight from the accumulator (w0 and the bias are folded into the MMA)
          const float2 z = make_float2(__uint_as_float(r[o]), __uint_as_float(r[o + 1]));
          float2 h;
          if (k + 4 * ((jc >> 3) & 1) < SAND_PP8) {
            h = sin_poly_rad2(z);
          } else {
#if SAND_ABL == 4   // ablation build (timing only): no sine
            h = z;
#else
            h = make_float2(__sinf(z.x), __sinf(z.y));
#endif
          }
          yv[k] = __ffma2_rn(a2, h, yv[k]);
          if (TAIL == SAND_TAIL_MULT) yv1[k] = __ffma2_rn(c2, h, yv1[k]);
          pk[k] = pack_bf16x2(h.x, h.y);
        }
      };
      // the 4 rows x 8 columns of a chunk (column offset jc of this group) are four 8x8 b16 matrices in the
      // m8n8 fragment layout: one stmatrix.x4 (lane provides the address of row lane % 8 of matrix lane / 8)
      auto st_chunk = [&](const int jc, const uint32_t (&pk)[4]) {
        const uint32_t u = (uint32_t)((c0 + jc) >> 3);
#if SAND_ABL == 1   // ablation build (timing only): no A-operand stores
        if (pk[0] == 0x12345678u && pk[1] == 0x9u) stmatrix_x4(aSt, pk);
#else
        stmatrix_x4(aSt + (u >> 3) * C::A_CHUNK + (((u & 7u) ^ (uint32_t)(lane & 7)) << 4), pk);
#endif
      };
      // pass-0 h (bf16) is held here until the pass-1 MMA of this layer, which still reads the old A operand,
      // has completed (acc_full of pass 1)
      uint32_t stash[NCHP][4];
      auto math = [&](auto st_c, auto pass_c) {
        constexpr int PO = decltype(pass_c)::value * C::HN;   // column offset of this pass
        constexpr bool ST = SAND_SPLIT_STORE ? decltype(st_c)::value : true;
        {
          const long long w0_ = (SAND_DIAG && p.prof) ? clock64() : 0;
          if (SAND_EPI_BARWAIT) {
            // one warp of the column group polls the mbarrier, the other three sleep in a named barrier
            // (16 spinning warps per CTA would flood the MIO queue the sines use with barrier polls)
            if ((ew & 3) == 0) mbar_wait(b_accfull + 16 * s + 8 * decltype(pass_c)::value, e.pe);
            named_bar_sync(5 + cq, 128);
          } else {
            mbar_wait(b_accfull + 16 * s + 8 * decltype(pass_c)::value, e.pe);
          }
          if (SAND_DIAG && p.prof) wt += clock64() - w0_;
          tc_fence_after();
        }
        if (decltype(pass_c)::value == 1 && ST && (SAND_SPLIT_STORE || store)) {
#pragma unroll
          for (int i = 0; i < NCHP; ++i) st_chunk(8 * i, stash[i]);
        }
        // K-chunks [0, KC/2) of the next A (pass-0 columns) are in place and the pass-0 accumulator has been
        // read: the next layer's MMA may start on them
        if (SAND_EARLY_LO && decltype(pass_c)::value == 1) publish_half(s, ST && (SAND_SPLIT_STORE || store), 0);
#pragma unroll
        for (int bb = 0; bb < NCHP / CB; ++bb) {
          uint32_t r0[4 * CB], r1[4 * CB];   // lane block 0 (rows R0, R1) and block 1 (rows R2, R3)
#if SAND_ABL == 3   // ablation build (timing only): no TMEM loads
#pragma unroll
          for (int q_ = 0; q_ < 4 * CB; ++q_) { r0[q_] = __float_as_uint(0.01f * (lane + q_ + bb)); r1[q_] = r0[q_] ^ 1u; }
#else
          tmem_ld_16x256b<CB>(tm + PO + bb * BW, r0);
          tmem_ld_16x256b<CB>(tm + PO + (16u << 16) + bb * BW, r1);
          tmem_wait_ld_dep(r0);
          tmem_wait_ld_dep(r1);
#endif
          if (SAND_DEFER_PUB == 1 && decltype(pass_c)::value == 0 && bb == 0) flush_pend();
#pragma unroll
          for (int i = 0; i < CB; ++i) {
            uint32_t pk[4];
            chunk(r0 + 4 * i, r1 + 4 * i, PO + bb * BW + 8 * i, pk);
            if (ST && (SAND_SPLIT_STORE || store)) {
              if (decltype(pass_c)::value == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) stash[bb * CB + i][k] = pk[k];
              } else {
                st_chunk(PO + bb * BW + 8 * i, pk);
              }
            }
          }
        }
      };
      using P0 = std::integral_constant<int, 0>;
      using P1 = std::integral_constant<int, 1>;
      if (!(SAND_DIAG && p.prof >= 2)) {   // diagnostic 2/3 (SAND_DIAG builds): no epilogue math
        if (SAND_SPLIT_STORE && store) {
          math(std::true_type{}, P0{});
          if (SAND_DEFER_PUB == 2) flush_pend();
          math(std::true_type{}, P1{});
        } else {
          math(std::false_type{}, P0{});
          if (SAND_DEFER_PUB == 2) flush_pend();
          math(std::false_type{}, P1{});
        }
      } else {
        mbar_wait(b_accfull + 16 * s, e.pe);
        mbar_wait(b_accfull + 16 * s + 8, e.pe);
        tc_fence_after();
        if (SAND_EARLY_LO) publish_half(s, false, 0);
      }
      e.pe ^= 1u;
      if (prod) {
        // Eq. 3: t_l = (a_l0 . h + c_l0)(a_l1 . h + c_l1) needs both full dot products of the row:
        // sum over the quad (4 column pairs), then over the 4 column quarters through shared memory
        float2* rb2 = red2 + ((s * 2 + e.kpar) * NGRP) * 128;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float s0 = quad_sum(yv[k].x + yv[k].y), s1 = quad_sum(yv1[k].x + yv1[k].y);
          if (tq == 0) rb2[cq * 128 + 32 * q + quad + 8 * k] = make_float2(s0, s1);
        }
        named_bar_sync(bar_q, 32 * NGRP);
        if (cq == 0) {
          const int rowl = 32 * q + lane;
          float s0 = tc0[l - 1], s1 = tc1[l - 1];
#pragma unroll
          for (int k = 0; k < NGRP; ++k) { const float2 v = rb2[k * 128 + rowl]; s0 += v.x; s1 += v.y; }
          e.yprod += s0 * s1;
        }
        e.kpar ^= 1u;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) e.ylin[k] += yv[k].x + yv[k].y;
      }
      const long long cp_ = (SAND_DIAG && p.prof) ? clock64() : 0;
      flush_pend();   // (already done inside math when deferral is on; a no-op then)
      if (SAND_DEFER_PUB && defer_ok) { pend = s; pend_store = store; }
      else publish(s, store);
      if (SAND_DIAG && p.prof) ep_pub += clock64() - cp_;
      const long long ct_ = (SAND_DIAG && p.prof) ? clock64() : 0;
      if (l == d) {
        // tile end: every row reduced over its quad (shuffles); each warp hands its column quarter's
        // partials to the IO warp (which adds the 4 quarters and the tail-bias prefix sum).  No barrier
        // among the epilogue warps; part[s] is reused once the IO warp has read it (part_free).
        mbar_wait(b_partfree + 8 * s, (uint32_t)((e.w.ti & 1) ^ 1));
        float* pq = part + s * NPL * 128;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float v = quad_sum(e.ylin[k]);
          if (tq == 0) pq[cq * 128 + 32 * q + quad + 8 * k] = v;
          e.ylin[k] = 0.f;
        }
        if (TAIL == SAND_TAIL_MULT && cq == 0) pq[NGRP * 128 + 32 * q + lane] = e.yprod;
        e.yprod = 0.f;
        __syncwarp();
        if (lane == 0) mbar_arrive(b_iodone + 8 * s);
      }
      if (SAND_DIAG && p.prof) ep_tend += clock64() - ct_;
      e.w.advance(tstride, T, s_tile_end, L);
      if (SAND_DIAG && p.prof) { ep_wait += wt; ep_busy += clock64() - c0_ - wt; ep_steps += 1; }
    };

    EpiSlot e0, e1;
    e0.w.start(pair, T, s_tile_end, L);
    e1.w.start(pair + npairs, T, s_tile_end, L);
    e0.pe = e1.pe = 0; e0.kpar = e1.kpar = 0;
    e0.yprod = e1.yprod = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) e0.ylin[k] = e1.ylin[k] = 0.f;
    const long long t_start = (SAND_DIAG && p.prof) ? clock64() : 0;
#pragma unroll 1
    while (!(e0.w.done && e1.w.done)) {
      // a step may defer its publish into the other slot's next step only if that step exists
      if (!e0.w.done) step(e0, 0, !e1.w.done);
      if (!e1.w.done) {
        bool nxt0 = !e0.w.done;
        step(e1, 1, nxt0);
      }
    }
    flush_pend();
    if (SAND_DIAG && p.prof && warp == 3 && lane == 0) {
      g_kprof[blockIdx.x][6] = ep_wait;
      g_kprof[blockIdx.x][7] = ep_busy;
      g_kprof[blockIdx.x][8] = clock64() - t_start;
      g_kprof[blockIdx.x][9] = ep_steps;
      g_kprof[blockIdx.x][12] = ep_pub;
      g_kprof[blockIdx.x][13] = ep_tend;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_cg2(tmem_base, C::TMEM_COLS);
}

// ------------------------------------------------------------------------------------ host side
template <int H>
static size_t smem_for2(long long pt_floats, int L, int tail, int nst) {
  using C = Tc2Shape<H>;
  const size_t tab_bytes = (size_t)((pt_floats + 3) & ~3ll) * 4;
  const size_t io_bytes = (size_t)C::NSLOT * (tail == SAND_TAIL_MULT ? C::NGRP + 1 : C::NGRP) * 128 * 4;
  const size_t red_bytes = tail == SAND_TAIL_MULT ? (size_t)C::NSLOT * 2 * C::NGRP * 128 * 8 : 0;
  return (size_t)C::NSLOT * C::A_BYTES + (size_t)nst * C::STAGE + C::ONES_BYTES + C::W1_BYTES + (size_t)C::NSLOT * C::A1_BYTES +
         tab_bytes + io_bytes + red_bytes + 4 * (size_t)(L + 2) * sizeof(long long) + (3 * nst + 9 * C::NSLOT) * 8 +
         16;
}

static constexpr size_t kSmemMax2 = 232448;

template <int H>
static int pick_nst2(long long pt_floats, int L, int tail) {
  int best = 0;
  for (int nst = 1; nst <= 8; ++nst)
    if (smem_for2<H>(pt_floats, L, tail, nst) <= kSmemMax2) best = nst;
  return best;
}

bool tc2_available(int H) { return H == 64 || H == 128 || H == 256; }

void tc2_table_layout(int L, int H, int tail, MlpDev* m, bool interleave) {
  auto al4 = [](long long v) { return (v + 3) & ~3ll; };
  m->pt_off_l1 = 0;
  m->pt_off_bias = 0;
  // interleaved (wide kernel): [L][H/2][4] = (bias_c, bias_c+1, a_c, a_c+1) per column pair, one 16-byte
  // shared load per 8-column chunk; folded (this kernel: bias in the MMA): a [L][H] only
  m->pt_off_a = interleave ? m->pt_off_bias + 2 : 0;
  m->pt_off_a1 = interleave ? al4(m->pt_off_bias + 2ll * L * H) : al4(m->pt_off_a + (long long)L * H);
  m->pt_off_c = al4(m->pt_off_a1 + (tail == SAND_TAIL_MULT ? (long long)(L - 1) * H : 0));
  m->pt_off_c1 = al4(m->pt_off_c + L);
  m->pt_off_csum = al4(m->pt_off_c1 + L);
  m->pt_floats = al4(m->pt_off_csum + L + 1);
}

bool tc2_usable(int L, int H, int tail) {
  if (!tc2_available(H)) return false;
  MlpDev m{};
  tc2_table_layout(L, H, tail, &m, false);
  switch (H) {
    case 64: return pick_nst2<64>(m.pt_floats, L, tail) > 0;
    case 128: return pick_nst2<128>(m.pt_floats, L, tail) > 0;
    case 256: return pick_nst2<256>(m.pt_floats, L, tail) > 0;
    default: return false;
  }
}

// Feature n of a layer's output (= accumulator column n, = K index n of the next layer) is produced by pass
// n / (H/2); within a pass cta_group::2 takes the first H/4 B rows from the even CTA and the next H/4 from the
// odd one.  So CTA r holds, per pass j, rows (features) j H/2 + r H/4 + [0, H/4).
static inline void tc2_row_owner(int H, int n, int* cta, int* pass, int* row) {
  const int HN = H / 2, QR = H / 4;
  *pass = n / HN;
  *cta = (n % HN) / QR;
  *row = n % QR;
}

size_t tc2_w1_offset(int H, int n, int k) {
  // layer-1 B image: [2 CTAs][pass 0 rows | pass 1 rows (H/4 each)][16 bf16] in the core-matrix layout of l1_off
  int cta, pass, row;
  tc2_row_owner(H, n, &cta, &pass, &row);
  return (size_t)cta * (H / 2) * 32 + l1_off((uint32_t)(pass * (H / 4) + row), (uint32_t)k);
}

static inline uint16_t bf16_rne_h(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)((u >> 16) | ((u & 0xFFFF) ? 0x40 : 0));  // inf/nan
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
// (hi, lo) bf16 split of v: hi = rne(v), lo = rne(v - hi) (v - hi is exact in float32)
static inline void bf16_split(float v, uint16_t* hi, uint16_t* lo) {
  *hi = bf16_rne_h(v);
  uint32_t u = (uint32_t)*hi << 16;
  float h;
  std::memcpy(&h, &u, 4);
  *lo = bf16_rne_h(v - h);
}

void tc2_build_host(int L, int H, int tail, float w0, const float* const* W, const float* const* b,
                    const float* const* a, const float* const* a1, const float* c, const float* c1, MlpDev* m,
                    std::vector<float>* tables, std::vector<uint16_t>* w1img, std::vector<uint8_t>* img) {
  tc2_table_layout(L, H, tail, m, false);
  std::vector<float>& pt = *tables;
  pt.assign((size_t)m->pt_floats, 0.f);
  for (int i = 0; i < L; ++i) {
    std::memcpy(&pt[m->pt_off_a + (size_t)i * H], a[i], sizeof(float) * H);
    pt[m->pt_off_c + i] = c[i];
    pt[m->pt_off_c1 + i] = c1[i];
  }
  if (tail == SAND_TAIL_MULT)
    for (int i = 1; i < L; ++i) std::memcpy(&pt[m->pt_off_a1 + (size_t)(i - 1) * H], a1[i], sizeof(float) * H);
  double cs = 0.0;
  pt[m->pt_off_csum] = 0.f;
  for (int d = 1; d <= L; ++d) {
    cs += (tail == SAND_TAIL_LINEAR || d == 1) ? c[d - 1] : 0.0;
    pt[m->pt_off_csum + d] = (float)cs;
  }
  // layer-1 split-BF16 B operand of w0 W_1, w0 b_1: row n = (W_hi x y z | W_lo x y z | W_hi x y z | b_hi b_lo | 0),
  // matching the IO warp's A row (x_hi | x_hi | x_lo | 1 1 | 0): x_hi W_hi + x_hi W_lo + x_lo W_hi + b
  w1img->assign((size_t)H * 16, 0);
  auto put = [&](int n, int k, uint16_t v) { (*w1img)[tc2_w1_offset(H, n, k) / 2] = v; };
  for (int n = 0; n < H; ++n) {
    for (int k = 0; k < 3; ++k) {
      uint16_t hi, lo;
      bf16_split(w0 * W[0][3 * n + k], &hi, &lo);
      put(n, k, hi);
      put(n, 3 + k, lo);
      put(n, 6 + k, hi);
    }
    uint16_t bhi, blo;
    bf16_split(w0 * b[0][n], &bhi, &blo);
    put(n, 9, bhi);
    put(n, 10, blo);
  }
  // hidden layers: per (layer, CTA, pass) one ring stage: [bias operand: H/4 rows x 16 bf16 with (b_hi, b_lo)
  // at k = BIAS_K, l1_off layout, padded to >= 1 KB][KC K-chunks of w0 W_l: H/4 rows x 128 B, SW128 K-major:
  // element (row, k) of chunk kc at (row/8)*1024 + (row%8)*128 + ((((k%64)/8) ^ (row%8)) * 16) + (k%8)*2]
  const int KC = H / 64, QR = H / 4;
  const size_t small = QR * 32 < 1024 ? 1024 : (size_t)QR * 32, chunk = (size_t)QR * 128, stage = small + KC * chunk;
  const int bias_k = Tc2Shape<64>::BIAS_K;
  img->assign(L >= 2 ? (size_t)(L - 1) * 4 * stage : 0, 0);
  for (int i = 1; i < L; ++i)
    for (int n = 0; n < H; ++n) {
      int cta, pass, row;
      tc2_row_owner(H, n, &cta, &pass, &row);
      uint8_t* base = img->data() + (((size_t)(i - 1) * 2 + cta) * 2 + pass) * stage;
      uint16_t bhi, blo;
      bf16_split(w0 * b[i][n], &bhi, &blo);
      std::memcpy(base + l1_off((uint32_t)row, (uint32_t)bias_k), &bhi, 2);
      std::memcpy(base + l1_off((uint32_t)row, (uint32_t)bias_k + 1), &blo, 2);
      for (int k = 0; k < H; ++k) {
        const int kc = k / 64, kk = k % 64;
        const size_t byte = small + kc * chunk + (size_t)(row / 8) * 1024 + (row % 8) * 128 +
                            (size_t)(((kk / 8) ^ (row % 8)) * 16) + (kk % 8) * 2;
        const uint16_t v = bf16_rne_h(w0 * W[i][(size_t)n * H + k]);
        std::memcpy(base + byte, &v, 2);
      }
    }
}

template <int H, int TAIL>
static cudaError_t launch_tc2_t(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                                float* out, int num_sms, cudaStream_t st) {
  const int nst = pick_nst2<H>(m.pt_floats, m.L, TAIL);
  if (!nst) return cudaErrorInvalidConfiguration;
  const size_t sm = smem_for2<H>(m.pt_floats, m.L, TAIL, nst);
  const int prof = m.kprof;
  Tc2Params p{m, pts, perm, meta, out, nst, prof};
  const int grid = num_sms & ~1;
  k_tmlp_tc2<H, TAIL><<<grid, Tc2Shape<H>::THREADS, sm, st>>>(p);
  cudaError_t e = cudaGetLastError();
#ifdef SAND_HANG_DEBUG
  {
    unsigned long long hh[4];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(hh, g_hang, sizeof hh);
    if (hh[0]) {
      const unsigned bar = (unsigned)(hh[2] >> 32);
      fprintf(stderr, "[hang] block %llu thread %llu (warp %llu) barrier smem 0x%x parity %llu\n", hh[1] >> 32,
              hh[1] & 0xFFFFFFFF, (hh[1] & 0xFFFFFFFF) / 32, bar, hh[2] & 1);
      unsigned long long z[4] = {0, 0, 0, 0};
      cudaMemcpyToSymbol(g_hang, z, sizeof z);
    }
  }
#endif
  if (SAND_DIAG && prof && e == cudaSuccess) {
    // diagnostic only (SAND_OPT_KPROF): synchronous dump of the per-role counters (CTA averages; MMA over leaders)
    static unsigned long long h[160][kProfSlots];
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(h, g_kprof, sizeof h);
    if (e == cudaSuccess) {
      double a[kProfSlots] = {0};
      for (int b = 0; b < grid; ++b)
        for (int k = 0; k < kProfSlots; ++k) a[k] += (double)h[b][k] / (k < 4 ? grid / 2 : grid);
      fprintf(stderr,
              "[kprof] nst %d | MMA: total %.0f wait_A %.0f wait_W %.0f jobs %.0f | producer: wait_empty %.0f "
              "loads %.0f | epilogue(w4): total %.0f wait_acc %.0f busy %.0f steps %.0f publish %.0f tile_end %.0f | IO: wait %.0f busy %.0f\n",
              nst, a[2], a[0], a[1], a[3], a[4], a[5], a[8], a[6], a[7], a[9], a[12], a[13], a[10], a[11]);
    }
  }
  return e;
}

template <int H, int TAIL>
static cudaError_t prep_tc2_t() {
  return cudaFuncSetAttribute(k_tmlp_tc2<H, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax2);
}

#define SAND_TC2_DISPATCH(FN, ...)                                                                    \
  do {                                                                                                \
    const bool mult = m_tail == SAND_TAIL_MULT;                                                       \
    switch (m_H) {                                                                                    \
      case 64: return mult ? FN<64, 1>(__VA_ARGS__) : FN<64, 0>(__VA_ARGS__);                         \
      case 128: return mult ? FN<128, 1>(__VA_ARGS__) : FN<128, 0>(__VA_ARGS__);                      \
      case 256: return mult ? FN<256, 1>(__VA_ARGS__) : FN<256, 0>(__VA_ARGS__);                      \
      default: return cudaErrorInvalidValue;                                                          \
    }                                                                                                 \
  } while (0)

cudaError_t launch_tmlp_tc2(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                            float* out, int num_sms, cudaStream_t st) {
  const int m_H = m.H, m_tail = m.tail;
  SAND_TC2_DISPATCH(launch_tc2_t, m, pts, perm, meta, out, num_sms, st);
}

cudaError_t prepare_tc2(int H, int tail) {
  const int m_H = H, m_tail = tail;
  SAND_TC2_DISPATCH(prep_tc2_t);
}

}  // namespace sand
