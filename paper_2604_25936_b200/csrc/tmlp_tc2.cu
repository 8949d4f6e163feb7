// tmlp_tc2.cu -- CTA-pair (cta_group::2) persistent fused T-MLP kernel (SAND_BF16, H in {64, 128, 256}).
//
// Computes, per binned 256-row tile of uniform exit depth d (Sec. 3.4):
//   layer 1   : h_1 = sin(w0 (W_1 x + b_1))   FP32 SIMT (K = 3, R20), t_1 = a_1 . h_1 + c_1
//   layer 2..d: Z = H_{l-1} W_l^T on tcgen05 (M = 256 over the CTA pair, N = H, BF16 in, FP32 in TMEM),
//               epilogue h_l = sin(w0 Z + w0 b_l), t_l (Eq. 2 linear or Eq. 3 product), bf16(h_l) -> A
//   output    : sdf[perm[row]] = y_d = sum_{l <= d} t_l (Eq. 2).
//
// Organisation (per CTA of the pair; "leader" = even CTA):
//   warp 0       weight producer: this CTA's half (H/2 rows) of every 64-wide K-chunk of W_l, bulk async
//                copy (TMA engine) into an NST-stage ring (w_full / w_empty mbarriers)
//   warp 1       leader: tcgen05.mma.cta_group::2 issuer; odd CTA: relays "my half landed" (w_peer)
//   warp 2       TMEM allocator (2 accumulator slots x H columns)
//   warps 4..19  16 epilogue warps = 4 TMEM lane quadrants x 4 column quarters.  ALL of them work on
//                one tile slot at a time, alternating slot 0 / slot 1 step by step, so the MMA of one slot
//                overlaps the epilogue of the other (ping-pong) and 4 warps per SM sub-partition hide the
//                epilogue's latencies.  A step = one layer of one slot.
// Every role walks the same deterministic step sequence (rounds: slot 0 then slot 1, a slot's steps are
// its tiles' layers 1..d); the MMA and producer skip layer-1 steps.  Because the MMA order is the
// epilogue order restricted to MMA steps, the ping-pong cannot deadlock.
//
// Sine split: of every 16 accumulator columns, the first NP go through an odd
// degree-7 polynomial on the FMA pipe (range reduction to [-pi/2, pi/2] by a magic-number round), the
// rest through MUFU.SIN, so MUFU and FMA pipes share the transcendental load.  The per-column bias /
// layer-1 tables are pre-scaled on the host for the path their column takes (w0 or w0/pi).
//
// Tails: LINEAR tails sum linearly over layers, so every thread keeps a running partial over its columns
// and the four column quarters of a row are reduced once per tile through SMEM; the tail biases enter as
// a prefix sum csum[d].  MULT (Eq. 3) products need both full dot products per layer: reduced per step.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "sand_internal.h"

namespace sand {

template <int H>
struct Tc2Shape {
  static constexpr int KC = H / 64;                // 64-wide K chunks (128-byte swizzle atoms)
  static constexpr int A_CHUNK = 128 * 128;        // one K-chunk of this CTA's 128 rows (bytes)
  static constexpr int A_BYTES = KC * A_CHUNK;
  static constexpr int W_CHUNK = H * 128;          // full K-chunk of W (both halves) in the image
  static constexpr int WH_CHUNK = (H / 2) * 128;   // this CTA's half (N/2 rows)
  static constexpr int NSLOT = 2;
  static constexpr int HQ = H / 4;                 // columns per epilogue thread (column quarter)
  static constexpr int NG = HQ / 16;               // 16-column TMEM load groups per thread
  static constexpr int TMEM_COLS = 2 * H <= 128 ? 128 : (2 * H <= 256 ? 256 : 512);
  static constexpr int THREADS = 128 + 512;
  static constexpr int TILE = 256;
  static_assert(H % 64 == 0 && H <= 256 && HQ % 16 == 0, "CTA-pair kernel: H in {64, 128, 192, 256}");
};

struct Tc2Params {
  MlpDev m;
  const float* pts;
  const uint32_t* perm;
  const QueryMeta* meta;
  float* out;
  int nst;
  int prof;   // diagnostic (env SAND_KPROF=1): per-role clock64 wait/busy counters -> g_kprof
};

// Diagnostic counters (only written when Tc2Params::prof != 0), per CTA:
//  0 MMA wait a_full  1 MMA wait weights  2 MMA loop total  3 MMA jobs  4 producer wait w_empty  5 loads
//  6 epi wait acc_full  7 epi layer-1 steps  8 epi hidden steps (excl. wait)  9 epi tile-end barrier
//  10 epi loop total  11 epi steps
constexpr int kProfSlots = 16;
__device__ unsigned long long g_kprof[160][kProfSlots];

// ------------------------------------------------------------------------------ step sequence
__device__ __forceinline__ int tile_depth2(long long t, const long long* te, int L) {
  for (int d = L; d >= 1; --d)
    if (t < te[d]) return d;
  return 0;
}

// Per-slot walk over this pair's tiles: tile i of slot s is unit + nunits * (2 i + s); each tile yields
// steps l = 1..d.  `next` advances one step; the caller interleaves slot 0 and slot 1 round by round.
struct SlotWalk {
  long long t;
  int d, l;
  bool done;
  __device__ __forceinline__ void set(long long t_, long long T, const long long* te, int L) {
    t = t_;
    done = t >= T;
    l = 1;
    d = done ? 0 : tile_depth2(t, te, L);
  }
};

// ------------------------------------------------------------------------------ sine paths
// Polynomial path: u = z / pi (pre-scaled), k = rint(u) by the 1.5 * 2^23 magic add, r = u - k in
// [-1/2, 1/2], sin(z) = (-1)^k sin(pi r), sin(pi r) = r (C1 + C3 r^2 + C5 r^4 + C7 r^6)
// (near-minimax on [-1/2, 1/2]; |error| < 8e-7 in FP32, below MUFU.SIN's).
__device__ __forceinline__ float2 sin_poly2(float2 u) {
  const float2 M = make_float2(12582912.0f, 12582912.0f);
  const float2 t = __fadd2_rn(u, M);
  const float2 k = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  float2 r = __ffma2_rn(k, make_float2(-1.0f, -1.0f), u);
  // odd k -> negate r (sin is odd): sign bit from the parity bit of t's mantissa
  uint32_t sx, sy;
  asm("shf.l.wrap.b32 %0, %1, %1, 31;" : "=r"(sx) : "r"(__float_as_uint(t.x)));
  asm("shf.l.wrap.b32 %0, %1, %1, 31;" : "=r"(sy) : "r"(__float_as_uint(t.y)));
  r.x = __uint_as_float(__float_as_uint(r.x) ^ (sx & 0x80000000u));
  r.y = __uint_as_float(__float_as_uint(r.y) ^ (sy & 0x80000000u));
  const float2 r2 = __fmul2_rn(r, r);
  float2 p = __ffma2_rn(r2, make_float2(-0.5546384453773499f, -0.5546384453773499f),
                        make_float2(2.5418999195098877f, 2.5418999195098877f));
  p = __ffma2_rn(p, r2, make_float2(-5.167142868041992f, -5.167142868041992f));
  p = __ffma2_rn(p, r2, make_float2(3.1415820121765137f, 3.1415820121765137f));
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
  float ylin;         // this thread's running partial of the linear tail terms
  float yprod;        // MULT: sum of the Eq. 3 products (column-quarter 0 only)
  int ti;             // tiles of this slot started so far (IO buffer = ti & 1, phase = (ti >> 1) & 1)
};

template <int H, int TAIL, int NP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Tc2Shape<H>::THREADS, 1)
    k_tmlp_tc2(const Tc2Params p) {
  using C = Tc2Shape<H>;
  constexpr int NSLOT = C::NSLOT;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int nst = p.nst;
  const int L = p.m.L;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // ---- shared memory carve-up (identical offsets in both CTAs: the pair MMA relies on it)
  const uint32_t sA = base;
  const uint32_t sW = sA + NSLOT * C::A_BYTES;
  float* tab = reinterpret_cast<float*>(gbase + (NSLOT * C::A_BYTES + nst * C::WH_CHUNK));
  const long long ntab = p.m.pt_floats;
  // IO staging, double-buffered per slot: io_in[slot][buf][row] = (x, y, z, perm row or ~0u if padding),
  // io_part[slot][buf][cq][row] = the column quarters' partial outputs of the tile
  float4* io_in = reinterpret_cast<float4*>(tab + ((ntab + 3) & ~3ll));
  float* io_part = reinterpret_cast<float*>(io_in + NSLOT * 2 * 128);
  float2* red2 = reinterpret_cast<float2*>(io_part + NSLOT * 2 * 4 * 128);   // MULT: [slot][kpar][cq][128]
  const int red2_floats = (TAIL == SAND_TAIL_MULT) ? NSLOT * 2 * 4 * 128 * 2 : 0;
  long long* meta_s = reinterpret_cast<long long*>(io_part + NSLOT * 2 * 4 * 128 + red2_floats);
  long long* s_tile_end = meta_s;
  long long* s_tile_begin = meta_s + kMaxBins;
  long long* s_start = meta_s + 2 * kMaxBins;
  long long* s_count = meta_s + 3 * kMaxBins;
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta_s + 4 * kMaxBins);
  const uint32_t b_wfull = smem_u32(bars);
  const uint32_t b_wempty = b_wfull + 8 * nst;
  const uint32_t b_wpeer = b_wempty + 8 * nst;
  const uint32_t b_afull = b_wpeer + 8 * nst;
  const uint32_t b_accfull = b_afull + 8 * NSLOT;
  const uint32_t b_iofull = b_accfull + 8 * NSLOT;     // [slot][buf]
  const uint32_t b_iodone = b_iofull + 8 * NSLOT * 2;  // [slot][buf]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * nst + 2 * NSLOT + 4 * NSLOT);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const float4* src = reinterpret_cast<const float4*>(p.m.pair_tables);
    float4* dst = reinterpret_cast<float4*>(tab);
    for (long long i = tid; i < (ntab + 3) / 4; i += blockDim.x) dst[i] = src[i];
    if (tid < kMaxBins) {
      s_tile_end[tid] = p.meta->tile_end[tid];
      s_tile_begin[tid] = p.meta->tile_begin[tid];
      s_start[tid] = p.meta->start[tid];
      s_count[tid] = p.meta->count[tid];
    }
  }
  constexpr uint32_t kEpiWarps = 16;
  if (tid == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(b_wfull + 8 * i, 1);
      mbar_init(b_wempty + 8 * i, 1);
      mbar_init(b_wpeer + 8 * i, 1);
    }
    // a_full: one arrive per epilogue warp of both CTAs
    for (int s = 0; s < NSLOT; ++s) { mbar_init(b_afull + 8 * s, 2 * kEpiWarps); mbar_init(b_accfull + 8 * s, 1); }
    for (int i = 0; i < 2 * NSLOT; ++i) { mbar_init(b_iofull + 8 * i, 1); mbar_init(b_iodone + 8 * i, kEpiWarps); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_cg2(smem_u32(tmem_slot), C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();   // both CTAs' barriers initialised before any remote arrive / multicast commit
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const long long T = p.meta->total_tiles;
  const long long tstride = 2ll * npairs;

  if (warp == 0 || warp == 1) {
    if (lane == 0) {
      // producer / MMA issuer / relay: walk the MMA steps (l >= 2) in the epilogue's order, one job of
      // lookahead.  Weight reuse: consecutive jobs of the same layer (the two slots' tiles usually run in
      // phase) share one load of W_l when the ring holds whole layers (R = nst / KC >= 1 layer slots);
      // load event e uses layer slot e % R.  Otherwise (R == 0) chunks stream through the ring per job.
      SlotWalk w0, w1;
      w0.set(pair, T, s_tile_end, L);
      w1.set(pair + npairs, T, s_tile_end, L);
      int turn = 0;
      auto adv = [&](SlotWalk& w) {
        if (w.l == w.d) w.set(w.t + tstride, T, s_tile_end, L);
        else ++w.l;
      };
      // next MMA job (slot, layer) or false: rounds of slot 0 then slot 1, layer-1 steps skipped
      auto next_job = [&](int& s, int& l) -> bool {
#pragma unroll 1
        while (!(w0.done && w1.done)) {
          SlotWalk& w = turn ? w1 : w0;
          const int ts = turn;
          turn ^= 1;
          if (w.done) continue;
          const int wl = w.l;
          adv(w);
          if (wl >= 2) { s = ts; l = wl; return true; }
        }
        return false;
      };
      const int R = nst / C::KC;
      const uint8_t* img = reinterpret_cast<const uint8_t*>(p.m.w_image) + rank * C::WH_CHUNK;
      const uint32_t peer_wpeer = mapa_shared(b_wpeer, 0);
      constexpr uint32_t ID = idesc_bf16(256, H);
      uint32_t pa0 = 0, pa1 = 0;
      int st = 0;            // streaming mode ring position
      uint32_t ph = 0;
      long long ev = -1;     // reuse mode: load events so far - 1
      int cs = 0, cl = 0, ns = 0, nl = 0, prev_l = -1;
      unsigned long long pc[6] = {0, 0, 0, 0, 0, 0};
      const long long t_start = p.prof ? clock64() : 0;
      bool have = next_job(cs, cl);
#pragma unroll 1
      while (have) {
        const bool have_n = next_job(ns, nl);
        if (R >= 1) {
          const bool load = cl != prev_l;
          if (load) ++ev;
          const int ls = (int)(ev % R);
          const uint32_t lph = (uint32_t)((ev / R) & 1);
          const bool release = !have_n || nl != cl;
          const uint32_t sbase = (uint32_t)(ls * C::KC);
          if (warp == 0) {
            if (load) {
              const uint8_t* src = img + (size_t)(cl - 2) * C::KC * C::W_CHUNK;
              if (p.prof) pc[5] += 1;
              for (int kc = 0; kc < C::KC; ++kc) {
                const uint32_t sg = sbase + kc;
                const long long c0_ = p.prof ? clock64() : 0;
                mbar_wait(b_wempty + 8 * sg, lph ^ 1u);
                if (p.prof) pc[4] += clock64() - c0_;
                mbar_arrive_expect_tx(b_wfull + 8 * sg, C::WH_CHUNK);
                bulk_g2s(sW + sg * C::WH_CHUNK, src + (size_t)kc * C::W_CHUNK, C::WH_CHUNK, b_wfull + 8 * sg);
              }
            }
          } else if (rank == 0) {
            uint32_t& pa = cs ? pa1 : pa0;
            long long c0_ = p.prof ? clock64() : 0;
            mbar_wait_cluster(b_afull + 8 * cs, pa);
            if (p.prof) { const long long c1_ = clock64(); pc[0] += c1_ - c0_; pc[3] += 1; }
            pa ^= 1u;
            tc_fence_after();
            const uint32_t acc = tmem_base + (uint32_t)(cs * H);
            const uint32_t a_base = sA + cs * C::A_BYTES;
            for (int kc = 0; kc < C::KC; ++kc) {
              const uint32_t sg = sbase + kc;
              if (load) {
                c0_ = p.prof ? clock64() : 0;
                mbar_wait(b_wfull + 8 * sg, lph);
                mbar_wait_cluster(b_wpeer + 8 * sg, lph);
                if (p.prof) pc[1] += clock64() - c0_;
                tc_fence_after();
              }
              const uint32_t w_base = sW + sg * C::WH_CHUNK;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_cg2(acc, desc_sw128(a_base + kc * C::A_CHUNK + 32 * k), desc_sw128(w_base + 32 * k), ID,
                             (kc | k) ? 1u : 0u);
              if (release) mma_commit_cg2_mc(b_wempty + 8 * sg, 0x3);
            }
            mma_commit_cg2_mc(b_accfull + 8 * cs, 0x3);
          } else if (load) {
            for (int kc = 0; kc < C::KC; ++kc) {
              mbar_wait(b_wfull + 8 * (sbase + kc), lph);
              mbar_arrive_remote(peer_wpeer + 8 * (sbase + kc));
            }
          }
        } else {
          // streaming: every job pulls its KC chunks through the nst-stage ring
          if (warp == 0) {
            const uint8_t* src = img + (size_t)(cl - 2) * C::KC * C::W_CHUNK;
            for (int kc = 0; kc < C::KC; ++kc) {
              mbar_wait(b_wempty + 8 * st, ph ^ 1u);
              mbar_arrive_expect_tx(b_wfull + 8 * st, C::WH_CHUNK);
              bulk_g2s(sW + st * C::WH_CHUNK, src + (size_t)kc * C::W_CHUNK, C::WH_CHUNK, b_wfull + 8 * st);
              if (++st == nst) { st = 0; ph ^= 1u; }
            }
          } else if (rank == 0) {
            uint32_t& pa = cs ? pa1 : pa0;
            mbar_wait_cluster(b_afull + 8 * cs, pa);
            pa ^= 1u;
            tc_fence_after();
            const uint32_t acc = tmem_base + (uint32_t)(cs * H);
            const uint32_t a_base = sA + cs * C::A_BYTES;
            for (int kc = 0; kc < C::KC; ++kc) {
              mbar_wait(b_wfull + 8 * st, ph);
              mbar_wait_cluster(b_wpeer + 8 * st, ph);
              tc_fence_after();
              const uint32_t w_base = sW + st * C::WH_CHUNK;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_cg2(acc, desc_sw128(a_base + kc * C::A_CHUNK + 32 * k), desc_sw128(w_base + 32 * k), ID,
                             (kc | k) ? 1u : 0u);
              mma_commit_cg2_mc(b_wempty + 8 * st, 0x3);
              if (++st == nst) { st = 0; ph ^= 1u; }
            }
            mma_commit_cg2_mc(b_accfull + 8 * cs, 0x3);
          } else {
            for (int kc = 0; kc < C::KC; ++kc) {
              mbar_wait(b_wfull + 8 * st, ph);
              mbar_arrive_remote(peer_wpeer + 8 * st);
              if (++st == nst) { st = 0; ph ^= 1u; }
            }
          }
        }
        prev_l = cl;
        cs = ns; cl = nl; have = have_n;
      }
      if (p.prof) {
        pc[2] = clock64() - t_start;
        if (warp == 1 && rank == 0)
          for (int k = 0; k < 4; ++k) g_kprof[blockIdx.x][k] = pc[k];
        if (warp == 0)
          for (int k = 4; k < 6; ++k) g_kprof[blockIdx.x][k] = pc[k];
      }
    }
  } else if (warp == 3) {
    // =========================== IO warp: every global access of the tile rows
    // Gathers each tile's points (perm -> pts) into io_in two tiles ahead of their layer-1 step and writes
    // each finished tile's outputs (sum of the 4 column-quarter partials + csum[d]).  The epilogue warps
    // thus issue no global memory operations, so the proxy fence of their A-operand publish
    // (MEMBAR.CTA) never waits on DRAM.  Events follow the epilogue's step order (tile ends).
    const float* tcs = tab + p.m.pt_off_csum;
    auto tile_rows = [&](long long t, long long& r0, long long& rend) {
      const int d = tile_depth2(t, s_tile_end, L);
      r0 = s_start[d] + (t - s_tile_begin[d]) * C::TILE + (long long)rank * 128;
      rend = s_start[d] + s_count[d];
    };
    auto load_perm = [&](long long t, uint32_t (&ix)[4]) {
      long long r0, rend;
      tile_rows(t, r0, rend);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const long long r = r0 + lane + 32 * k;
        ix[k] = r < rend ? __ldg(p.perm + r) : 0xFFFFFFFFu;
      }
    };
    auto fill = [&](int s, int b, const uint32_t (&ix)[4]) {
      float4* dst = io_in + (s * 2 + b) * 128;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t i = ix[k] == 0xFFFFFFFFu ? 0u : ix[k];
        const float x = __ldg(p.pts + 3ull * i), y = __ldg(p.pts + 3ull * i + 1), z = __ldg(p.pts + 3ull * i + 2);
        dst[lane + 32 * k] = make_float4(x, y, z, __uint_as_float(ix[k]));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(b_iofull + 8 * (s * 2 + b));
    };
    SlotWalk w0, w1;
    w0.set(pair, T, s_tile_end, L);
    w1.set(pair + npairs, T, s_tile_end, L);
    uint32_t nx0[4], nx1[4];   // perm rows of the next tile to fill, per slot
    int ti0 = 0, ti1 = 0;      // tiles finished per slot
    for (int s = 0; s < NSLOT; ++s) {
      const long long t0 = pair + (long long)npairs * s;
      uint32_t ix[4];
      for (int i = 0; i < 2; ++i)
        if (t0 + i * tstride < T) { load_perm(t0 + i * tstride, ix); fill(s, i, ix); }
      uint32_t (&nx)[4] = s ? nx1 : nx0;
      if (t0 + 2 * tstride < T) load_perm(t0 + 2 * tstride, nx);
    }
    unsigned long long io_wait = 0, io_busy = 0;
    auto tile_end = [&](SlotWalk& w, int s, int& ti, uint32_t (&nx)[4]) {
      const int b = ti & 1;
      const long long c0_ = p.prof ? clock64() : 0;
      mbar_wait(b_iodone + 8 * (s * 2 + b), (uint32_t)((ti >> 1) & 1));
      const long long c1_ = p.prof ? clock64() : 0;
      const float cs = tcs[w.d];
      const float4* src = io_in + (s * 2 + b) * 128;
      const float* part = io_part + (s * 2 + b) * 4 * 128;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int row = lane + 32 * k;
        const uint32_t ix = __float_as_uint(src[row].w);
        const float y = cs + part[row] + part[128 + row] + part[256 + row] + part[384 + row];
        if (ix != 0xFFFFFFFFu) p.out[ix] = y;
      }
      __syncwarp();
      const long long t2 = w.t + 2 * tstride;
      if (t2 < T) {
        fill(s, b, nx);
        if (t2 + tstride < T) load_perm(t2 + tstride, nx);
      }
      ++ti;
      if (p.prof) { io_wait += c1_ - c0_; io_busy += clock64() - c1_; }
    };
#pragma unroll 1
    while (!(w0.done && w1.done)) {
      if (!w0.done) {
        if (w0.l == w0.d) { tile_end(w0, 0, ti0, nx0); w0.set(w0.t + tstride, T, s_tile_end, L); }
        else ++w0.l;
      }
      if (!w1.done) {
        if (w1.l == w1.d) { tile_end(w1, 1, ti1, nx1); w1.set(w1.t + tstride, T, s_tile_end, L); }
        else ++w1.l;
      }
    }
    if (p.prof && lane == 0) { g_kprof[blockIdx.x][12] = io_wait; g_kprof[blockIdx.x][13] = io_busy; }
  } else if (warp >= 4) {
    // =========================== epilogue (16 warps, both slots, step by step)
    const int ew = warp - 4;
    const int q = warp & 3;                  // TMEM lane quadrant = warp % 4
    const int cq = ew >> 2;                  // column quarter
    const int row = 32 * q + lane;           // TMEM lane / local A row
    const int c0 = cq * C::HQ;
    const uint32_t tm_row = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
    const uint32_t a_row = sA + (row >> 3) * 1024 + (row & 7) * 128;
    const uint32_t swz = row & 7;
    const float2 SM2 = make_float2(p.m.omega0, p.m.omega0);
    const float2 SP2 = make_float2(p.m.omega0 * 0.31830988618379067f, p.m.omega0 * 0.31830988618379067f);
    const float* t1 = tab + p.m.pt_off_l1;     // [H/2][8] layer-1 pair table
    const float* tb = tab + p.m.pt_off_bias;   // [L-1][H]
    const float* ta = tab + p.m.pt_off_a;      // [L][H]
    const float* ta1 = tab + p.m.pt_off_a1;    // [L-1][H] (MULT)
    const float* tc0 = tab + p.m.pt_off_c;     // [L]
    const float* tc1 = tab + p.m.pt_off_c1;    // [L] (MULT, index l-1)
    const uint32_t bar_q = 1 + q;              // per-quadrant named barrier (MULT reductions)
    const uint32_t afull_dst0 = rank == 0 ? b_afull : mapa_shared(b_afull, 0);
    unsigned long long ep[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};

    auto init_slot = [&](EpiSlot& e, long long t0) {
      e.w.set(t0, T, s_tile_end, L);
      e.pe = 0; e.kpar = 0; e.ylin = 0.f; e.yprod = 0.f; e.ti = 0;
    };
    auto publish = [&](int s) {
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(afull_dst0 + 8 * s);
        else mbar_arrive_remote(afull_dst0 + 8 * s);
      }
    };

    // one epilogue step of slot S
    auto step = [&](EpiSlot& e, const int s) {
      const int d = e.w.d, l = e.w.l;
      const long long step_t0 = p.prof ? clock64() : 0;
      long long hid_t0 = step_t0;
      const uint32_t aS = a_row + s * C::A_BYTES;
      float2 yv = make_float2(0.f, 0.f), yv1 = make_float2(0.f, 0.f);
      if (l == 1) {
        // ---------------- new tile: layer 1 (FP32 SIMT, K = 3) + tail 1
        const long long cw_ = p.prof ? clock64() : 0;
        mbar_wait(b_iofull + 8 * (s * 2 + (e.ti & 1)), (uint32_t)((e.ti >> 1) & 1));
        if (p.prof) ep[5] += clock64() - cw_;
        const float4 pt = io_in[(s * 2 + (e.ti & 1)) * 128 + row];
        const float2 X = make_float2(pt.x, pt.x), Y = make_float2(pt.y, pt.y), Z = make_float2(pt.z, pt.z);
        const bool store = d >= 2;
#pragma unroll
        for (int g = 0; g < C::NG; ++g) {
          uint32_t pk[8];
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) {
            const int j4 = c0 + 16 * g + 4 * qd;
            const float4 a4 = *reinterpret_cast<const float4*>(ta + j4);
#pragma unroll
            for (int hp = 0; hp < 2; ++hp) {
              const int pr = 2 * qd + hp;
              const int j = j4 + 2 * hp;
              const float4 wa = *reinterpret_cast<const float4*>(t1 + 4 * j);       // wx0 wx1 wy0 wy1
              const float4 wb = *reinterpret_cast<const float4*>(t1 + 4 * j + 4);   // wz0 wz1 b0 b1
              float2 z = __ffma2_rn(make_float2(wa.x, wa.y), X, make_float2(wb.z, wb.w));
              z = __ffma2_rn(make_float2(wa.z, wa.w), Y, z);
              z = __ffma2_rn(make_float2(wb.x, wb.y), Z, z);
              const float2 h = (2 * pr < NP) ? sin_poly2(z) : make_float2(__sinf(z.x), __sinf(z.y));
              yv = __ffma2_rn(hp ? make_float2(a4.z, a4.w) : make_float2(a4.x, a4.y), h, yv);
              pk[pr] = pack_bf16x2(h.x, h.y);
            }
          }
          if (store) {
            const uint32_t u = (uint32_t)(c0 / 8 + 2 * g);
            st_shared_v4(aS + (u >> 3) * C::A_CHUNK + (((u & 7u) ^ swz) << 4), pk[0], pk[1], pk[2], pk[3]);
            st_shared_v4(aS + ((u + 1) >> 3) * C::A_CHUNK + ((((u + 1) & 7u) ^ swz) << 4), pk[4], pk[5], pk[6],
                            pk[7]);
          }
        }
        e.ylin += yv.x + yv.y;
        if (store) publish(s);
      } else {
        // ---------------- hidden layer l: accumulator -> sin -> tail, bf16 h -> A (if l < d)
        long long c0_ = p.prof ? clock64() : 0;
        mbar_wait(b_accfull + 8 * s, e.pe);
        if (p.prof) { const long long c1_ = clock64(); ep[6] += c1_ - c0_; hid_t0 = c1_; }
        e.pe ^= 1u;
        tc_fence_after();
        const bool store = l != d;
        const float* bias = tb + (l - 2) * H;
        const float* a = ta + (l - 1) * H;
        const float* a1 = ta1 + (l - 2) * H;
        const uint32_t tm = tm_row + (uint32_t)(s * H);
        uint32_t ra[16], rb[16];
        tmem_ld16(tm, ra);
#pragma unroll
        for (int g = 0; g < C::NG; ++g) {
          uint32_t (&r)[16] = (g & 1) ? rb : ra;
          uint32_t (&rn)[16] = (g & 1) ? ra : rb;
          tmem_wait_ld_dep(r);
          if (g + 1 < C::NG) tmem_ld16(tm + 16 * (g + 1), rn);
          uint32_t pk[8];
#pragma unroll
          for (int qd = 0; qd < 4; ++qd) {
            const int j4 = c0 + 16 * g + 4 * qd;
            const float4 b4 = *reinterpret_cast<const float4*>(bias + j4);
            const float4 a4 = *reinterpret_cast<const float4*>(a + j4);
            float4 c4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (TAIL == SAND_TAIL_MULT) c4 = *reinterpret_cast<const float4*>(a1 + j4);
#pragma unroll
            for (int hp = 0; hp < 2; ++hp) {
              const int pr = 2 * qd + hp;
              const float2 b2 = hp ? make_float2(b4.z, b4.w) : make_float2(b4.x, b4.y);
              const float2 acc = make_float2(__uint_as_float(r[2 * pr]), __uint_as_float(r[2 * pr + 1]));
              float2 h;
              if (2 * pr < NP) {
                h = sin_poly2(__ffma2_rn(acc, SP2, b2));
              } else {
                const float2 z = __ffma2_rn(acc, SM2, b2);
                h = make_float2(__sinf(z.x), __sinf(z.y));
              }
              yv = __ffma2_rn(hp ? make_float2(a4.z, a4.w) : make_float2(a4.x, a4.y), h, yv);
              if (TAIL == SAND_TAIL_MULT)
                yv1 = __ffma2_rn(hp ? make_float2(c4.z, c4.w) : make_float2(c4.x, c4.y), h, yv1);
              pk[pr] = pack_bf16x2(h.x, h.y);
            }
          }
          if (store) {
            const uint32_t u = (uint32_t)(c0 / 8 + 2 * g);
            st_shared_v4(aS + (u >> 3) * C::A_CHUNK + (((u & 7u) ^ swz) << 4), pk[0], pk[1], pk[2], pk[3]);
            st_shared_v4(aS + ((u + 1) >> 3) * C::A_CHUNK + ((((u + 1) & 7u) ^ swz) << 4), pk[4], pk[5], pk[6],
                            pk[7]);
          }
        }
        if (store) publish(s);
        else tc_fence_before();
        if (TAIL == SAND_TAIL_MULT) {
          // Eq. 3: t_l = (a_l0 . h + c_l0)(a_l1 . h + c_l1) needs both full dot products of the row
          float2* rb2 = red2 + ((s * 2 + e.kpar) * 4) * 128;
          rb2[cq * 128 + row] = make_float2(yv.x + yv.y, yv1.x + yv1.y);
          named_bar_sync(bar_q, 128);
          if (cq == 0) {
            float s0 = tc0[l - 1], s1 = tc1[l - 1];
#pragma unroll
            for (int k = 0; k < 4; ++k) { const float2 v = rb2[k * 128 + row]; s0 += v.x; s1 += v.y; }
            e.yprod += s0 * s1;
          }
          e.kpar ^= 1u;
        } else {
          e.ylin += yv.x + yv.y;
        }
      }
      if (p.prof) {
        const long long c1_ = clock64();
        if (l == 1) ep[7] += c1_ - step_t0; else ep[8] += c1_ - hid_t0;
        ep[11] += 1;
      }
      if (l == d) {
        // ---------------- tile end: hand this thread's partial of y_d to the IO warp
        io_part[((s * 2 + (e.ti & 1)) * 4 + cq) * 128 + row] = e.ylin + e.yprod;
        __syncwarp();
        if (lane == 0) mbar_arrive(b_iodone + 8 * (s * 2 + (e.ti & 1)));
        ++e.ti;
        e.ylin = 0.f;
        e.yprod = 0.f;
        e.w.set(e.w.t + tstride, T, s_tile_end, L);
      } else {
        ++e.w.l;
      }
    };

    EpiSlot e0, e1;
    init_slot(e0, pair);
    init_slot(e1, pair + npairs);
    const long long t_start = p.prof ? clock64() : 0;
#pragma unroll 1
    while (!(e0.w.done && e1.w.done)) {
      if (!e0.w.done) step(e0, 0);
      if (!e1.w.done) step(e1, 1);
    }
    if (p.prof && warp == 4 && lane == 0) {
      ep[10] = clock64() - t_start;
      for (int k = 6; k < 12; ++k) g_kprof[blockIdx.x][k] = ep[k];
      g_kprof[blockIdx.x][14] = ep[5];
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_cg2(tmem_base, C::TMEM_COLS);
}

// ------------------------------------------------------------------------------------ host side
template <int H>
static size_t smem_for2(long long pt_floats, int tail, int nst) {
  using C = Tc2Shape<H>;
  const size_t tab_bytes = (size_t)((pt_floats + 3) & ~3ll) * 4;
  const size_t io_bytes = (size_t)C::NSLOT * 2 * 128 * 16 + (size_t)C::NSLOT * 2 * 4 * 128 * 4;
  const size_t red_bytes = tail == SAND_TAIL_MULT ? (size_t)C::NSLOT * 2 * 4 * 128 * 8 : 0;
  return 1024 + (size_t)C::NSLOT * C::A_BYTES + (size_t)nst * C::WH_CHUNK + tab_bytes + io_bytes + red_bytes +
         4 * kMaxBins * sizeof(long long) + (3 * nst + 6 * C::NSLOT) * 8 + 16;
}

static constexpr size_t kSmemMax2 = 232448;

template <int H>
static int pick_nst2(long long pt_floats, int tail) {
  int best = 0;
  for (int nst = 2; nst <= 8; ++nst)
    if (smem_for2<H>(pt_floats, tail, nst) <= kSmemMax2) best = nst;
  return best;
}

bool tc2_available(int H) { return H == 64 || H == 128 || H == 256; }

int tc2_npoly() {
  static int np = -1;
  if (np < 0) {
    np = kPairPolyDefault;
    if (const char* ev = getenv("SAND_NPOLY")) {
      const int v = atoi(ev);
      if (v == 0 || v == 4 || v == 6 || v == 8) np = v;
    }
  }
  return np;
}

template <int H, int TAIL, int NP>
static cudaError_t launch_tc2_t(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                                float* out, int num_sms, cudaStream_t st) {
  const int nst = pick_nst2<H>(m.pt_floats, TAIL);
  if (!nst) return cudaErrorInvalidConfiguration;
  const size_t sm = smem_for2<H>(m.pt_floats, TAIL, nst);
  static const int prof = getenv("SAND_KPROF") ? atoi(getenv("SAND_KPROF")) : 0;
  Tc2Params p{m, pts, perm, meta, out, nst, prof};
  const int grid = num_sms & ~1;
  k_tmlp_tc2<H, TAIL, NP><<<grid, Tc2Shape<H>::THREADS, sm, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (prof && e == cudaSuccess) {
    // diagnostic only: synchronous dump of the per-role counters
    unsigned long long h[160][kProfSlots];
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(h, g_kprof, sizeof h);
    if (e == cudaSuccess) {
      double a[kProfSlots] = {0};
      int nl = 0, nf = 0;
      for (int b = 0; b < grid; ++b) {
        for (int k = 4; k < 15; ++k) a[k] += (double)h[b][k];
        if ((b & 1) == 0) { for (int k = 0; k < 4; ++k) a[k] += (double)h[b][k]; ++nl; }
        ++nf;
      }
      for (int k = 0; k < 4; ++k) a[k] /= nl;
      for (int k = 4; k < 15; ++k) a[k] /= nf;
      fprintf(stderr,
              "[kprof] MMA: total %.0f wait_a %.0f wait_w %.0f jobs %.0f | prod: wait_empty %.0f loads %.0f | "
              "epi(w4): total %.0f wait_acc %.0f wait_io %.0f l1 %.0f hidden %.0f steps %.0f | io: wait %.0f busy %.0f"
              " | nst %d\n",
              a[2], a[0], a[1], a[3], a[4], a[5], a[10], a[6], a[14], a[7], a[8], a[11], a[12], a[13], nst);
    }
  }
  return e;
}

template <int H, int TAIL, int NP>
static cudaError_t prep_tc2_t() {
  return cudaFuncSetAttribute(k_tmlp_tc2<H, TAIL, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax2);
}

// The polynomial share is a template parameter; the bench configuration (H = 256, LINEAR) is built for
// every supported share (tuning), the others for the default share only.
#define SAND_TC2_DISPATCH(FN, ...)                                                                    \
  do {                                                                                                \
    const bool mult = m_tail == SAND_TAIL_MULT;                                                       \
    const int np = m_np;                                                                              \
    if (m_H == 256 && !mult) {                                                                        \
      switch (np) {                                                                                   \
        case 0: return FN<256, 0, 0>(__VA_ARGS__);                                                    \
        case 4: return FN<256, 0, 4>(__VA_ARGS__);                                                    \
        case 6: return FN<256, 0, 6>(__VA_ARGS__);                                                    \
        default: return FN<256, 0, 8>(__VA_ARGS__);                                                   \
      }                                                                                               \
    }                                                                                                 \
    if (np != kPairPolyDefault) return cudaErrorInvalidValue;                                          \
    switch (m_H) {                                                                                    \
      case 64: return mult ? FN<64, 1, kPairPolyDefault>(__VA_ARGS__) : FN<64, 0, kPairPolyDefault>(__VA_ARGS__); \
      case 128: return mult ? FN<128, 1, kPairPolyDefault>(__VA_ARGS__) : FN<128, 0, kPairPolyDefault>(__VA_ARGS__); \
      case 256: return FN<256, 1, kPairPolyDefault>(__VA_ARGS__);                                      \
      default: return cudaErrorInvalidValue;                                                          \
    }                                                                                                 \
  } while (0)

cudaError_t launch_tmlp_tc2(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                            float* out, int num_sms, cudaStream_t st) {
  const int m_H = m.H, m_tail = m.tail, m_np = m.pt_npoly;
  SAND_TC2_DISPATCH(launch_tc2_t, m, pts, perm, meta, out, num_sms, st);
}

cudaError_t prepare_tc2(int H, int tail) {
  const int m_H = H, m_tail = tail, m_np = tc2_npoly();
  SAND_TC2_DISPATCH(prep_tc2_t);
}

}  // namespace sand
