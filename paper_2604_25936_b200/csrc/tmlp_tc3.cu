// tmlp_tc3.cu -- CTA-pair fused T-MLP kernel for wide layers (SAND_BF16, H = 336; BASELINE configs[3]).
//
// Same computation as tmlp_tc2.cu (Eq. 2; adaptive depth Sec. 3.4) for
// a width whose FP32 accumulator (336 TMEM columns per 128 rows) leaves no room for a second tile slot.
// Instead of two tiles, ONE 256-row tile per pair is split into two N-halves that play the two slots:
//   half A = columns [0, 192) (exactly K-chunks 0..2 of the next layer), half B = [192, HP), with the
//   width padded to HP = 352 (zero weights / tables beyond 336, so padded h are sin(0) = 0).
// Step order (epilogue and MMA alike): per tile, for l = 1..d: (A, l), (B, l).
//   MMA job (A, l >= 2): D_A = H_{l-1} W_l[A]^T -- its K-chunks 0..2 need the epilogue of (A, l-1), its
//     K-chunks 3..5 the epilogue of (B, l-1); job (B, l) then has all of H_{l-1}.  So the first 57% of
//     job (A, l) runs under the epilogue of (B, l-1) and job (B, l) under the epilogue of (A, l).
//   Layer 1 per half: one K = 16 split-BF16 MMA (as tmlp_tc2.cu) on the IO warp's operand.
// Warp roles, TMEM loads (16x256b, 4 rows per thread), MUFU sine, stmatrix A stores, IO warp and the
// tile-end partial hand-off are those of tmlp_tc2.cu.  LINEAR tails only (MULT runs tmlp_tc.cu).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#include <type_traits>
#include <vector>

#include "ptx.cuh"

#ifndef SAND_DIAG
#define SAND_DIAG 0   // 1: diagnostic modes SAND_KPROF=2/3 (timing studies; build with SAND_BUILD_DEFS=-DSAND_DIAG=1)
#endif
#include "sand_internal.h"

namespace sand {

template <int H>
struct Tc3Shape {
  static constexpr int HP = (H + 31) / 32 * 32;     // padded width
  static constexpr int NA = 192;                    // half A = K-chunks 0..2
  static constexpr int NB = HP - NA;                // half B
  static constexpr int KC = (HP + 63) / 64;         // 64-wide K-chunks of the A operand (last may be partial)
  static constexpr int KSTEPS = HP / 16;            // K = 16 MMA steps per job
  static constexpr int A_CHUNK = 128 * 128;         // one K-chunk of this CTA's 128 rows (bytes)
  static constexpr int A_BYTES = KC * A_CHUNK;
  static constexpr int RA = NA / 2, RB = NB / 2;    // B rows per CTA of each half
  static constexpr int STAGE = 2 * RA * 128;        // two K-chunks of the larger half (ring slot bytes)
  static constexpr int NSJ = (KC + 1) / 2;          // ring stages per job
  static constexpr int W1_BYTES = (RA + RB) * 32;   // layer-1 B operand, this CTA's rows of both halves
  static constexpr int A1_BYTES = 128 * 32;
  static constexpr int THREADS = 96 + 512;
  static constexpr int TILE = 256;
  static_assert(NB > 0 && NB <= 256 && NB % 32 == 0 && H > 256, "wide kernel: 256 < H <= 448");
};

struct Tc3Params {
  MlpDev m;
  const float* pts;
  const uint32_t* perm;
  const QueryMeta* meta;
  float* out;
  int nst;
  int prof;   // diagnostic (env SAND_KPROF=1): clock64 wait counters per role -> g_kprof3
};

// Diagnostic counters per CTA (written only when prof != 0): 0 MMA wait a_full[A], 1 MMA wait a_full[B]
// (mid-job), 2 MMA wait weights, 3 MMA wait layer-1 (a_full + a1_full), 4 MMA loop total, 5 producer
// wait w_empty, 6 epi wait acc[A], 7 epi wait acc[B] (step B), 8 epi wait acc[B] (before A stores),
// 9 epi total, 10 epi steps, 11 IO wait, 12 epi wait part_free.
constexpr int kProf3 = 13;
__device__ unsigned long long g_kprof3[160][kProf3];
#define P3T() (p.prof ? clock64() : 0ll)

__device__ __forceinline__ int tile_depth3(long long t, const long long* te, int L) {
  for (int d = L; d >= 1; --d)
    if (t < te[d]) return d;
  return 0;
}

// Walk over this pair's tiles (t = pair + npairs * i) and their steps (A,1),(B,1),...,(A,d),(B,d).
struct WideWalk {
  long long t;
  int d, l, half, ti;
  bool done;
  __device__ __forceinline__ void set(long long t_, long long T, const long long* te, int L) {
    t = t_;
    done = t >= T;
    l = 1;
    half = 0;
    d = done ? 0 : tile_depth3(t, te, L);
  }
  __device__ __forceinline__ void advance(long long stride, long long T, const long long* te, int L) {
    if (half == 0) { half = 1; return; }
    half = 0;
    if (l == d) { ++ti; set(t + stride, T, te, L); }
    else ++l;
  }
};

__device__ __forceinline__ void st_shared_v4w(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ float2 sin_mufu2(float2 z) { return make_float2(__sinf(z.x), __sinf(z.y)); }

template <int H>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Tc3Shape<H>::THREADS, 1)
    k_tmlp_wide(const Tc3Params p) {
  using C = Tc3Shape<H>;
  constexpr int HP = C::HP;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = smem_u32(smem_raw);
  if (base & 1023u) __trap();
  uint8_t* gbase = smem_raw;
  const int nst = p.nst;
  const int L = p.m.L;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // ---- shared memory (identical offsets in both CTAs)
  const uint32_t sA = base;                          // one tile: KC x 16 KB, SW128 K-major
  const uint32_t sW = sA + C::A_BYTES;               // weight ring, nst x STAGE
  const uint32_t sW1 = sW + nst * C::STAGE;          // layer-1 B operand (both halves)
  const uint32_t sA1 = sW1 + C::W1_BYTES;            // layer-1 A operand
  float* tab = reinterpret_cast<float*>(gbase + ((sA1 + C::A1_BYTES) - base));
  const long long ntab = p.m.pt_floats;
  float* part = tab + ((ntab + 3) & ~3ll);           // [cq][128] tile-end partials
  const int nb = L + 2;
  long long* meta_s = reinterpret_cast<long long*>(part + 4 * 128);
  long long* s_tile_end = meta_s;
  long long* s_tile_begin = meta_s + nb;
  long long* s_start = meta_s + 2 * nb;
  long long* s_count = meta_s + 3 * nb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta_s + 4 * nb);
  const uint32_t b_wfull = smem_u32(bars);
  const uint32_t b_wempty = b_wfull + 8 * nst;
  const uint32_t b_wpeer = b_wempty + 8 * nst;
  const uint32_t b_afull = b_wpeer + 8 * nst;      // [half] epilogue step done (A written / acc read)
  const uint32_t b_accfull = b_afull + 16;         // [half]
  const uint32_t b_a1full = b_accfull + 16;        // layer-1 A written (leader: 2 arrivals)
  const uint32_t b_a1free = b_a1full + 8;          // layer-1 MMAs done with A1
  const uint32_t b_iodone = b_a1free + 8;          // all epilogue warps wrote their tile partials
  const uint32_t b_partfree = b_iodone + 8;        // IO warp read the partials
  const uint32_t b_bhead = b_partfree + 8;         // job (B, l >= 2) has read K-chunks 0..2 (A cols 0..191)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * nst + 10);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const float4* src = reinterpret_cast<const float4*>(p.m.pair_tables);
    float4* dst = reinterpret_cast<float4*>(tab);
    for (long long i = tid; i < (ntab + 3) / 4; i += blockDim.x) dst[i] = src[i];
    const uint4* w1s = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(p.m.w1_image) +
                                                      rank * C::W1_BYTES);
    uint4* w1d = reinterpret_cast<uint4*>(gbase + (sW1 - base));
    for (int i = tid; i < C::W1_BYTES / 16; i += blockDim.x) w1d[i] = w1s[i];
    if (tid < nb) {
      s_tile_end[tid] = p.meta->tile_end[tid];
      s_tile_begin[tid] = p.meta->tile_begin[tid];
      s_start[tid] = p.meta->start[tid];
      s_count[tid] = p.meta->count[tid];
    }
    fence_proxy_async_smem();
  }
  constexpr uint32_t kEpiWarps = 16;
  if (tid == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(b_wfull + 8 * i, 1);
      mbar_init(b_wempty + 8 * i, 1);
      mbar_init(b_wpeer + 8 * i, 1);
    }
    for (int s = 0; s < 2; ++s) { mbar_init(b_afull + 8 * s, 2 * kEpiWarps); mbar_init(b_accfull + 8 * s, 1); }
    mbar_init(b_a1full, 2);
    mbar_init(b_a1free, 1);
    mbar_init(b_iodone, kEpiWarps);
    mbar_init(b_partfree, 1);
    mbar_init(b_bhead, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_cg2(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const long long T = p.meta->total_tiles;
  const long long tstride = npairs;

  if (warp == 0 || warp == 1) {
    if (lane == 0) {
      // producer / MMA issuer / relay, one job per epilogue step
      WideWalk w;
      w.ti = 0;
      w.set(pair, T, s_tile_end, L);
      // wide image: [L-1][2 CTA ranks][half A: KC chunks x RA rows | half B: KC chunks x RB rows][128 B]
      const size_t layer_bytes = (size_t)2 * C::KC * (C::RA + C::RB) * 128;
      const uint8_t* img = reinterpret_cast<const uint8_t*>(p.m.w_image_pair) +
                           (size_t)rank * C::KC * (C::RA + C::RB) * 128;
      const uint32_t peer_wpeer = mapa_shared(b_wpeer, 0);
      constexpr uint32_t IDA = idesc_bf16(256, C::NA), IDB = idesc_bf16(256, C::NB);
      uint32_t paA = 0, paB = 0, pa1 = 0;
      int st = 0;
      uint32_t ph = 0;
      bool first_a = true, first_b = true;
      unsigned long long pc[kProf3] = {};
      const long long t_start = P3T();
#pragma unroll 1
      while (!w.done) {
        const int l = w.l, hf = w.half;
        const int rows = hf ? C::RB : C::RA;
        const uint32_t acc = tmem_base + (uint32_t)(hf ? C::NA : 0);
        const uint32_t ID = hf ? IDB : IDA;
        if (l == 1) {
          if (warp == 1 && rank == 0) {
            const long long t0_ = P3T();
            // acc of this half free: the epilogue finished the previous tile's last step of this half
            if (hf == 0) {
              if (!first_a) { mbar_wait_cluster(b_afull, paA); paA ^= 1u; }
              first_a = false;
              mbar_wait_cluster(b_a1full, pa1);
              pa1 ^= 1u;
            } else {
              if (!first_b) { mbar_wait_cluster(b_afull + 8, paB); paB ^= 1u; }
              first_b = false;
            }
            if (p.prof) pc[3] += clock64() - t0_;
            tc_fence_after();
            mma_bf16_cg2(acc, desc_nosw(sA1, 128, 256), desc_nosw(sW1 + (hf ? C::RA * 32 : 0), 128, 256), ID, 0u);
            if (hf) mma_commit_cg2_mc(b_a1free, 0x3);
            mma_commit_cg2_mc(b_accfull + 8 * hf, 0x3);
          }
        } else {
          const uint8_t* src = img + (size_t)(l - 2) * layer_bytes + (hf ? (size_t)C::KC * C::RA * 128 : 0);
          const uint32_t chunk = (uint32_t)rows * 128;
          if (warp == 0) {
            for (int j = 0; j < C::NSJ && !(SAND_DIAG && p.prof == 3); ++j) {
              const int nch = (2 * j + 1 < C::KC) ? 2 : 1;
              const long long t0_ = P3T();
              mbar_wait_lazy(b_wempty + 8 * st, ph ^ 1u);
              if (p.prof) pc[5] += clock64() - t0_;
              mbar_arrive_expect_tx(b_wfull + 8 * st, nch * chunk);
              bulk_g2s(sW + st * C::STAGE, src + (size_t)(2 * j) * chunk, nch * chunk, b_wfull + 8 * st);
              if (++st == nst) { st = 0; ph ^= 1u; }
            }
          } else if (rank == 0) {
            // job (A, l): K-chunks 0..2 need epilogue (A, l-1), K-chunks 3.. need (B, l-1)
            long long t0_ = P3T();
            if (hf == 0) { mbar_wait_cluster(b_afull, paA); paA ^= 1u; }
            if (p.prof) pc[0] += clock64() - t0_;
            tc_fence_after();
            // descriptors precomputed (the single issuing thread's scalar work per MMA would otherwise
            // exceed the tensor pipe's N/2 clk per instruction); K-step k of a chunk = +32 B = +2
            const uint64_t a_d0 = desc_sw128(sA);
            const uint32_t chunk16 = (uint32_t)rows * 8;   // chunk bytes >> 4
#pragma unroll
            for (int j = 0; j < C::NSJ; ++j) {
              t0_ = P3T();
              if (!(SAND_DIAG && p.prof == 3)) {   // diagnostic 3: no weight streaming (stale ring contents)
                mbar_wait(b_wfull + 8 * st, ph);
                mbar_wait_cluster(b_wpeer + 8 * st, ph);
              }
              if (p.prof) pc[2] += clock64() - t0_;
              tc_fence_after();
              const uint64_t w_d = desc_sw128(sW + st * C::STAGE);
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                const int kc = 2 * j + c;
                if (kc >= C::KC) break;
                if (hf == 0 && kc == 3) {
                  t0_ = P3T();
                  mbar_wait_cluster(b_afull + 8, paB);
                  if (p.prof) pc[1] += clock64() - t0_;
                  paB ^= 1u;
                  tc_fence_after();
                }
                const uint64_t wc = w_d + (uint64_t)(c * chunk16);
                const int nk = (kc * 64 + 64 <= HP) ? 4 : (HP - kc * 64) / 16;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  if (k < nk)
                    mma_bf16_cg2(acc, a_d0 + (uint64_t)(kc * (C::A_CHUNK >> 4) + 2 * k), wc + (uint64_t)(2 * k), ID,
                                 (kc | k) ? 1u : 0u);
                // half A of the operand may be overwritten (epilogue (A, l)) once job B is past it
                if (hf == 1 && kc == 2) mma_commit_cg2_mc(b_bhead, 0x3);
              }
              mma_commit_cg2_mc(b_wempty + 8 * st, 0x3);
              if (++st == nst) { st = 0; ph ^= 1u; }
            }
            mma_commit_cg2_mc(b_accfull + 8 * hf, 0x3);
          } else {
            for (int j = 0; j < C::NSJ && !(SAND_DIAG && p.prof == 3); ++j) {
              mbar_wait(b_wfull + 8 * st, ph);
              mbar_arrive_remote(peer_wpeer + 8 * st);
              if (++st == nst) { st = 0; ph ^= 1u; }
            }
          }
        }
        w.advance(tstride, T, s_tile_end, L);
      }
      if (p.prof) {
        pc[4] = clock64() - t_start;
        if (warp == 1) for (int k = 0; k < 5; ++k) g_kprof3[blockIdx.x][k] = pc[k];
        else g_kprof3[blockIdx.x][5] = pc[5];
      }
    }
  } else if (warp == 2) {
    // =========================== IO warp (one tile in flight per pair)
    const uint32_t a1full_dst = rank == 0 ? b_a1full : mapa_shared(b_a1full, 0);
    const float* tcs = tab + p.m.pt_off_csum;
    auto load_perm = [&](long long t, uint32_t (&ix)[4]) {
      const int d = tile_depth3(t, s_tile_end, L);
      const long long r0 = s_start[d] + (t - s_tile_begin[d]) * C::TILE + (long long)rank * 128;
      const long long rend = s_start[d] + s_count[d];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const long long r = r0 + lane + 32 * k;
        ix[k] = r < rend ? __ldg(p.perm + r) : 0xFFFFFFFFu;
      }
    };
    auto fill = [&](const uint32_t (&ix)[4]) {
      float x[4], y[4], z[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const size_t i = ix[k] == 0xFFFFFFFFu ? 0 : ix[k];
        x[k] = __ldg(p.pts + 3 * i); y[k] = __ldg(p.pts + 3 * i + 1); z[k] = __ldg(p.pts + 3 * i + 2);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int row = lane + 32 * k;
        const uint32_t hxy = pack_bf16x2(x[k], y[k]);
        const uint32_t hz1 = pack_bf16x2(z[k], 1.0f);
        const float xh = __uint_as_float(hxy << 16), yh = __uint_as_float(hxy & 0xFFFF0000u);
        const float zh = __uint_as_float(hz1 << 16);
        const uint32_t lxy = pack_bf16x2(x[k] - xh, y[k] - yh);
        const uint32_t lz1 = pack_bf16x2(z[k] - zh, 1.0f);
        st_shared_v4w(sA1 + l1_off((uint32_t)row, 0), hxy, (hz1 & 0xFFFFu) | (hxy << 16), (hxy >> 16) | (hz1 << 16), lxy);
        st_shared_v4w(sA1 + l1_off((uint32_t)row, 8), lz1, 0x3F80u, 0u, 0u);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(a1full_dst);
        else mbar_arrive_remote(a1full_dst);
      }
    };
    WideWalk w;
    w.ti = 0;
    w.set(pair, T, s_tile_end, L);
    uint32_t cur[4], nxt[4], pre[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) cur[k] = nxt[k] = pre[k] = 0xFFFFFFFFu;
    if (!w.done) { load_perm(w.t, cur); fill(cur); }
    if (w.t + tstride < T) load_perm(w.t + tstride, nxt);
    uint32_t pa1f = 0, piod = 0;
    unsigned long long io_wait = 0;
#pragma unroll 1
    while (!w.done) {
      if (w.l == 1 && w.half == 1) {
        // after this tile's layer-1 MMAs: refill A1 with the next tile
        const long long t1 = w.t + tstride;
        if (t1 < T) {
          mbar_wait_lazy(b_a1free, pa1f);
          pa1f ^= 1u;
          fill(nxt);
          if (t1 + tstride < T) load_perm(t1 + tstride, pre);
        } else {
          mbar_wait_lazy(b_a1free, pa1f);
          pa1f ^= 1u;
        }
      }
      if (w.l == w.d && w.half == 1) {
        const long long t0_ = P3T();
        mbar_wait_lazy(b_iodone, piod);
        if (p.prof) io_wait += clock64() - t0_;
        piod ^= 1u;
        const float cs = tcs[w.d];
        float y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = lane + 32 * k;
          y[k] = cs + part[r] + part[128 + r] + part[256 + r] + part[384 + r];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(b_partfree);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (cur[k] != 0xFFFFFFFFu) p.out[cur[k]] = y[k];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 4; ++k) { cur[k] = nxt[k]; nxt[k] = pre[k]; }
      }
      w.advance(tstride, T, s_tile_end, L);
    }
    if (p.prof && lane == 0) g_kprof3[blockIdx.x][11] = io_wait;
  } else if (warp >= 3) {
    // =========================== epilogue (16 warps; steps (A, l), (B, l) of the current tile)
    const int ew = warp - 3;
    const int q = warp & 3;
    const int cq = ew >> 2;
    const int quad = lane >> 2, tq = lane & 3;
    const uint32_t tm_q = tmem_base + ((uint32_t)(32 * q) << 16);
    const uint32_t a_st = sA + (uint32_t)(4 * q + (lane >> 3)) * 1024 + (uint32_t)(lane & 7) * 128;
    const float2 SM2 = make_float2(p.m.omega0, p.m.omega0);
    const float* tba = tab + p.m.pt_off_bias;  // [L][HP/2][bias pair, a pair], row 0 bias = 0
    const uint32_t afull_dst0 = rank == 0 ? b_afull : mapa_shared(b_afull, 0);
    auto quad_sum = [](float v) {
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      return v;
    };
    float ylin[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t pe[2] = {0u, 0u};
    uint32_t ppf = 1u;   // part_free parity: first tile passes immediately
    uint32_t pbh = 0;      // b_bhead parity (one phase per hidden-layer job B)
    unsigned long long ep[5] = {};
    const long long t_start = P3T();
    // Columns [c0, c0 + NCH * 8) of one half: TMEM -> sin -> tail partials, h packed to BF16 in registers.
    // The A-operand stores of half A (l >= 2) must wait until job (B, l) -- issued after job (A, l) and
    // reading all of H_{l-1} -- is past K-chunks 0..2 (b_bhead); half B's job is complete by then
    // (acc_full[B]).  Layer-1 jobs read the A1 buffer, not the A operand.
    // Chunks are stored as they are computed, except that with wait_b the first HOLD chunks are held in
    // registers until b_bhead (by then job B is normally past K-chunk 2).
    auto half_cols = [&](auto nch_c, int c0, int l, bool store, bool wait_b) {
      constexpr int NCH = decltype(nch_c)::value;
      constexpr int HOLD = 2;
      const float* ba = tba + (l - 1) * 2 * HP + (c0 + 2 * tq) * 2;
      float2 yv[4] = {};
      uint32_t held[HOLD > 0 ? HOLD : 1][4];
      auto put = [&](int ci, const uint32_t (&pk)[4]) {
        const uint32_t u = (uint32_t)((c0 + 8 * ci) >> 3);
        stmatrix_x4(a_st + (u >> 3) * C::A_CHUNK + (((u & 7u) ^ (uint32_t)(lane & 7)) << 4), pk);
      };
      auto release = [&]() {
        const long long t0_ = P3T();
        mbar_wait(b_bhead, pbh);
        if (p.prof) ep[2] += clock64() - t0_;
        pbh ^= 1u;
#pragma unroll
        for (int ci = 0; ci < HOLD; ++ci)
          if (ci < NCH) put(ci, held[ci]);
      };
#pragma unroll
      for (int i0 = 0; i0 < NCH; i0 += 2) {
        if (SAND_DIAG && p.prof >= 2) break;   // diagnostic (SAND_DIAG builds): no epilogue work
        uint32_t r0[8], r1[8];
        if (i0 + 1 < NCH) {
          tmem_ld_16x256b<2>(tm_q + c0 + 8 * i0, r0);
          tmem_ld_16x256b<2>(tm_q + (16u << 16) + c0 + 8 * i0, r1);
          tmem_wait_ld_dep(r0);
          tmem_wait_ld_dep(r1);
        } else {
          uint32_t s0[4], s1[4];
          tmem_ld_16x256b<1>(tm_q + c0 + 8 * i0, s0);
          tmem_ld_16x256b<1>(tm_q + (16u << 16) + c0 + 8 * i0, s1);
          tmem_wait_ld_dep(s0);
          tmem_wait_ld_dep(s1);
#pragma unroll
          for (int e = 0; e < 4; ++e) { r0[e] = s0[e]; r1[e] = s1[e]; r0[4 + e] = 0u; r1[4 + e] = 0u; }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (i0 + i < NCH) {
            const int ci = i0 + i;
            const int jc = 8 * ci;
            const float4 ba4 = *reinterpret_cast<const float4*>(ba + 2 * jc);
            const float2 b2 = make_float2(ba4.x, ba4.y), a2 = make_float2(ba4.z, ba4.w);
            uint32_t pk[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t* r = k < 2 ? r0 : r1;
              const int o = 4 * i + 2 * (k & 1);
              const float2 h = sin_mufu2(__ffma2_rn(make_float2(__uint_as_float(r[o]), __uint_as_float(r[o + 1])), SM2, b2));
              yv[k] = __ffma2_rn(a2, h, yv[k]);
              pk[k] = pack_bf16x2(h.x, h.y);
            }
            if (store) {
              if (ci < HOLD) {
                if (wait_b) {
#pragma unroll
                  for (int k = 0; k < 4; ++k) held[ci][k] = pk[k];
                } else {
                  put(ci, pk);
                }
              } else {
                if (ci == HOLD && wait_b) release();
                put(ci, pk);
              }
            }
          }
        }
      }
      if (store && wait_b && (NCH <= HOLD || (SAND_DIAG && p.prof >= 2))) release();   // (diagnostic modes skip the loop)
#pragma unroll
      for (int k = 0; k < 4; ++k) ylin[k] += yv[k].x + yv[k].y;
    };
    WideWalk w;
    w.ti = 0;
    w.set(pair, T, s_tile_end, L);
#pragma unroll 1
    while (!w.done) {
      const int hf = w.half, l = w.l, d = w.d;
      {
        const long long t0_ = P3T();
        mbar_wait(b_accfull + 8 * hf, pe[hf]);
        pe[hf] ^= 1u;
        if (p.prof) ep[hf] += clock64() - t0_;
      }
      ep[4] += 1;
      const bool store = l != d;
      // every hidden-layer job B completes one b_bhead phase: consumed by the half-A stores, or here
      if (hf == 1 && l >= 2 && !store) { mbar_wait(b_bhead, pbh); pbh ^= 1u; }
      tc_fence_after();
      if (hf == 0) half_cols(std::integral_constant<int, C::NA / 32>{}, cq * (C::NA / 4), l, store, l >= 2);
      else half_cols(std::integral_constant<int, C::NB / 32>{}, C::NA + cq * (C::NB / 4), l, store, false);
      if (store) fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(afull_dst0 + 8 * hf);
        else mbar_arrive_remote(afull_dst0 + 8 * hf);
      }
      if (l == d && hf == 1) {
        const long long t0_ = P3T();
        mbar_wait(b_partfree, ppf);
        ppf ^= 1u;
        if (p.prof) ep[3] += clock64() - t0_;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float v = quad_sum(ylin[k]);
          if (tq == 0) part[cq * 128 + 32 * q + quad + 8 * k] = v;
          ylin[k] = 0.f;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(b_iodone);
      }
      w.advance(tstride, T, s_tile_end, L);
    }
    if (p.prof && warp == 3 && lane == 0) {
      g_kprof3[blockIdx.x][6] = ep[0];
      g_kprof3[blockIdx.x][7] = ep[1];
      g_kprof3[blockIdx.x][8] = ep[2];
      g_kprof3[blockIdx.x][9] = clock64() - t_start;
      g_kprof3[blockIdx.x][10] = ep[4];
      g_kprof3[blockIdx.x][12] = ep[3];
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_cg2(tmem_base, 512);
}

// ------------------------------------------------------------------------------------ host side
static constexpr size_t kSmemMax3 = 232448;

template <int H>
static size_t smem_for3(long long pt_floats, int L, int nst) {
  using C = Tc3Shape<H>;
  return (size_t)C::A_BYTES + (size_t)nst * C::STAGE + C::W1_BYTES + C::A1_BYTES +
         (size_t)((pt_floats + 3) & ~3ll) * 4 + 4 * 128 * 4 + 4 * (size_t)(L + 2) * 8 + (3 * nst + 10) * 8 + 16;
}

bool tc3_available(int H, int tail) { return H == 336 && tail == SAND_TAIL_LINEAR; }

int tc3_padded_width(int H) { return (H + 31) / 32 * 32; }

bool tc3_usable(int L, int H, int tail) {
  if (!tc3_available(H, tail)) return false;
  MlpDev m{};
  tc2_table_layout(L, tc3_padded_width(H), tail, &m, true);
  return smem_for3<336>(m.pt_floats, L, 2) <= kSmemMax3;
}

void tc3_build_host(int L, int H, float w0, const float* const* W, const float* const* b, const float* const* a,
                    const float* c, MlpDev* m, std::vector<float>* tables, std::vector<uint16_t>* w1img,
                    std::vector<uint8_t>* img) {
  using C = Tc3Shape<336>;
  const int HP = C::HP;
  tc2_table_layout(L, HP, SAND_TAIL_LINEAR, m, true);
  tables->assign((size_t)m->pt_floats, 0.f);
  for (int i = 1; i < L; ++i)
    for (int j = 0; j < H; ++j) (*tables)[m->pt_off_bias + (size_t)i * 2 * HP + (size_t)(j / 2) * 4 + (j & 1)] = w0 * b[i][j];
  for (int i = 0; i < L; ++i) {
    for (int j = 0; j < H; ++j) (*tables)[m->pt_off_bias + (size_t)i * 2 * HP + (size_t)(j / 2) * 4 + 2 + (j & 1)] = a[i][j];
    (*tables)[m->pt_off_c + i] = c[i];
  }
  double cs = 0.0;
  for (int d = 1; d <= L; ++d) {
    cs += c[d - 1];
    (*tables)[m->pt_off_csum + d] = (float)cs;
  }
  auto bf = [](float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
  };
  auto lo_of = [&](float v, uint16_t hi) {
    uint32_t u = (uint32_t)hi << 16;
    float h;
    std::memcpy(&h, &u, 4);
    return bf(v - h);
  };
  // global output unit of (rank, half, local row)
  auto unit = [&](int r, int hf, int n) { return hf == 0 ? r * C::RA + n : C::NA + r * C::RB + n; };
  // layer-1 split-BF16 B operand: [rank][half A rows | half B rows] x 16, l1_off layout per half
  w1img->assign((size_t)2 * C::W1_BYTES / 2, 0);
  for (int r = 0; r < 2; ++r)
    for (int hf = 0; hf < 2; ++hf) {
      const int rows = hf ? C::RB : C::RA;
      uint8_t* basep = reinterpret_cast<uint8_t*>(w1img->data()) + (size_t)r * C::W1_BYTES + (hf ? C::RA * 32 : 0);
      for (int n = 0; n < rows; ++n) {
        const int u = unit(r, hf, n);
        if (u >= H) continue;
        auto put = [&](int k, uint16_t v) { *reinterpret_cast<uint16_t*>(basep + l1_off((uint32_t)n, (uint32_t)k)) = v; };
        for (int k = 0; k < 3; ++k) {
          const float wv = W[0][3 * u + k];
          const uint16_t hi = bf(wv);
          put(k, hi);
          put(3 + k, lo_of(wv, hi));
          put(6 + k, hi);
        }
        const uint16_t bhi = bf(b[0][u]);
        put(9, bhi);
        put(10, lo_of(b[0][u], bhi));
      }
    }
  // hidden layers: [L-1][rank][half A: KC x RA rows | half B: KC x RB rows][128 B], SW128 K-major
  const size_t per_rank = (size_t)C::KC * (C::RA + C::RB) * 128;
  img->assign((size_t)(L > 1 ? L - 1 : 0) * 2 * per_rank, 0);
  for (int i = 1; i < L; ++i)
    for (int r = 0; r < 2; ++r)
      for (int hf = 0; hf < 2; ++hf) {
        const int rows = hf ? C::RB : C::RA;
        uint8_t* hb = img->data() + ((size_t)(i - 1) * 2 + r) * per_rank + (hf ? (size_t)C::KC * C::RA * 128 : 0);
        for (int kc = 0; kc < C::KC; ++kc) {
          uint8_t* cb = hb + (size_t)kc * rows * 128;
          for (int n = 0; n < rows; ++n) {
            const int u = unit(r, hf, n);
            for (int kk = 0; kk < 64; ++kk) {
              const int k = 64 * kc + kk;
              if (u >= H || k >= H) continue;
              const size_t byte = (size_t)(n / 8) * 1024 + (n % 8) * 128 + ((((kk / 8) ^ (n % 8)) * 16)) + (kk % 8) * 2;
              *reinterpret_cast<uint16_t*>(cb + byte) = bf(W[i][(size_t)u * H + k]);
            }
          }
        }
      }
}

cudaError_t launch_tmlp_tc3(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                            float* out, int num_sms, cudaStream_t st) {
  if (m.H != 336) return cudaErrorInvalidValue;
  int nst = 0;
  for (int n = 2; n <= 6; ++n)
    if (smem_for3<336>(m.pt_floats, m.L, n) <= kSmemMax3) nst = n;
  if (!nst) return cudaErrorInvalidConfiguration;
  const size_t sm = smem_for3<336>(m.pt_floats, m.L, nst);
  const int prof = m.kprof;
  Tc3Params p{m, pts, perm, meta, out, nst, prof};
  const int grid = num_sms & ~1;
  k_tmlp_wide<336><<<grid, Tc3Shape<336>::THREADS, sm, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (prof && e == cudaSuccess) {
    static unsigned long long h[160][kProf3];
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(h, g_kprof3, sizeof h);
    if (e == cudaSuccess) {
      double a[kProf3] = {0};
      int nl = 0;
      for (int b = 0; b < grid; ++b) {
        for (int k = 0; k < kProf3; ++k)
          if (k > 4 || (b & 1) == 0) a[k] += (double)h[b][k];
        nl += (b & 1) == 0;
      }
      for (int k = 0; k < kProf3; ++k) a[k] /= (k <= 4 ? nl : grid);
      fprintf(stderr,
              "[kprof3] nst %d | MMA total %.0f wait_aA %.0f wait_aB %.0f wait_W %.0f wait_l1 %.0f | prod wait_empty "
              "%.0f | epi total %.0f steps %.0f wait_accA %.0f wait_accB %.0f wait_accB_store %.0f wait_part %.0f | "
              "IO wait %.0f\n",
              nst, a[4], a[0], a[1], a[2], a[3], a[5], a[9], a[10], a[6], a[7], a[8], a[12], a[11]);
    }
  }
  return e;
}

cudaError_t prepare_tc3() {
  return cudaFuncSetAttribute(k_tmlp_wide<336>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax3);
}

}  // namespace sand
