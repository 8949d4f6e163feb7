// tmlp_tc2.cu -- CTA-pair (cta_group::2) persistent fused T-MLP kernel (SAND_BF16, H in {128, 256}).
//
// Same computation as tmlp_tc.cu (Eq. 2 / Eq. 3 of PAPER.md, per binned tile of uniform exit depth),
// re-tiled for the B200 CTA pair: a cluster of two CTAs on one TPC processes 256-row tiles; the even
// CTA issues tcgen05.mma.cta_group::2 with M = 256 (rows 0-127 = even CTA's A in its SMEM and its
// TMEM lanes, rows 128-255 = odd CTA's) and N = H, where each CTA streams only HALF of every weight
// K-chunk (N/2 rows).  Per SM that halves the L2 -> SMEM weight bytes per FLOP against the 1-CTA
// kernel (32 instead of 64 B/clk at full MMA rate for H = 256), which is what bounds the 1-CTA kernel.
//
// Synchronisation (all mbarriers; "leader" = even CTA of the pair):
//   w_full[st]  (each CTA)  its own half-chunk landed (bulk-copy transaction bytes)
//   w_peer[st]  (leader)    relay thread of the odd CTA: "my half of stage st landed"
//   w_empty[st] (each CTA)  MMAs of stage st done (multicast tcgen05.commit from the leader)
//   a_full[s]   (leader)    slot s activations of both CTAs written (2 arrivals, one per CTA)
//   acc_full[s] (each CTA)  slot s accumulator complete (multicast tcgen05.commit)
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "sand_internal.h"
#include "tmlp_common.cuh"

namespace sand {

template <int H>
struct Tc2Shape {
  static constexpr int KC = H / 64;
  static constexpr int A_CHUNK = 128 * 128;        // one K-chunk of this CTA's 128 rows
  static constexpr int A_BYTES = KC * A_CHUNK;
  static constexpr int W_CHUNK = H * 128;          // full K-chunk of W (both halves) in the image
  static constexpr int WH_CHUNK = (H / 2) * 128;   // this CTA's half (N/2 rows)
  static constexpr int NSLOT = 2;
  static constexpr int NHALF = 2;                  // epilogue warpgroups per slot (column halves)
  static constexpr int HC = H / NHALF;             // columns per epilogue warpgroup
  static constexpr int TMEM_COLS = 2 * H <= 256 ? 256 : 512;
  static constexpr int THREADS = 128 + 128 * NSLOT * NHALF;
  static constexpr int TILE = 256;
  static_assert(H % 64 == 0 && H <= 256, "CTA-pair kernel: H in {64, 128, 192, 256}");
};

struct Tc2Params {
  MlpDev m;
  const float* pts;
  const uint32_t* perm;
  const QueryMeta* meta;
  float* out;
  int nst;
};

template <int H, int TAIL>
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
  const long long ntab = p.m.tables_floats;
  long long* meta_s = reinterpret_cast<long long*>(tab + ((ntab + 3) & ~3ll));
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
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * nst + 2 * NSLOT);
  float* ybuf = reinterpret_cast<float*>(bars + 3 * nst + 2 * NSLOT + 2);   // [NSLOT][2][128] tail partials

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const float4* src = reinterpret_cast<const float4*>(p.m.tables);
    float4* dst = reinterpret_cast<float4*>(tab);
    for (long long i = tid; i < (ntab + 3) / 4; i += blockDim.x) dst[i] = src[i];
    if (tid < kMaxBins) {
      s_tile_end[tid] = p.meta->tile_end[tid];
      s_tile_begin[tid] = p.meta->tile_begin[tid];
      s_start[tid] = p.meta->start[tid];
      s_count[tid] = p.meta->count[tid];
    }
  }
  if (tid == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(b_wfull + 8 * i, 1);
      mbar_init(b_wempty + 8 * i, 1);
      mbar_init(b_wpeer + 8 * i, 1);
    }
    for (int s = 0; s < NSLOT; ++s) { mbar_init(b_afull + 8 * s, 2); mbar_init(b_accfull + 8 * s, 1); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_cg2(smem_u32(tmem_slot), C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();   // both CTAs' barriers initialised before any remote arrive / multicast commit
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const long long T = p.meta->total_tiles;

  if (warp == 0) {
    // =========================== weight producer (both CTAs: own half of every chunk)
    if (lane == 0) {
      JobGen<NSLOT> gen;
      gen.init(T, s_tile_end, L, pair, npairs);
      int s, l, st = 0;
      uint32_t ph = 0;
      const uint8_t* img = reinterpret_cast<const uint8_t*>(p.m.w_image) + rank * C::WH_CHUNK;
      while (gen.next(s, l)) {
        const uint8_t* src = img + (size_t)(l - 2) * C::KC * C::W_CHUNK;
        for (int kc = 0; kc < C::KC; ++kc) {
          mbar_wait(b_wempty + 8 * st, ph ^ 1u);
          mbar_arrive_expect_tx(b_wfull + 8 * st, C::WH_CHUNK);
          bulk_g2s(sW + st * C::WH_CHUNK, src + (size_t)kc * C::W_CHUNK, C::WH_CHUNK, b_wfull + 8 * st);
          if (++st == nst) { st = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      JobGen<NSLOT> gen;
      gen.init(T, s_tile_end, L, pair, npairs);
      int s, l, st = 0;
      uint32_t ph = 0;
      if (rank == 0) {
        // =========================== MMA issuer (leader CTA)
        constexpr uint32_t ID = idesc_bf16(256, H);
        uint32_t pa[NSLOT] = {0, 0};
        while (gen.next(s, l)) {
          mbar_wait_cluster(b_afull + 8 * s, pa[s]);
          pa[s] ^= 1u;
          tc_fence_after();
          const uint32_t acc = tmem_base + (uint32_t)(s * H);
          const uint32_t a_base = sA + s * C::A_BYTES;
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
          mma_commit_cg2_mc(b_accfull + 8 * s, 0x3);
        }
      } else {
        // =========================== relay (odd CTA): "my half of stage st landed" -> leader
        const uint32_t peer_wpeer = mapa_shared(b_wpeer, 0);
        while (gen.next(s, l)) {
          for (int kc = 0; kc < C::KC; ++kc) {
            mbar_wait(b_wfull + 8 * st, ph);
            mbar_arrive_remote(peer_wpeer + 8 * st);
            if (++st == nst) { st = 0; ph ^= 1u; }
          }
        }
      }
    }
  } else if (warp >= 4) {
    // =========================== epilogue warpgroups (both CTAs)
    // warpgroup (s, hh): tile slot s, accumulator columns [hh*HC, hh*HC + HC); thread = local row.
    const int wg = (warp - 4) >> 2;
    const int s = wg / C::NHALF, hh = wg % C::NHALF;
    const int q = warp & 3;
    const int row = 32 * q + lane;                          // TMEM lane / local A row
    const int prow = (int)rank * 128 + row;                 // row within the 256-row pair tile
    const int c_lo = hh * C::HC;
    const uint32_t tm_row = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(s * H + c_lo);
    const uint32_t a_row = sA + s * C::A_BYTES + (row >> 3) * 1024 + (row & 7) * 128;
    const uint32_t swz = row & 7;
    const float4* w1 = reinterpret_cast<const float4*>(tab + p.m.off_w1);
    const float w0 = p.m.omega0;
    const uint32_t afull_dst = rank == 0 ? b_afull + 8 * s : mapa_shared(b_afull + 8 * s, 0);
    const bool signaller = (hh == 0 && q == 0 && lane == 0);
    const uint32_t bar_pub = 1 + s, bar_red = 1 + NSLOT + s;
    constexpr uint32_t kSlotThreads = 128 * C::NHALF;
    auto publish_A = [&]() {
      // every writer: generic->async proxy fence + TMEM-read ordering, then one arrive per CTA
      fence_proxy_async_smem();
      tc_fence_before();
      named_bar_sync(bar_pub, kSlotThreads);
      if (signaller) {
        if (rank == 0) mbar_arrive(afull_dst);
        else mbar_arrive_remote(afull_dst);
      }
    };
    uint32_t pe = 0;
    // software prefetch of the next tile's point (perm -> pts) behind the current tile's work
    auto tile_of = [&](int i) { return (long long)pair + (long long)npairs * ((long long)NSLOT * i + s); };
    auto row_index = [&](long long t, int& d, bool& valid) -> uint32_t {
      d = tile_depth(t, s_tile_end, L);
      const long long r0 = s_start[d] + (t - s_tile_begin[d]) * C::TILE;
      valid = (r0 + prow) < (s_start[d] + s_count[d]);
      return p.perm[valid ? r0 + prow : r0];
    };
    long long t = tile_of(0);
    int d = 0;
    bool valid = false;
    uint32_t idx = 0;
    float px = 0.f, py = 0.f, pz = 0.f;
    if (t < T) {
      idx = row_index(t, d, valid);
      px = p.pts[3ll * idx]; py = p.pts[3ll * idx + 1]; pz = p.pts[3ll * idx + 2];
    }
#pragma unroll 1
    for (int i = 0; t < T; ++i) {
      const long long tn = tile_of(i + 1);
      int dn = 0;
      bool valid_n = false;
      uint32_t idx_n = 0;
      if (tn < T) idx_n = row_index(tn, dn, valid_n);
      // ---------------- layer 1 (FP32 SIMT, K = 3) + tail 1, columns [c_lo, c_lo + HC)
      float2 acc = make_float2(hh == 0 ? tab[p.m.off_c] : 0.0f, 0.0f);
      {
        const float4* a4p = reinterpret_cast<const float4*>(tab + p.m.off_a);
        const float2 X = make_float2(px, px), Y = make_float2(py, py), Z = make_float2(pz, pz);
#pragma unroll 1
        for (int u = c_lo / 8; u < (c_lo + C::HC) / 8; ++u) {
          float hv[8];
#pragma unroll
          for (int jj = 0; jj < 8; jj += 2) {
            const float4 wa = w1[8 * u + jj], wb = w1[8 * u + jj + 1];
            float2 z = __ffma2_rn(make_float2(wa.x, wb.x), X, make_float2(wa.w, wb.w));
            z = __ffma2_rn(make_float2(wa.y, wb.y), Y, z);
            z = __ffma2_rn(make_float2(wa.z, wb.z), Z, z);
            hv[jj] = __sinf(z.x);
            hv[jj + 1] = __sinf(z.y);
          }
          const float4 a0 = a4p[2 * u], a1v = a4p[2 * u + 1];
          acc = __ffma2_rn(make_float2(a0.x, a0.y), make_float2(hv[0], hv[1]), acc);
          acc = __ffma2_rn(make_float2(a0.z, a0.w), make_float2(hv[2], hv[3]), acc);
          acc = __ffma2_rn(make_float2(a1v.x, a1v.y), make_float2(hv[4], hv[5]), acc);
          acc = __ffma2_rn(make_float2(a1v.z, a1v.w), make_float2(hv[6], hv[7]), acc);
          if (d >= 2) {
            const uint32_t addr = a_row + (u >> 3) * C::A_CHUNK + ((((uint32_t)u & 7u) ^ swz) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(pack_bf16x2(hv[0], hv[1])),
                         "r"(pack_bf16x2(hv[2], hv[3])), "r"(pack_bf16x2(hv[4], hv[5])),
                         "r"(pack_bf16x2(hv[6], hv[7]))
                         : "memory");
          }
        }
      }
      float y = acc.x + acc.y;
      if (d >= 2) publish_A();
      // next tile's coordinates: the perm load above has landed by now
      float pxn = 0.f, pyn = 0.f, pzn = 0.f;
      if (tn < T) { pxn = p.pts[3ll * idx_n]; pyn = p.pts[3ll * idx_n + 1]; pzn = p.pts[3ll * idx_n + 2]; }
      // ---------------- layers 2..d
#pragma unroll 1
      for (int l = 2; l <= d; ++l) {
        mbar_wait(b_accfull + 8 * s, pe);
        pe ^= 1u;
        tc_fence_after();
        const bool store = (l != d);
        const float* bias = tab + p.m.off_bias + (long long)(l - 2) * H;
        const float* a = tab + p.m.off_a + (long long)(l - 1) * H;
        const float* a1 = tab + p.m.off_a1 + (long long)(l - 2) * H;
        float2 s0 = make_float2(0.0f, 0.0f), s1 = make_float2(0.0f, 0.0f);
        constexpr int NC = C::HC / 16;
        uint32_t ra[16], rb[16];
        tmem_ld16(tm_row, ra);
#pragma unroll 1
        for (int c = 0; c < NC; c += 2) {
          tmem_wait_ld_dep(ra);
          if (c + 1 < NC) tmem_ld16(tm_row + 16 * (c + 1), rb);
          epi_cols<16, TAIL>(ra, c_lo + 16 * c, bias, a, a1, w0, s0, s1, store, a_row, swz, C::A_CHUNK);
          if (c + 1 < NC) {
            tmem_wait_ld_dep(rb);
            if (c + 2 < NC) tmem_ld16(tm_row + 16 * (c + 2), ra);
            epi_cols<16, TAIL>(rb, c_lo + 16 * (c + 1), bias, a, a1, w0, s0, s1, store, a_row, swz, C::A_CHUNK);
          }
        }
        if (TAIL == SAND_TAIL_MULT) {
          // Eq. 3 needs both full dot products: reduce the two column halves through SMEM
          float* yb = ybuf + (s * 2 + 0) * 256;
          if (hh == 1) { yb[row] = s0.x + s0.y; yb[128 + row] = s1.x + s1.y; }
          tc_fence_before();
          named_bar_sync(bar_red, kSlotThreads);
          if (hh == 0)
            y += (s0.x + s0.y + yb[row] + tab[p.m.off_c + (l - 1)]) *
                 (s1.x + s1.y + yb[128 + row] + tab[p.m.off_c1 + (l - 2)]);
          named_bar_sync(bar_red, kSlotThreads);
        } else {
          y += s0.x + s0.y + (hh == 0 ? tab[p.m.off_c + (l - 1)] : 0.0f);
        }
        if (store) publish_A();
        else tc_fence_before();
      }
      // combine the two column halves' partial y (double-buffered by tile parity)
      float* yb = ybuf + (s * 2 + 1) * 256 + (i & 1) * 128;
      if (hh == 1) yb[row] = y;
      named_bar_sync(bar_red, kSlotThreads);
      if (hh == 0 && valid) p.out[idx] = y + yb[row];
      t = tn; d = dn; valid = valid_n; idx = idx_n; px = pxn; py = pyn; pz = pzn;
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
static size_t smem_for2(int L, int tail, int nst) {
  using C = Tc2Shape<H>;
  const size_t tables = (size_t)4 * H + (size_t)(L - 1) * H + (size_t)L * H + L +
                        (tail == SAND_TAIL_MULT ? (size_t)(L - 1) * H + (L - 1) : 0);
  const size_t tab_bytes = ((tables + 3) & ~(size_t)3) * 4;
  return 1024 + (size_t)C::NSLOT * C::A_BYTES + (size_t)nst * C::WH_CHUNK + tab_bytes +
         4 * kMaxBins * sizeof(long long) + (3 * nst + 2 * C::NSLOT) * 8 + 16 + C::NSLOT * 2 * 256 * 4;
}

static constexpr size_t kSmemMax2 = 232448;

template <int H>
static int pick_nst2(int L, int tail) {
  int best = 0;
  for (int nst = 2; nst <= 8; ++nst)
    if (smem_for2<H>(L, tail, nst) <= kSmemMax2) best = nst;
  return best;
}

size_t tc2_smem_bytes(int L, int H, int tail) {
  switch (H) {
    case 128: { const int n = pick_nst2<128>(L, tail); return n ? smem_for2<128>(L, tail, n) : 0; }
    case 256: { const int n = pick_nst2<256>(L, tail); return n ? smem_for2<256>(L, tail, n) : 0; }
    default: return 0;
  }
}

template <int H, int TAIL>
static cudaError_t launch_tc2_t(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                                float* out, int num_sms, cudaStream_t st) {
  const int nst = pick_nst2<H>(m.L, TAIL);
  if (!nst) return cudaErrorInvalidConfiguration;
  const size_t sm = smem_for2<H>(m.L, TAIL, nst);
  Tc2Params p{m, pts, perm, meta, out, nst};
  k_tmlp_tc2<H, TAIL><<<num_sms & ~1, Tc2Shape<H>::THREADS, sm, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_tmlp_tc2(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                            float* out, int num_sms, cudaStream_t st) {
  const bool mult = m.tail == SAND_TAIL_MULT;
  switch (m.H) {
    case 128: return mult ? launch_tc2_t<128, 1>(m, pts, perm, meta, out, num_sms, st)
                          : launch_tc2_t<128, 0>(m, pts, perm, meta, out, num_sms, st);
    case 256: return mult ? launch_tc2_t<256, 1>(m, pts, perm, meta, out, num_sms, st)
                          : launch_tc2_t<256, 0>(m, pts, perm, meta, out, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t prepare_tc2(int H, int tail) {
  const bool mult = tail == SAND_TAIL_MULT;
  auto set = [](const void* f) {
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax2);
  };
  switch (H) {
    case 128: return mult ? set((const void*)k_tmlp_tc2<128, 1>) : set((const void*)k_tmlp_tc2<128, 0>);
    case 256: return mult ? set((const void*)k_tmlp_tc2<256, 1>) : set((const void*)k_tmlp_tc2<256, 0>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sand
