// tmlp_tc.cu -- persistent fused T-MLP kernel on 5th-generation tensor cores (SAND_BF16).
//
// Computes, for every binned 128-point tile of uniform exit depth d (Sec. 3.4):
//   layer 1   : h_1 = sin(w0 (W_1 x + b_1))                 FP32 FFMA (K = 3), t_1 = a_1 . h_1 + c_1
//   layer 2..d: Z = H_{l-1} W_l^T  on tcgen05 (A = bf16 h_{l-1} in SMEM, B = bf16 W_l streamed into
//               SMEM by the bulk-copy (TMA) engine, FP32 accumulator in TMEM), epilogue
//               h_l = sin(w0 Z + w0 b_l), t_l = a_l . h_l + c_l (Eq. 2) or the Eq. 3 product,
//               y += t_l, bf16(h_l) -> SMEM as the next layer's A operand
//   output    : sdf[perm[row]] = y_d  (the tail "fused at the exit layer" is the last addend).
//
// Warp roles (one CTA per SM, persistent over tiles):
//   warp 0      : weight producer -- cp.async.bulk of 64-column K-chunks of W_l (pre-swizzled SW128
//                 K-major image) into a ring of NST stages (w_full / w_empty mbarriers)
//   warp 1      : MMA issuer (one thread) -- tcgen05.mma kind::f16, M = 128, N = H (two MMAs if
//                 H > 256), tcgen05.commit -> w_empty (stage free) and acc_full (layer done)
//   warp 2      : TMEM allocator
//   warps 4..   : NSLOT epilogue warpgroups; warpgroup s owns tile slot s (its own A buffer and TMEM
//                 accumulator), thread = tile row = TMEM lane.  With NSLOT = 2 the MMA of one slot
//                 overlaps the sin/tail epilogue of the other (ping-pong).
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "sand_internal.h"
#include "tmlp_common.cuh"

namespace sand {

template <int H>
struct TcShape {
  static constexpr int KC = (H + 63) / 64;          // 64-column K chunks (128-byte swizzle atoms)
  static constexpr int A_CHUNK = kTileM * 128;      // bytes of one A K-chunk (128 rows x 128 B)
  static constexpr int A_BYTES = KC * A_CHUNK;
  static constexpr int W_CHUNK = H * 128;           // bytes of one W K-chunk (H rows x 128 B)
  static constexpr int N0 = H <= 256 ? H : ((H / 2 + 15) / 16) * 16;
  static constexpr int N1 = H - N0;
  static constexpr int NSLOT = (2 * H <= 512) ? 2 : 1;
  static constexpr int COLS_NEEDED = NSLOT * H;
  static constexpr int TMEM_COLS = COLS_NEEDED <= 32 ? 32 : COLS_NEEDED <= 64 ? 64 : COLS_NEEDED <= 128 ? 128
                                   : COLS_NEEDED <= 256 ? 256 : 512;
  static constexpr int THREADS = 128 + 128 * NSLOT;
  static_assert(H % 16 == 0, "H must be a multiple of 16");
  static_assert(N0 % 16 == 0 && N1 % 16 == 0 && N0 <= 256 && N1 <= 256, "bad N split");
};

struct TcParams {
  MlpDev m;
  const float* pts;
  const uint32_t* perm;
  const QueryMeta* meta;
  float* out;
  int nst;  // weight ring stages
};

template <int H, int TAIL>
__global__ void __launch_bounds__(TcShape<H>::THREADS, 1) k_tmlp_tc(const TcParams p) {
  using C = TcShape<H>;
  constexpr int NSLOT = C::NSLOT;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int nst = p.nst;
  const int L = p.m.L;
  // ---- shared memory carve-up
  const uint32_t sA = base;                                   // NSLOT x A_BYTES
  const uint32_t sW = sA + NSLOT * C::A_BYTES;                // nst x W_CHUNK
  float* tab = reinterpret_cast<float*>(gbase + (NSLOT * C::A_BYTES + nst * C::W_CHUNK));
  const long long ntab = p.m.tables_floats;
  long long* meta_s = reinterpret_cast<long long*>(tab + ((ntab + 3) & ~3ll));
  long long* s_tile_end = meta_s;
  long long* s_tile_begin = meta_s + kMaxBins;
  long long* s_start = meta_s + 2 * kMaxBins;
  long long* s_count = meta_s + 3 * kMaxBins;
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta_s + 4 * kMaxBins);
  const uint32_t b_wfull = smem_u32(bars);
  const uint32_t b_wempty = b_wfull + 8 * nst;
  const uint32_t b_afull = b_wempty + 8 * nst;
  const uint32_t b_accfull = b_afull + 8 * NSLOT;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * nst + 2 * NSLOT);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // ---- prologue: tables + metadata to SMEM, barriers, TMEM
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
    for (int i = 0; i < nst; ++i) { mbar_init(b_wfull + 8 * i, 1); mbar_init(b_wempty + 8 * i, 1); }
    for (int s = 0; s < NSLOT; ++s) { mbar_init(b_afull + 8 * s, 128); mbar_init(b_accfull + 8 * s, 1); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const long long T = p.meta->total_tiles;

  if (warp == 0) {
    // =========================== weight producer ===========================
    if (lane == 0) {
      JobGen<NSLOT> gen;
      gen.init(T, s_tile_end, L, blockIdx.x, gridDim.x);
      int s, l, st = 0;
      uint32_t ph = 0;
      const uint8_t* img = reinterpret_cast<const uint8_t*>(p.m.w_image);
      while (gen.next(s, l)) {
        const uint8_t* src = img + (size_t)(l - 2) * C::KC * C::W_CHUNK;
        for (int kc = 0; kc < C::KC; ++kc) {
          mbar_wait(b_wempty + 8 * st, ph ^ 1u);
          mbar_arrive_expect_tx(b_wfull + 8 * st, C::W_CHUNK);
          bulk_g2s(sW + st * C::W_CHUNK, src + (size_t)kc * C::W_CHUNK, C::W_CHUNK, b_wfull + 8 * st);
          if (++st == nst) { st = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // =========================== MMA issuer ===========================
    if (lane == 0) {
      JobGen<NSLOT> gen;
      gen.init(T, s_tile_end, L, blockIdx.x, gridDim.x);
      constexpr uint32_t ID0 = idesc_bf16(128, C::N0);
      constexpr uint32_t ID1 = idesc_bf16(128, C::N1 > 0 ? C::N1 : 16);
      int s, l, st = 0;
      uint32_t ph = 0, pa[NSLOT];
#pragma unroll
      for (int i = 0; i < NSLOT; ++i) pa[i] = 0;
      while (gen.next(s, l)) {
        mbar_wait(b_afull + 8 * s, pa[s]);
        pa[s] ^= 1u;
        tc_fence_after();
        const uint32_t acc = tmem_base + (uint32_t)(s * H);
        const uint32_t a_base = sA + s * C::A_BYTES;
        for (int kc = 0; kc < C::KC; ++kc) {
          mbar_wait(b_wfull + 8 * st, ph);
          tc_fence_after();
          const uint32_t w_base = sW + st * C::W_CHUNK;
          const int ksteps = (H - 64 * kc) >= 64 ? 4 : (H - 64 * kc) / 16;
          for (int k = 0; k < ksteps; ++k) {
            const uint64_t ad = desc_sw128(a_base + kc * C::A_CHUNK + 32 * k);
            const uint64_t bd = desc_sw128(w_base + 32 * k);
            const uint32_t accum = (kc | k) ? 1u : 0u;
            mma_bf16(acc, ad, bd, ID0, accum);
            if (C::N1 > 0) mma_bf16(acc + C::N0, ad, desc_sw128(w_base + C::N0 * 128 + 32 * k), ID1, accum);
          }
          mma_commit(b_wempty + 8 * st);
          if (++st == nst) { st = 0; ph ^= 1u; }
        }
        mma_commit(b_accfull + 8 * s);
      }
    }
  } else if (warp >= 4) {
    // =========================== epilogue warpgroups ===========================
    const int s = (warp - 4) >> 2;
    const int q = warp & 3;
    const int row = 32 * q + lane;
    const uint32_t tm_row = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(s * H);
    const uint32_t a_row = sA + s * C::A_BYTES + (row >> 3) * 1024 + (row & 7) * 128;
    const uint32_t swz = row & 7;
    const float4* w1 = reinterpret_cast<const float4*>(tab + p.m.off_w1);
    const float w0 = p.m.omega0;
    uint32_t pe = 0;
#pragma unroll 1
    for (int i = 0;; ++i) {
      const long long t = (long long)blockIdx.x + (long long)gridDim.x * ((long long)NSLOT * i + s);
      if (t >= T) break;
      const int d = tile_depth(t, s_tile_end, L);
      const long long r0 = s_start[d] + (t - s_tile_begin[d]) * kTileM;
      const bool valid = (r0 + row) < (s_start[d] + s_count[d]);
      const uint32_t idx = p.perm[valid ? r0 + row : r0];
      const float px = p.pts[3ll * idx], py = p.pts[3ll * idx + 1], pz = p.pts[3ll * idx + 2];
      // ---------------- layer 1 (FP32 SIMT, K = 3) + tail 1
      float2 acc = make_float2(tab[p.m.off_c], 0.0f);
      {
        const float4* a4p = reinterpret_cast<const float4*>(tab + p.m.off_a);
        const float2 X = make_float2(px, px), Y = make_float2(py, py), Z = make_float2(pz, pz);
#pragma unroll 1
        for (int u = 0; u < H / 8; ++u) {
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
      if (d >= 2) {
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(b_afull + 8 * s);
      }
      // ---------------- layers 2..d: TMEM accumulator -> sin -> tail -> next A
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
        constexpr int NC = H / 32;
        uint32_t ra[32], rb[32];
        tmem_ld32(tm_row, ra);
#pragma unroll 1
        for (int c = 0; c < NC; c += 2) {
          tmem_wait_ld_dep(ra);
          if (c + 1 < NC) tmem_ld32(tm_row + 32 * (c + 1), rb);
          epi_cols<32, TAIL>(ra, 32 * c, bias, a, a1, w0, s0, s1, store, a_row, swz, C::A_CHUNK);
          if (c + 1 < NC) {
            tmem_wait_ld_dep(rb);
            if (c + 2 < NC) tmem_ld32(tm_row + 32 * (c + 2), ra);
            epi_cols<32, TAIL>(rb, 32 * (c + 1), bias, a, a1, w0, s0, s1, store, a_row, swz, C::A_CHUNK);
          }
        }
        if (H % 32) {
          uint32_t rc[16];
          tmem_ld16(tm_row + 32 * NC, rc);
          tmem_wait_ld_dep(rc);
          epi_cols<16, TAIL>(rc, 32 * NC, bias, a, a1, w0, s0, s1, store, a_row, swz, C::A_CHUNK);
        }
        if (TAIL == SAND_TAIL_MULT)
          y += (s0.x + s0.y + tab[p.m.off_c + (l - 1)]) * (s1.x + s1.y + tab[p.m.off_c1 + (l - 2)]);
        else
          y += s0.x + s0.y + tab[p.m.off_c + (l - 1)];
        tc_fence_before();
        if (store) {
          fence_proxy_async_smem();
          mbar_arrive(b_afull + 8 * s);
        }
      }
      if (valid) p.out[idx] = y;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, C::TMEM_COLS);
}

// ------------------------------------------------------------------------------------ host side
template <int H>
static size_t smem_for(int L, int tail, int nst) {
  using C = TcShape<H>;
  const size_t tables = (size_t)4 * H + (size_t)(L - 1) * H + (size_t)L * H + L +
                        (tail == SAND_TAIL_MULT ? (size_t)(L - 1) * H + (L - 1) : 0);
  const size_t tab_bytes = ((tables + 3) & ~(size_t)3) * 4;
  return 1024 + (size_t)C::NSLOT * C::A_BYTES + (size_t)nst * C::W_CHUNK + tab_bytes +
         4 * kMaxBins * sizeof(long long) + (2 * nst + 2 * C::NSLOT) * 8 + 16;
}

static constexpr size_t kSmemMax = 232448;  // 227 KB opt-in per CTA on sm_100

template <int H>
static int pick_nst(int L, int tail) {
  int best = 0;
  for (int nst = 2; nst <= 8; ++nst)
    if (smem_for<H>(L, tail, nst) <= kSmemMax) best = nst;
  return best;
}

bool tc_supported_H(int H) { return H == 64 || H == 128 || H == 256 || H == 336; }

size_t tc_smem_bytes(int L, int H, int tail) {
  int nst = 0;
  size_t b = 0;
  switch (H) {
    case 64: nst = pick_nst<64>(L, tail); b = nst ? smem_for<64>(L, tail, nst) : 0; break;
    case 128: nst = pick_nst<128>(L, tail); b = nst ? smem_for<128>(L, tail, nst) : 0; break;
    case 256: nst = pick_nst<256>(L, tail); b = nst ? smem_for<256>(L, tail, nst) : 0; break;
    case 336: nst = pick_nst<336>(L, tail); b = nst ? smem_for<336>(L, tail, nst) : 0; break;
    default: return 0;
  }
  return b;
}

template <int H, int TAIL>
static cudaError_t launch_tc_t(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                               float* out, int num_sms, cudaStream_t st) {
  const int nst = pick_nst<H>(m.L, TAIL);
  if (!nst) return cudaErrorInvalidConfiguration;
  const size_t sm = smem_for<H>(m.L, TAIL, nst);
  TcParams p{m, pts, perm, meta, out, nst};
  k_tmlp_tc<H, TAIL><<<num_sms, TcShape<H>::THREADS, sm, st>>>(p);
  return cudaGetLastError();
}

template <int H, int TAIL>
static cudaError_t prep_tc_t() {
  return cudaFuncSetAttribute(k_tmlp_tc<H, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
}



int tmlp_tile_rows(int H, int prec, int pair_mode) {
  if (prec == SAND_F16X3) return 256;
  return (prec == SAND_BF16 && pair_mode && (tc2_available(H) || tc3_available(H, SAND_TAIL_LINEAR))) ? 256 : kTileM;
}

cudaError_t launch_tmlp_tc(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                           float* out, int num_sms, cudaStream_t st, int pair_mode) {
  if (pair_mode == 2 && m.tc4_w1 && tc4_runs(m.L, m.H, m.tail, SAND_BF16, pair_mode))
    return launch_tmlp_tc4(m, pts, perm, meta, out, num_sms, st);
  if (pair_mode && tc2_available(m.H)) return launch_tmlp_tc2(m, pts, perm, meta, out, num_sms, st);
  if (pair_mode && tc3_available(m.H, m.tail)) return launch_tmlp_tc3(m, pts, perm, meta, out, num_sms, st);
  const bool mult = m.tail == SAND_TAIL_MULT;
#define SAND_TC_CASE(HH)                                                                     \
  case HH:                                                                                   \
    return mult ? launch_tc_t<HH, SAND_TAIL_MULT>(m, pts, perm, meta, out, num_sms, st)      \
                : launch_tc_t<HH, SAND_TAIL_LINEAR>(m, pts, perm, meta, out, num_sms, st);
  switch (m.H) {
    SAND_TC_CASE(64)
    SAND_TC_CASE(128)
    SAND_TC_CASE(256)
    SAND_TC_CASE(336)
    default: return cudaErrorInvalidValue;
  }
#undef SAND_TC_CASE
}

cudaError_t prepare_simt(int L, int H, int tail);

cudaError_t prepare_tmlp_kernels(int L, int H, int tail, int prec) {
  if (prec == SAND_FP32) return simt_supported_H(H) ? prepare_simt(L, H, tail) : cudaSuccess;   // wide: launch-time
  const bool mult = tail == SAND_TAIL_MULT;
  if (tc2_available(H)) {
    const cudaError_t e = prepare_tc2(H, tail);
    if (e != cudaSuccess) return e;
  }
  if (tc4_available(H, tail)) {
    const cudaError_t e = prepare_tc4(H, tail);
    if (e != cudaSuccess) return e;
  }
  if (tc3_available(H, tail)) {
    const cudaError_t e = prepare_tc3();
    if (e != cudaSuccess) return e;
  }
  switch (H) {
    case 64: return mult ? prep_tc_t<64, 1>() : prep_tc_t<64, 0>();
    case 128: return mult ? prep_tc_t<128, 1>() : prep_tc_t<128, 0>();
    case 256: return mult ? prep_tc_t<256, 1>() : prep_tc_t<256, 0>();
    case 336: return mult ? prep_tc_t<336, 1>() : prep_tc_t<336, 0>();
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sand
