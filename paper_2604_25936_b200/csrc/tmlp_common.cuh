// tmlp_common.cuh -- device helpers shared by the 1-CTA and CTA-pair tcgen05 T-MLP kernels:
// the tile -> depth map, the deterministic MMA job sequence and the fused sin/tail epilogue.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "sand_internal.h"

namespace sand {

struct SlotState {
  long long t;
  int i, d, l, done;
};

__device__ __forceinline__ int tile_depth(long long t, const long long* tile_end, int L) {
  for (int d = L; d >= 1; --d)
    if (t < tile_end[d]) return d;
  return 0;
}

template <int NSLOT>
struct JobGen {
  SlotState S[NSLOT];
  int cur;
  long long T;
  const long long* tile_end;
  int L;
  int unit, nunits;  // this CTA's (or CTA pair's) index among `nunits` persistent workers
  __device__ __forceinline__ void set_tile(int s) {
    const long long t = (long long)unit + (long long)nunits * ((long long)NSLOT * S[s].i + s);
    S[s].t = t;
    if (t >= T) {
      S[s].done = 1;
    } else {
      S[s].d = tile_depth(t, tile_end, L);
      S[s].l = 2;
    }
  }
  __device__ __forceinline__ void init(long long T_, const long long* te, int L_, int unit_, int nunits_) {
    T = T_; tile_end = te; L = L_; cur = 0; unit = unit_; nunits = nunits_;
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) { S[s].i = 0; S[s].done = 0; set_tile(s); }
  }
  // Next MMA job (slot, layer) in round-robin order; tiles without remaining H x H layers (depth 1
  // or finished) are skipped.  Producer and MMA warps run identical copies of this generator.
  __device__ __forceinline__ bool next(int& s_out, int& l_out) {
#pragma unroll 1
    for (int tries = 0; tries < NSLOT; ++tries) {
      const int s = cur;
      cur = (cur + 1 == NSLOT) ? 0 : cur + 1;
      while (!S[s].done && S[s].l > S[s].d) { S[s].i++; set_tile(s); }
      if (!S[s].done) {
        s_out = s;
        l_out = S[s].l++;
        return true;
      }
    }
    return false;
  }
};

// Epilogue of NCOL accumulator columns [c0, c0 + NCOL) of one tile row (one thread):
// h = sin(w0 * z + w0 * b), tail partial sums s0 (+ s1 for Eq. 3), bf16(h) -> next A operand.
template <int NCOL, int TAIL>
__device__ __forceinline__ void epi_cols(const uint32_t (&r)[NCOL], int c0, const float* __restrict__ bias,
                                         const float* __restrict__ a, const float* __restrict__ a1, float w0,
                                         float2& s0, float2& s1, bool store, uint32_t a_row, uint32_t swz,
                                         int a_chunk) {
  const float2 W0 = make_float2(w0, w0);
#pragma unroll
  for (int g8 = 0; g8 < NCOL / 8; ++g8) {
    float hv[8];
#pragma unroll
    for (int q4 = 0; q4 < 2; ++q4) {
      const int j = c0 + 8 * g8 + 4 * q4;
      const int k = 8 * g8 + 4 * q4;
      const float4 b4 = *reinterpret_cast<const float4*>(bias + j);
      const float4 a4 = *reinterpret_cast<const float4*>(a + j);
      const float2 z01 = __ffma2_rn(make_float2(__uint_as_float(r[k]), __uint_as_float(r[k + 1])), W0,
                                    make_float2(b4.x, b4.y));
      const float2 z23 = __ffma2_rn(make_float2(__uint_as_float(r[k + 2]), __uint_as_float(r[k + 3])), W0,
                                    make_float2(b4.z, b4.w));
      const float h0 = __sinf(z01.x), h1 = __sinf(z01.y), h2 = __sinf(z23.x), h3 = __sinf(z23.y);
      s0 = __ffma2_rn(make_float2(a4.x, a4.y), make_float2(h0, h1), s0);
      s0 = __ffma2_rn(make_float2(a4.z, a4.w), make_float2(h2, h3), s0);
      if (TAIL == SAND_TAIL_MULT) {
        const float4 c4 = *reinterpret_cast<const float4*>(a1 + j);
        s1 = __ffma2_rn(make_float2(c4.x, c4.y), make_float2(h0, h1), s1);
        s1 = __ffma2_rn(make_float2(c4.z, c4.w), make_float2(h2, h3), s1);
      }
      hv[4 * q4 + 0] = h0; hv[4 * q4 + 1] = h1; hv[4 * q4 + 2] = h2; hv[4 * q4 + 3] = h3;
    }
    if (store) {
      const uint32_t u = (uint32_t)(c0 / 8 + g8);
      const uint32_t addr = a_row + (u >> 3) * a_chunk + (((u & 7u) ^ swz) << 4);
      asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(pack_bf16x2(hv[0], hv[1])),
                   "r"(pack_bf16x2(hv[2], hv[3])), "r"(pack_bf16x2(hv[4], hv[5])), "r"(pack_bf16x2(hv[6], hv[7]))
                   : "memory");
    }
  }
}

}  // namespace sand
