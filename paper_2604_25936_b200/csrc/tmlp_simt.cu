// tmlp_simt.cu -- FP32 SIMT T-MLP kernel (SAND_FP32 precision; BASELINE.json configs[0]).
//
// Evaluates Eq. 2 with Eq. 3 tails for binned tiles of 128 points of
// one uniform exit depth d: h_1 = sin(w0 (W_1 x + b_1)), h_i = sin(w0 (W_i h_{i-1} + b_i)),
// y_d = sum_{i<=d} t_i.  One thread = one point; the hidden vector lives in registers (H <= 64); the
// hidden weights live in shared memory and are read as warp-uniform broadcasts.  The sine is a
// two-constant Cody-Waite reduction to [-pi, pi] followed by MUFU.SIN (~4e-7 absolute, FP32-grade for a
// SIREN layer's |z| <~ 100; libm sinf cost ~5x the instructions: C0 0.265 ms before), well inside the
// north star's 1e-4 FP32 tolerance.  Small-H configs (C0 is 4 x 64) are
// FMA/launch bound, not tensor bound: at H = 64 an H x H layer is 4096 FMAs per point.
#include <cstdint>
#include <cuda_runtime.h>

#include "sand_internal.h"

namespace sand {

__device__ __forceinline__ float simt_sin(float x) {
  const float k = rintf(x * 0.159154943091895f);
  float r = fmaf(-k, 6.28318548202514648f, x);
  r = fmaf(-k, -1.7484555314695172e-7f, r);
  return __sinf(r);
}

template <int H, int TAIL>
__global__ void __launch_bounds__(kTileM) k_tmlp_simt(MlpDev m, const float* __restrict__ pts,
                                                      const uint32_t* __restrict__ perm,
                                                      const QueryMeta* __restrict__ meta,
                                                      float* __restrict__ out) {
  extern __shared__ __align__(16) float sm[];
  const int L = m.L;
  const long long nw = (long long)(L - 1) * H * H;
  float* sw = sm;                  // hidden weights [(L-1)][H][H]
  float* st = sm + nw;             // tables
  for (long long i = threadIdx.x; i < nw; i += blockDim.x) sw[i] = m.w_hidden[i];
  for (long long i = threadIdx.x; i < m.tables_floats; i += blockDim.x) st[i] = m.tables[i];
  __shared__ long long s_tile_end[kMaxBins], s_tile_begin[kMaxBins], s_start[kMaxBins], s_count[kMaxBins];
  if (threadIdx.x < kMaxBins) {
    s_tile_end[threadIdx.x] = meta->tile_end[threadIdx.x];
    s_tile_begin[threadIdx.x] = meta->tile_begin[threadIdx.x];
    s_start[threadIdx.x] = meta->start[threadIdx.x];
    s_count[threadIdx.x] = meta->count[threadIdx.x];
  }
  __syncthreads();
  const long long T = meta->total_tiles;
  const float4* w1 = reinterpret_cast<const float4*>(st + m.off_w1);
  const float w0 = m.omega0;
  for (long long t = blockIdx.x; t < T; t += gridDim.x) {
    int d = 0;
    for (int dd = L; dd >= 1; --dd)
      if (t < s_tile_end[dd]) { d = dd; break; }
    const long long row = s_start[d] + (t - s_tile_begin[d]) * kTileM + threadIdx.x;
    if (row >= s_start[d] + s_count[d]) continue;
    const uint32_t idx = perm[row];
    const float px = pts[3ll * idx], py = pts[3ll * idx + 1], pz = pts[3ll * idx + 2];
    float h[H];
    float y = st[m.off_c];
    {
      const float* a = st + m.off_a;
#pragma unroll
      for (int j = 0; j < H; ++j) {
        const float4 w = w1[j];
        h[j] = simt_sin(fmaf(w.z, pz, fmaf(w.y, py, fmaf(w.x, px, w.w))));
        y = fmaf(a[j], h[j], y);
      }
    }
    for (int l = 2; l <= d; ++l) {
      const float* W = sw + (long long)(l - 2) * H * H;
      const float* bias = st + m.off_bias + (long long)(l - 2) * H;
      const float* a = st + m.off_a + (long long)(l - 1) * H;
      float hn[H];
#pragma unroll
      for (int j = 0; j < H; ++j) {
        const float4* Wr = reinterpret_cast<const float4*>(W + j * H);
        float z = 0.0f;
#pragma unroll
        for (int k = 0; k < H / 4; ++k) {
          const float4 w = Wr[k];
          z = fmaf(w.x, h[4 * k], z);
          z = fmaf(w.y, h[4 * k + 1], z);
          z = fmaf(w.z, h[4 * k + 2], z);
          z = fmaf(w.w, h[4 * k + 3], z);
        }
        hn[j] = simt_sin(fmaf(z, w0, bias[j]));
      }
      float s0 = st[m.off_c + (l - 1)], s1 = 0.0f;
      if (TAIL == SAND_TAIL_MULT) s1 = st[m.off_c1 + (l - 2)];
      const float* a1 = st + m.off_a1 + (long long)(l - 2) * H;
#pragma unroll
      for (int j = 0; j < H; ++j) {
        h[j] = hn[j];
        s0 = fmaf(a[j], h[j], s0);
        if (TAIL == SAND_TAIL_MULT) s1 = fmaf(a1[j], h[j], s1);
      }
      y += (TAIL == SAND_TAIL_MULT) ? s0 * s1 : s0;
    }
    out[idx] = y;
  }
}

bool simt_supported_H(int H) { return H == 16 || H == 32 || H == 64; }

size_t simt_smem_bytes(int L, int H, int tail) {
  const size_t tables = (size_t)4 * H + (size_t)(L - 1) * H + (size_t)L * H + L +
                        (tail == SAND_TAIL_MULT ? (size_t)(L - 1) * H + (L - 1) : 0) + 16;
  return ((size_t)(L - 1) * H * H + tables) * sizeof(float);
}

template <int H, int TAIL>
static cudaError_t prep_simt(int L) {
  const size_t sm = simt_smem_bytes(L, H, TAIL);
  return cudaFuncSetAttribute(k_tmlp_simt<H, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
}

template <int H>
static cudaError_t launch_h(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                            float* out, int num_sms, cudaStream_t st) {
  const size_t sm = simt_smem_bytes(m.L, H, m.tail);
  const int grid = num_sms * 4;
  if (m.tail == SAND_TAIL_MULT)
    k_tmlp_simt<H, SAND_TAIL_MULT><<<grid, kTileM, sm, st>>>(m, pts, perm, meta, out);
  else
    k_tmlp_simt<H, SAND_TAIL_LINEAR><<<grid, kTileM, sm, st>>>(m, pts, perm, meta, out);
  return cudaGetLastError();
}

cudaError_t launch_tmlp_simt(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                             float* out, int num_sms, cudaStream_t st) {
  switch (m.H) {
    case 16: return launch_h<16>(m, pts, perm, meta, out, num_sms, st);
    case 32: return launch_h<32>(m, pts, perm, meta, out, num_sms, st);
    case 64: return launch_h<64>(m, pts, perm, meta, out, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t prepare_simt(int L, int H, int tail) {
  const bool mult = tail == SAND_TAIL_MULT;
  switch (H) {
    case 16: return mult ? prep_simt<16, 1>(L) : prep_simt<16, 0>(L);
    case 32: return mult ? prep_simt<32, 1>(L) : prep_simt<32, 0>(L);
    case 64: return mult ? prep_simt<64, 1>(L) : prep_simt<64, 0>(L);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sand
