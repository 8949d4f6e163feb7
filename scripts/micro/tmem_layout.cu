// Where does tcgen05.mma.cta_group::2 with M = 128 (64 rows per CTA) put D in TMEM, and can a second
// accumulator live at TMEM lane offset 16 (M=128 pair MMAs of two row-slots sharing columns)?
// D[row][n] = (row + 1) + 256 * n  (rows 0..127 across the pair, n < 64), via K = 16 operands.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_25936_b200/csrc/ptx.cuh"
using namespace sand;
__device__ __forceinline__ uint16_t bf(float f) { uint32_t u = __float_as_uint(f); return (uint16_t)((u + 0x7FFF + ((u >> 16) & 1)) >> 16); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(float* out, int lane_off) {
  __shared__ __align__(1024) uint8_t sa[64 * 32];   // A: 64 rows x 16 bf16 (this CTA's rows)
  __shared__ __align__(1024) uint8_t sb[32 * 32];   // B: this CTA's 32 of N = 64 rows x 16 bf16
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t rank = cluster_ctarank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 64 * 16; i += 128) {
    const int r = i / 16, kk = i % 16;
    const float v = kk == 0 ? (float)(rank * 64 + r + 1) : (kk == 1 ? 256.f : 0.f);
    *reinterpret_cast<uint16_t*>(sa + l1_off(r, kk)) = bf(v);
  }
  for (int i = tid; i < 32 * 16; i += 128) {
    const int n = i / 16, kk = i % 16;
    const int ng = rank * 32 + n;
    const float v = kk == 0 ? 1.f : (kk == 1 ? (float)ng : 0.f);
    *reinterpret_cast<uint16_t*>(sb + l1_off(n, kk)) = bf(v);
  }
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc_cg2(smem_u32(&tslot), 256);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (rank == 0 && tid == 0) {
    const uint32_t id = idesc_bf16(128, 64);
    mma_bf16_cg2(tb, desc_nosw(smem_u32(sa), 128, 256), desc_nosw(smem_u32(sb), 128, 256), id, 0u);
    mma_bf16_cg2(tb + ((uint32_t)lane_off << 16) + 128, desc_nosw(smem_u32(sa), 128, 256), desc_nosw(smem_u32(sb), 128, 256), id, 0u);
    mma_commit_cg2_mc(smem_u32(&bar), 0x3);
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  uint32_t r[16];
  for (int cb = 0; cb < 256; cb += 16) {
    tmem_ld16(tb + ((uint32_t)(32 * warp) << 16) + cb, r);
    tmem_wait_ld();
    for (int j = 0; j < 16; ++j) out[((size_t)rank * 128 + 32 * warp + lane) * 256 + cb + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_cg2(tb, 256);
}
int main() {
  float* d; cudaMalloc(&d, 2 * 128 * 256 * 4);
  static float h[2 * 128 * 256];
  for (int lo : {0, 16, 64}) {
    cudaMemset(d, 0, 2 * 128 * 256 * 4);
    k<<<2, 128>>>(d, lo);
    cudaError_t e = cudaDeviceSynchronize();
    printf("lane offset %d: %s\n", lo, cudaGetErrorString(e));
    if (e) return 1;
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    for (int rk = 0; rk < 2; ++rk) {
      for (int base : {0, 128}) {
        printf("  CTA %d cols %3d..: lanes holding D (lane:row/n) ", rk, base);
        int shown = 0;
        for (int ln = 0; ln < 128; ++ln) {
          const float v0 = h[((size_t)rk * 128 + ln) * 256 + base], v1 = h[((size_t)rk * 128 + ln) * 256 + base + 1];
          if (v0 != 0.f) { if (shown < 40) printf("%d:%g/%g ", ln, v0 - 1, (v1 - v0) / 256); ++shown; }
        }
        printf(" [%d lanes]\n", shown);
      }
    }
  }
  return 0;
}
