// Microbenchmarks for the K3 design: TMEM read bandwidth (tcgen05.ld), MUFU.SIN, FFMA vs FFMA2.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ void tld(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void tld<16>(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
    : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),
      "=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(taddr));
}

__global__ void __launch_bounds__(512, 1) k_tmem(int iters, int nw_active, unsigned long long* out_cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  if (warp < nw_active) {
    uint32_t r[16], q[16];
    int col = (warp >> 2) * 16;
    for (int i = 0; i < iters; ++i) {
      tld<16>(base + (col & 511), r);
      tld<16>(base + ((col + 64) & 511), q);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 16; ++k) acc ^= r[k] ^ q[k];
      col += 128;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out_cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot) : "memory");
}

__global__ void __launch_bounds__(512, 1) k_mufu(int iters, unsigned long long* out_cyc, float* sink) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __sinf(a[k]) + 1.5f;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out_cyc[blockIdx.x] = t1 - t0;
  float s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1234.5f) sink[0] = s;
}

__global__ void __launch_bounds__(512, 1) k_ffma(int iters, unsigned long long* out_cyc, float* sink, int use2) {
  float a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = threadIdx.x * 1e-3f + k;
  const float b = 0.999f, c = 1e-3f;
  __syncthreads();
  long long t0 = clock64();
  if (use2) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 16; k += 2) {
        float2 v = __ffma2_rn(make_float2(a[k], a[k + 1]), make_float2(b, b), make_float2(c, c));
        a[k] = v.x; a[k + 1] = v.y;
      }
    }
  } else {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 16; ++k) a[k] = fmaf(a[k], b, c);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out_cyc[blockIdx.x] = t1 - t0;
  float s = 0; for (int k = 0; k < 16; ++k) s += a[k];
  if (s == 1234.5f) sink[0] = s;
}

int main() {
  unsigned long long* d_c; cudaMalloc(&d_c, 148 * 8); unsigned long long h[148];
  uint32_t* sink; cudaMalloc(&sink, 64);
  int iters = 4096;
  for (int nw : {4, 8, 16}) {
    k_tmem<<<148, 512>>>(iters, nw, d_c, sink); cudaDeviceSynchronize();
    k_tmem<<<148, 512>>>(iters, nw, d_c, sink);
    cudaError_t e = cudaDeviceSynchronize(); if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d_c, sizeof h, cudaMemcpyDeviceToHost);
    double bytes = (double)iters * nw * 2 * 32 * 16 * 4;
    printf("TMEM ld: %2d warps: %.1f B/clk/SM (cyc %llu)\n", nw, bytes / h[0], h[0]);
  }
  for (int nthr : {128, 256, 512}) {
    k_mufu<<<148, nthr>>>(iters, d_c, (float*)sink); cudaDeviceSynchronize();
    k_mufu<<<148, nthr>>>(iters, d_c, (float*)sink); cudaDeviceSynchronize();
    cudaMemcpy(h, d_c, sizeof h, cudaMemcpyDeviceToHost);
    printf("MUFU sin: %d thr: %.2f sins/clk/SM\n", nthr, (double)iters * 8 * nthr / h[0]);
  }
  for (int u2 : {0, 1}) {
    k_ffma<<<148, 512>>>(iters, d_c, (float*)sink, u2); cudaDeviceSynchronize();
    k_ffma<<<148, 512>>>(iters, d_c, (float*)sink, u2); cudaDeviceSynchronize();
    cudaMemcpy(h, d_c, sizeof h, cudaMemcpyDeviceToHost);
    printf("%s: %.1f fma/clk/SM\n", u2 ? "FFMA2" : "FFMA", (double)iters * 16 * 512 / h[0]);
  }
  return 0;
}
