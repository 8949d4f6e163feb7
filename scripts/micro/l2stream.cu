// L2 -> SMEM bulk-copy streaming rate: every CTA (one per SM) streams 16 KB chunks of a small (L2-
// resident) weight image through an N-stage mbarrier ring, consuming each chunk immediately.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(128, 1) k(const uint8_t* img, int img_chunks, int nst, int iters, int chunk,
                                            unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  uint32_t ph[16] = {0};
  int issued = 0;
  // prologue
  for (; issued < nst && issued < iters; ++issued) {
    int st = issued % nst;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[st])), "r"(chunk));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + st * chunk)),
                 "l"(img + (size_t)((issued + blockIdx.x) % img_chunks) * chunk), "r"(chunk), "r"(su(&bar[st])) : "memory");
  }
  for (int i = 0; i < iters; ++i) {
    int st = i % nst;
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(su(&bar[st])), "r"(ph[st]));
    ph[st] ^= 1;
    if (issued < iters) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[st])), "r"(chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + st * chunk)),
                   "l"(img + (size_t)((issued + blockIdx.x) % img_chunks) * chunk), "r"(chunk), "r"(su(&bar[st])) : "memory");
      ++issued;
    }
  }
  cyc[blockIdx.x] = clock64() - t0;
}
int main() {
  uint8_t* img; cudaMalloc(&img, 1 << 20); cudaMemset(img, 1, 1 << 20);
  unsigned long long* c; cudaMalloc(&c, 148 * 8); unsigned long long h[148];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int chunk : {8192, 16384, 32768, 65536}) for (int nst : {1, 2, 3, 4, 8}) {
    if (nst * chunk > 196608) continue;
    int iters = 2000;
    k<<<148, 128, nst * chunk>>>(img, (1 << 20) / chunk, nst, iters, chunk, c);
    cudaError_t e = cudaDeviceSynchronize(); if (e) { printf("%s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("chunk %5d nst %2d: %.1f B/clk/SM (slowest CTA), latency-equiv %.0f clk per chunk\n", chunk, nst,
           (double)iters * chunk / mx, mx / iters * nst);
  }
  return 0;
}
