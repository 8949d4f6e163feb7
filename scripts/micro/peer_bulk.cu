// Can a cp.async.bulk issued by CTA 1 of a pair (destination: CTA 1's own shared memory) signal its completion on an
// mbarrier of CTA 0 (shared::cluster address)?  CTA 0 expects 2 x 16 KB on its barrier (its own copy + CTA 1's);
// bounded waits, prints ok / timeout and the data check.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_25936_b200/csrc/ptx.cuh"
using namespace sand;
__global__ void __cluster_dims__(2, 1, 1) k(const uint4* src, int* result, int mode) {
  __shared__ __align__(128) uint4 buf[1024];   // 16 KB
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  __syncthreads();
  cluster_sync();
  const uint32_t bar0 = mapa_shared(smem_u32(&bar), 0);   // leader's barrier, cluster address
  if (threadIdx.x == 0) {
    if (rank == 0) mbar_arrive_expect_tx(smem_u32(&bar), mode ? 2 * 16384 : 16384);
  }
  cluster_sync();
  if (threadIdx.x == 0) {
    const uint32_t dst = smem_u32(buf);
    if (rank == 0) {
      bulk_g2s(dst, src, 16384, smem_u32(&bar));
    } else if (mode) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(src + 1024), "r"(16384), "r"(bar0) : "memory");
    }
  }
  int ok = 0;
  if (rank == 0 && threadIdx.x == 0) {
    for (long i = 0; i < (1l << 24); ++i)
      if (mbar_test(smem_u32(&bar), 0)) { ok = 1; break; }
    result[0] = ok;
  }
  cluster_sync();
  if (rank == 1 && threadIdx.x == 0 && mode) {
    // CTA 1's data landed in CTA 1's buffer?
    int good = 1;
    for (int i = 0; i < 1024; ++i) good &= buf[i].x == (uint32_t)(1024 + i);
    result[1] = good;
  }
  if (rank == 0 && threadIdx.x == 0) {
    int good = 1;
    for (int i = 0; i < 1024; ++i) good &= buf[i].x == (uint32_t)i;
    result[2] = good;
  }
}
int main() {
  uint4* src; int* res;
  cudaMalloc(&src, 2 * 16384); cudaMalloc(&res, 16);
  uint4 h[2048];
  for (int i = 0; i < 2048; ++i) h[i] = make_uint4(i, 0, 0, 0);
  cudaMemcpy(src, h, sizeof h, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    int r[4] = {-1, -1, -1, -1};
    cudaMemcpy(res, r, 16, cudaMemcpyHostToDevice);
    k<<<2, 32>>>(src, res, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(r, res, 16, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %s | leader barrier completed %d | CTA1 data ok %d | CTA0 data ok %d\n", mode,
           mode ? "CTA 1 copy signals CTA 0's barrier" : "control: leader copy only", cudaGetErrorString(e), r[0], r[1], r[2]);
  }
  return 0;
}
