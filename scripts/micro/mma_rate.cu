// tcgen05.mma cta_group::2 (M = 256, BF16, both operands SW128 K-major in SMEM) issue-rate microbenchmark:
// one pair per 2 SMs, the leader issues `jobs` jobs of KSTEPS MMAs (K = 16 each) into TMEM, committing
// each job to an mbarrier and keeping at most 2 jobs in flight.  Reports clk per MMA per N.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_25936_b200/csrc -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"
using namespace sand;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1)
    k_rate(int N, int ksteps, int jobs, int ldtm, int cevery, int tcol, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar[0]), 1);
    mbar_init(smem_u32(&bar[1]), 1);
    mbar_init(smem_u32(&bar[2]), 1);
    mbar_init(smem_u32(&bar[3]), 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm + (base - smem_u32(sm)))[i] = 0x3c003c00u ^ (uint32_t)(i * 2654435761u & 0x007f007fu);
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc_cg2(smem_u32(&tslot), 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tm = tslot;
  const uint32_t sA = base, sB = base + 6 * 16384;
  const uint32_t id = idesc_bf16(256, N);
  long long t0 = clock64();
  if (threadIdx.x == 0 && rank == 0) {
    uint32_t ph[2] = {0, 0};
    long long tissue = 0;
    for (int j = 0; j < jobs; ++j) {
      const int s = j & 1;
      if (j >= 2) { mbar_wait(smem_u32(&bar[s]), ph[s]); ph[s] ^= 1u; }
      tc_fence_after();
      const long long ti0 = clock64();
      if (cevery == 200) {
        // tc2-like: A alternates between two 64 KB slot buffers, B rotates over two 32 KB ring stages,
        // accumulator alternates TMEM columns 0 / 256, commit per stage; 16 MMAs (K = 256) per job
        const uint64_t a0 = desc_sw128(sA + (uint32_t)s * 65536u);
        const uint32_t acc = tm + (uint32_t)(s * 256);
#pragma unroll
        for (int st = 0; st < 2; ++st) {
          const uint64_t b0 = desc_sw128(sA + 131072u + (uint32_t)st * 32768u);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            mma_bf16_cg2(acc, a0 + (uint64_t)((st * 2 + (k >> 2)) * (16384 >> 4) + 2 * (k & 3)),
                         b0 + (uint64_t)((k >> 2) * (16384 >> 4) + 2 * (k & 3)), id, (st | k) ? 1u : 0u);
          mma_commit_cg2_mc(smem_u32(&bar[2]), 0x3);
        }
      } else if (cevery == 100) {
        // precomputed descriptors, fully unrolled (22 K-steps: 5 chunks of 4 + 2)
        const uint64_t a0 = desc_sw128(sA), b0 = desc_sw128(sB);
        const uint64_t bstep = (uint64_t)((N / 2) * 128 >> 4);
#pragma unroll
        for (int k = 0; k < 22; ++k) {
          mma_bf16_cg2(tm, a0 + (uint64_t)((k >> 2) * (16384 >> 4) + 2 * (k & 3)), b0 + (uint64_t)(k >> 2) * bstep + 2 * (k & 3),
                       id, k ? 1u : 0u);
          if (tcol == 8 && (k & 7) == 7) mma_commit_cg2_mc(smem_u32(&bar[2]), 0x3);
          if (tcol == 9 && (k & 7) == 7) mma_commit_cg2_mc(smem_u32(&bar[2 + ((k >> 3) & 1)]), 0x3);
        }
      } else {
      for (int k = 0; k < ksteps; ++k) {
        mma_bf16_cg2(tm, desc_sw128(sA + (k >> 2) * 16384 + 32 * (k & 3)),
                     desc_sw128(sB + (k >> 2) * (N / 2) * 128 + 32 * (k & 3)), id, k ? 1u : 0u);
        if (cevery > 0 && (k % cevery) == cevery - 1) mma_commit_cg2_mc(smem_u32(&bar[2]), 0x3);
      }
      }
      tissue += clock64() - ti0;
      mma_commit_cg2_mc(smem_u32(&bar[s]), 0x3);
    }
    for (int s = 0; s < 2; ++s) { mbar_wait(smem_u32(&bar[(jobs + s) & 1]), ph[(jobs + s) & 1]); }
    out[blockIdx.x] = clock64() - t0;
    out[200 + blockIdx.x] = tissue;
  } else if (ldtm == 3 && warp >= 1) {
    // compute-bound competing warps (MUFU + FMA), like the epilogue
    float x = 0.001f * threadIdx.x, y = 0.f;
    for (int i = 0; i < jobs * 40; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) { x = __sinf(x * 1.0001f + 0.1f); y = fmaf(x, 0.5f, y); }
    }
    if (y == 0.12345f) out[1000] = 1;
  } else if (ldtm >= 2 && warp >= 1) {
    // concurrent shared-memory traffic from 15 warps (both CTAs): 2 = 16 B stores, 3 = 16 B loads
    const uint32_t reg = base + 6 * 16384 + 6 * 128 * 128 + (uint32_t)(warp * 512 + (threadIdx.x & 31) * 16);
    uint32_t acc = 0;
    volatile uint32_t* stop = reinterpret_cast<volatile uint32_t*>(&tslot);
    for (int i = 0; i < jobs * 8; ++i) {
      if (ldtm == 2) {
        asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(reg), "r"(i) : "memory");
      } else {
        uint32_t a, b, c, d;
        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(reg) : "memory");
        acc += a ^ d;
      }
    }
    (void)stop;
    if (acc == 0x12345) out[1000] = acc;
  } else if (ldtm == 1 && warp >= 1 && rank == 0) {
    // optional TMEM read traffic concurrent with the MMAs (as an epilogue would do)
    uint32_t r[8], acc = 0;
    const uint32_t tq = tm + ((uint32_t)(32 * (warp & 3)) << 16) + 384;
    for (int i = 0; i < jobs * ksteps * 2; ++i) {
      tmem_ld_16x256b<2>(tq + (i & 7) * 16, r);
      tmem_wait_ld_dep(r);
      acc += r[0] ^ r[7];
    }
    if (acc == 0x12345) out[1000] = acc;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 0) tmem_dealloc_cg2(tm, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 2000 * 8);
  const int smem = 196608 + 1024 + 16 * 512;
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int Ns[] = {128, 192, 256};
  struct Cfg { int N, ldtm, cevery, tcol; };
  const Cfg cfgs[] = {{256, 0, 200, 0}, {256, 3, 200, 0}, {256, 3, 0, 0}};
  for (int rep = 0; rep < 2; ++rep)
  for (const Cfg& c : cfgs) {
      const int N = c.N, ldtm = c.ldtm;
      const int ks = (c.cevery == 200 ? 16 : 22), jobs = 2000;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k_rate<<<148, 512, smem>>>(N, ks, jobs, ldtm, c.cevery, c.tcol, d);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[400];
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      double iss = 0;
      for (int b = 0; b < 148; b += 2) iss += h[200 + b] / 74.0;
      double mx = 0;
      for (int b = 0; b < 148; b += 2) mx = h[b] > mx ? h[b] : mx;
      const double per = mx / ((double)jobs * ks);
      float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
      printf("rep %d N %3d commit-every %3d tmem-col %3d: %.1f clk/MMA (N/2 = %d), issue-loop %.1f, %.3f ms -> %.2f GHz\n", rep, N, c.cevery, c.tcol, per,
             N / 2, iss / ((double)jobs * ks), ms, mx / (ms * 1e6));
  }
  return 0;
}
