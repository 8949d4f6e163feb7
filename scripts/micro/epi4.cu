// Slot-team epilogue throughput on sm_100a: W warps per SMSP (one CTA per SM), each thread one TMEM lane,
// per 32-column batch: [tcgen05.ld 32x32b.x32] 32 x (FMUL.RZ + MUFU.SIN), 16 FFMA2 tail with LDS.128
// broadcast coefficients, 16 F2FP packs, 4 STS.128 into an SW128-like row.  Prints cycles per MUFU per SMSP
// (floor: 8) for each mode.  MODE bits: 1 = sines, 2 = tail, 4 = pack + stores, 8 = TMEM loads,
// 16 = consume the previous batch's sines (software-pipelined by one batch), 32 = pack by integer rounding
// (bits + 0x8000, PRMT) instead of F2FP, 64 = pack to FP16 (cvt.rn.f16x2.f32), 128 = integer pack via IMAD.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2604_25936_b200/csrc/ptx.cuh"
using namespace sand;

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
// odd polynomial sine of z (radians) on the FMA pipe, two lanes at a time: k = rint(z / 2 pi) by the 1.5 2^23
// magic add, r = z - 2 pi k in [-pi, pi], sin r = r P(r^2), degree 7 (|err| < 2.6e-4) or 9 (< 6.2e-6)
template <int DEG>
__device__ __forceinline__ float2 sin_poly2(float2 z) {
  const float2 t = __ffma2_rn(z, make_float2(0.15915494309189535f, 0.15915494309189535f),
                              make_float2(12582912.0f, 12582912.0f));
  const float2 k = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 r = __ffma2_rn(k, make_float2(-6.283185307179586f, -6.283185307179586f), z);
  const float2 r2 = __fmul2_rn(r, r);
  float2 p;
  if (DEG == 9) {
    p = __ffma2_rn(r2, make_float2(2.1478720100276405e-06f, 2.1478720100276405e-06f),
                   make_float2(-0.00019264993898104876f, -0.00019264993898104876f));
    p = __ffma2_rn(p, r2, make_float2(0.008308985270559788f, 0.008308985270559788f));
    p = __ffma2_rn(p, r2, make_float2(-0.16662438213825226f, -0.16662438213825226f));
    p = __ffma2_rn(p, r2, make_float2(0.9999793767929077f, 0.9999793767929077f));
  } else {
    p = __ffma2_rn(r2, make_float2(-0.0001450767886126414f, -0.0001450767886126414f),
                   make_float2(0.007958059199154377f, 0.007958059199154377f));
    p = __ffma2_rn(p, r2, make_float2(-0.16566696763038635f, -0.16566696763038635f));
    p = __ffma2_rn(p, r2, make_float2(0.9992758631706238f, 0.9992758631706238f));
  }
  return __fmul2_rn(p, r);
}
template <int MODE>
__device__ __forceinline__ uint32_t pk2(float lo, float hi) {
  if (MODE & 32) {
    return __byte_perm(__float_as_uint(lo) + 0x8000u, __float_as_uint(hi) + 0x8000u, 0x7632);
  } else if (MODE & 128) {
    uint32_t a, b;
    asm("mad.lo.u32 %0, %1, 1, 32768;" : "=r"(a) : "r"(__float_as_uint(lo)));
    asm("mad.lo.u32 %0, %1, 1, 32768;" : "=r"(b) : "r"(__float_as_uint(hi)));
    return __byte_perm(a, b, 0x7632);
  } else if (MODE & 64) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
  }
  return pack_bf16x2(lo, hi);
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned long long* cyc, float* sink) {
  __shared__ __align__(1024) uint8_t abuf[32 * 1024];
  __shared__ __align__(16) float tab[256];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = 0.001f * i;
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) & 1) * 256;
  const int row = 32 * (warp & 3) + lane;
  const uint32_t a_row = smem_u32(abuf) + (uint32_t)(row >> 3) * 1024 +
                         (uint32_t)(row & 7) * 128;
  const uint32_t rx = row & 7;
  const uint32_t ta = smem_u32(tab);
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(0.01f * (threadIdx.x + i));
  float hp[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) hp[i] = 0.f;
  float2 y0 = make_float2(0.f, 0.f), y1 = make_float2(0.f, 0.f);
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const int cb = (it & 7) * 32;
    if (MODE & 8) {
      tmem_ld32(tm + (uint32_t)cb, r);
      tmem_wait_ld_dep(r);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] ^= (uint32_t)it & 1u;
    }
    float h[32];
    constexpr int NP = (MODE >> 8) & 15;   // polynomial pairs per 16 pairs
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      if ((MODE & 1) && (i / 2) < NP) {
        const float2 hh = sin_poly2<(MODE & 4096) ? 9 : 7>(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])));
        h[i] = hh.x; h[i + 1] = hh.y;
      } else {
        h[i] = (MODE & 1) ? __sinf(__uint_as_float(r[i])) : __uint_as_float(r[i]) * 0.5f;
        h[i + 1] = (MODE & 1) ? __sinf(__uint_as_float(r[i + 1])) : __uint_as_float(r[i + 1]) * 0.5f;
      }
    }
    const float* hc = (MODE & 16) ? hp : h;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      if (MODE & 2) {
        const float4 aa = lds128f(ta + (uint32_t)(cb + 8 * g) * 4);
        const float4 ab = lds128f(ta + (uint32_t)(cb + 8 * g + 4) * 4);
        y0 = __ffma2_rn(make_float2(aa.x, aa.y), make_float2(hc[8 * g + 0], hc[8 * g + 1]), y0);
        y1 = __ffma2_rn(make_float2(aa.z, aa.w), make_float2(hc[8 * g + 2], hc[8 * g + 3]), y1);
        y0 = __ffma2_rn(make_float2(ab.x, ab.y), make_float2(hc[8 * g + 4], hc[8 * g + 5]), y0);
        y1 = __ffma2_rn(make_float2(ab.z, ab.w), make_float2(hc[8 * g + 6], hc[8 * g + 7]), y1);
      }
      if (MODE & 4) {
        const uint32_t kk = (uint32_t)(cb + 8 * g);
        const uint32_t addr = a_row + ((kk >> 6) & 1) * 16384 + ((((kk & 63) >> 3) ^ rx) << 4);
        sts128(addr, pk2<MODE>(hc[8 * g], hc[8 * g + 1]), pk2<MODE>(hc[8 * g + 2], hc[8 * g + 3]),
               pk2<MODE>(hc[8 * g + 4], hc[8 * g + 5]), pk2<MODE>(hc[8 * g + 6], hc[8 * g + 7]));
      }
    }
    if (!(MODE & 2) && !(MODE & 4)) {
#pragma unroll
      for (int i = 0; i < 32; ++i) y0.x += hc[i];
    }
    if (MODE & 16) {
#pragma unroll
      for (int i = 0; i < 32; ++i) hp[i] = h[i];
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (y0.x + y0.y + y1.x + y1.y == 1.2345f) sink[0] = 1.f;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tslot, 512);
}

int main() {
  unsigned long long* c;
  cudaMalloc(&c, 148 * 8);
  float* sink;
  cudaMalloc(&sink, 8);
  unsigned long long h[148];
  const int iters = 4096;
  auto run = [&](auto kern, const char* name, int mode) {
    for (int w : {1, 2, 4}) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
      kern<<<148, 128 * w>>>(iters, c, sink);
      kern<<<148, 128 * w>>>(iters, c, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
      cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int b = 0; b < 148; ++b) mx = h[b] > mx ? h[b] : mx;
      // per SMSP: w warps x iters x 32 sines
      printf("%-28s W=%d  %.2f clk per 32-lane element-instr per SMSP (MUFU floor 8)\n", name, w, mx / (w * iters * 32.0));
    }
    (void)mode;
  };
  run(k<1 | 2 | 4 | 8 | 32 | (2 << 8)>, "poly2 int: full", 0);
  run(k<1 | 2 | 4 | 8 | 32 | (4 << 8)>, "poly4 int: full", 0);
  run(k<1 | 2 | 4 | 8 | 32 | (6 << 8)>, "poly6 int: full", 0);
  run(k<1 | 2 | 4 | 8 | (2 << 8)>, "poly2 f2fp: full", 0);
  run(k<1 | 2 | 4 | 8 | (4 << 8)>, "poly4 f2fp: full", 0);
  run(k<1 | 2 | 4 | 8 | (6 << 8)>, "poly6 f2fp: full", 0);
  run(k<1 | 2 | 4 | 8 | (8 << 8)>, "poly8 f2fp: full", 0);
  run(k<1 | 2 | 4 | 8 | 64 | (4 << 8)>, "poly4 f16pack: full", 0);
  return 0;
}
