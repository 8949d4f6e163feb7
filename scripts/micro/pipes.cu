// Throughput of the epilogue's instruction classes on sm_100a: 16 warps / SM (4 per SMSP), 8 independent
// chains per thread, cycles per warp-instruction per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#define N 8
template <int OP>
__global__ void __launch_bounds__(512, 1) k(int iters, float s, unsigned long long* cyc, float* sink) {
  float2 v[N]; uint32_t u[N];
#pragma unroll
  for (int i = 0; i < N; ++i) { v[i] = make_float2(0.001f * (threadIdx.x + i), 0.002f * i); u[i] = threadIdx.x * 7 + i; }
  const float2 S = make_float2(s, s * 0.5f), B = make_float2(0.25f, -0.125f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (OP == 0) v[i].x = fmaf(v[i].x, v[i].y, B.x);                      // FFMA 3 reg (y varies)
      if (OP == 1) v[i].x = fmaf(v[i].x, 0.999f, 0.0001f);                  // FFMA imm
      if (OP == 2) v[i] = __ffma2_rn(v[i], S, B);                            // FFMA2 (uniform operands)
      if (OP == 3) v[i] = __ffma2_rn(v[i], v[(i + 1) % N], v[i]);            // FFMA2 3 reg
      if (OP == 4) v[i] = __fmul2_rn(v[i], S);                               // FMUL2
      if (OP == 5) { float r; asm volatile("sin.approx.f32 %0, %1;" : "=f"(r) : "f"(v[i].x)); v[i].x = r; }  // FMUL.RZ + MUFU
      if (OP == 6) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i].x), "f"(v[i].y)); u[i] ^= r; v[i].x += 1.0f; }  // F2FP (+FADD)
      if (OP == 7) { __half2 h = *reinterpret_cast<__half2*>(&u[i]); h = __hfma2(h, h, h); u[i] = *reinterpret_cast<uint32_t*>(&h); }  // HFMA2 3 reg
      if (OP == 8) v[i].x = v[i].x * 0.999f;                                 // FMUL imm
      if (OP == 9) v[i] = __fadd2_rn(v[i], B);                               // FADD2
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float acc = 0; for (int i = 0; i < N; ++i) acc += v[i].x + v[i].y + (float)u[i];
  if (acc == 1.2345f) sink[0] = acc;
}
int main() {
  unsigned long long* c; cudaMalloc(&c, 148 * 8); float* sink; cudaMalloc(&sink, 8);
  unsigned long long h[148];
  const int iters = 4096;
  const char* names[] = {"FFMA r", "FFMA imm", "FFMA2 uni", "FFMA2 r", "FMUL2 uni", "sin(FMUL.RZ+MUFU)", "F2FP+FADD", "HFMA2 r", "FMUL imm", "FADD2 uni"};
  auto run = [&](auto kern, int op) {
    kern<<<148, 512>>>(iters, 1.0001f, c, sink); cudaDeviceSynchronize();
    kern<<<148, 512>>>(iters, 1.0001f, c, sink);
    cudaError_t e = cudaDeviceSynchronize(); if (e) { printf("%s\n", cudaGetErrorString(e)); return; }
    cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    // per SMSP: 4 warps x iters x N instructions
    printf("%-20s %.2f clk per warp-instr per SMSP\n", names[op], (double)h[0] / (4.0 * iters * N));
  };
  run(k<0>, 0); run(k<1>, 1); run(k<2>, 2); run(k<3>, 3); run(k<4>, 4); run(k<5>, 5); run(k<6>, 6); run(k<7>, 7); run(k<8>, 8); run(k<9>, 9);
  return 0;
}
