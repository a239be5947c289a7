// Throughput of the SFU exp2 variants on sm_100a (diagnostics for the tile softmax).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

template <int V>
__global__ void k(float* out, int iters, long long* cyc) {
  uint32_t x[8];
  for (int i = 0; i < 8; ++i) x[i] = 0x3c003c00u ^ (threadIdx.x + i);  // 1.0 halves
  float xf[8];
  for (int i = 0; i < 8; ++i) xf[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (V == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(xf[i]));
      if (V == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[i]));
      if (V == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x[i]));
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += xf[i] + __uint_as_float(x[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 8);
  const int iters = 4096;
  const char* names[3] = {"ex2.f32", "ex2.f16x2", "ex2.bf16x2"};
  for (int v = 0; v < 3; ++v) {
    for (int warps = 4; warps <= 16; warps *= 2) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      auto launch = [&]() {
        if (v == 0) k<0><<<148, warps * 32>>>(out, iters, cyc);
        if (v == 1) k<1><<<148, warps * 32>>>(out, iters, cyc);
        if (v == 2) k<2><<<148, warps * 32>>>(out, iters, cyc);
      };
      launch(); cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double ops = double(warps) * 32 * iters * 8;  // instructions x lanes per SM
      printf("%-11s warps/SM %2d: %.2f lane-instr/clk/SM (%.2f elements/clk/SM)\n", names[v], warps,
             ops / c, ops / c * (v ? 2 : 1));
    }
  }
  return 0;
}
