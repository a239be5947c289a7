// Cycles of the tile softmax exp phase (one thread = one 128-column row) in isolation,
// one warp per SMSP (diagnostics for psa_tile2.cuh).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../include/psa.h"
#include "../../paper_2412_03594_b200/csrc/psa_kernel.h"
#include "../../paper_2412_03594_b200/csrc/psa_plan.h"
#include "../../paper_2412_03594_b200/csrc/psa_tile2.cuh"
using namespace psa;
using namespace psa::tile2;

template <int kEmu, int kVariant>
__global__ void k(uint32_t* out, int iters, long long* cyc, float sc, float m) {
  uint32_t r[4][32];
  for (int c = 0; c < 4; ++c)
    for (int e = 0; e < 32; ++e) r[c][e] = __float_as_uint(-0.01f * ((threadIdx.x * 7 + c * 32 + e) % 97));
  float l0 = 0.f, l1 = 0.f;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float nm = -m - 0.001f * it;
    uint32_t pr[4][16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        float x0, x1, y0, y1;
        ffma2(x0, x1, __uint_as_float(r[c][2 * e]), __uint_as_float(r[c][2 * e + 1]), sc, nm);
        if (kEmu > 0 && ((c * 16 + e) % kEmu) == kEmu - 1) {
          exp2_poly2(y0, y1, x0, x1);
        } else {
          y0 = dev::ex2(x0);
          y1 = dev::ex2(x1);
        }
        if (kVariant == 0) fadd2(l0, l1, y0, y1);
        pr[c][e] = pack2<__nv_bfloat16>(y0, y1);
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int e = 0; e < 16; ++e) acc ^= pr[c][e];
    asm volatile("" ::: "memory");
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(l0 + l1);
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 8);
  const int iters = 2000;
  auto run = [&](auto kern, const char* name, int warps) {
    kern<<<148, warps * 32>>>(out, iters, cyc, 0.127f, 1.0f);
    kern<<<148, warps * 32>>>(out, iters, cyc, 0.127f, 1.0f);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s warps/SM %d: %.0f cycles per 128-col row block\n", name, warps, double(c) / iters);
  };
  for (int w : {4, 8}) {
    run(k<4, 0>, "emu every 4 (current)", w);
    run(k<0, 0>, "all MUFU", w);
    run(k<2, 0>, "emu every 2", w);
    run(k<4, 1>, "emu every 4, no row sum", w);
  }
  return 0;
}
