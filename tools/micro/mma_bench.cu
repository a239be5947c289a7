// tcgen05.mma issue/execute rate for the attention tile shapes (diagnostics).
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2412_03594_b200/csrc/psa_device.cuh"
using namespace psa;

template <int kMode>
__global__ void k(long long* cyc, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tm;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { dev::mbar_init(&bar, 1); dev::fence_mbar_init(); }
  dev::fence_proxy_async_smem();
  if (threadIdx.x < 32) dev::tmem_alloc<512>(&tm);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t t = tm;
  if (threadIdx.x == 0) {
    const uint32_t a0 = dev::smem_u32(base), b0 = dev::smem_u32(base + 32768);
    // modes: 0 SS M128 N64 K16; 1 SS M128 N128; 2 TS M128 N128 (A in TMEM, B MN-major); 3 SS M128 N256
    const uint32_t N = kMode == 0 ? 64 : kMode == 3 ? 256 : 128;
    const uint32_t idesc = dev::umma_idesc_f16(1, 128, N, 0, kMode == 2 ? 1 : 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t kk = it & 7;
      const uint64_t a = dev::umma_desc_sw128(a0 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
      if (kMode == 2) {
        const uint64_t b = dev::umma_desc_sw128(b0 + (kk & 3) * 2048, 8192, 1024);
        dev::mma_f16_ts(t + 256, t + (kk & 3) * 8, b, idesc, 1u);
      } else {
        const uint64_t b = dev::umma_desc_sw128(b0 + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024);
        dev::mma_f16_ss(t, a, b, idesc, 1u);
      }
    }
    long long t1 = clock64();
    dev::mma_commit(&bar);
    dev::mbar_wait(&bar, 0);
    long long t2 = clock64();
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) dev::tmem_dealloc<512>(t);
}

int main() {
  long long* cyc;
  cudaMalloc(&cyc, 16);
  const int iters = 4096;
  const char* names[4] = {"SS M128 N64  K16", "SS M128 N128 K16", "TS M128 N128 K16", "SS M128 N256 K16"};
  auto run = [&](auto kern, int m) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    kern<<<148, 128, 100 * 1024>>>(cyc, iters);
    kern<<<148, 128, 100 * 1024>>>(cyc, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long c[2];
    cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
    const double flop = 2.0 * 128 * (m == 0 ? 64 : m == 3 ? 256 : 128) * 16;
    printf("%s: issue %.1f cyc/instr, complete %.1f cyc/instr (%.0f flop/clk/SM) %s\n", names[m],
           double(c[0]) / iters, double(c[1]) / iters, flop * iters / c[1], cudaGetErrorString(e));
  };
  run(k<0>, 0);
  run(k<1>, 1);
  run(k<2>, 2);
  run(k<3>, 3);
  return 0;
}
