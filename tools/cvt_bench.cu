// Microbenchmark: per-SM throughput of MUFU.EX2, the e4m3x2 / bf16x2 packing
// conversions (F2FP), and mixes of them, to see which pipe the FP8 softmax's
// P conversion competes for.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/cvt_bench tools/cvt_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void __launch_bounds__(512, 1) bench(unsigned long long* out, float seed, int iters) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed + threadIdx.x * 1e-3f + i * 0.1f;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      if (MODE == 0 || MODE == 3 || MODE == 4) {  // ex2 x2
        float a, b;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(x[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(x[i + 1]));
        x[i] = a * 0.5f; x[i + 1] = b * 0.5f;
      }
      if (MODE == 1 || MODE == 3) {  // e4m3x2 pack
        uint16_t r;
        asm volatile("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(x[i]), "f"(x[i + 1]));
        acc += r;
      }
      if (MODE == 2 || MODE == 4) {  // bf16x2 pack
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[i + 1]));
        acc += r;
      }
      if (MODE == 1 || MODE == 2) { x[i] += 1e-7f; x[i + 1] -= 1e-7f; }
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 0x1234567u) out[1] = acc + __float_as_uint(x[0] + x[3] + x[5] + x[7]);
}

template <int MODE>
void run(const char* name, int warps_per_ops) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int iters = 4096;
  bench<MODE><<<148, 512>>>(d, 0.3f, iters);
  bench<MODE><<<148, 512>>>(d, 0.3f, iters);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  // per SM: 16 warps x 32 threads x iters x 4 pairs
  const double pairs = 16.0 * 32 * iters * 4;
  std::printf("%-24s %8.2f pair-ops/clk/SM   %s\n", name, pairs / h, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("ex2 x2", 0);
  run<1>("e4m3x2 cvt", 0);
  run<2>("bf16x2 cvt", 0);
  run<3>("ex2 x2 + e4m3x2 cvt", 0);
  run<4>("ex2 x2 + bf16x2 cvt", 0);
  return 0;
}
