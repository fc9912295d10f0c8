// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM, with 4, 8 or
// 16 reading warps, alone or while one thread streams TS-MMAs (A from TMEM) into
// other TMEM columns. Answers whether TMEM reads bound the softmax phases.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tmem_bench tools/tmem_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2407_08608_b200/csrc/sm100_ptx.cuh"

using namespace fa3b;

constexpr int SMEM = 100 * 1024;

template <int WARPS, bool MMA>
__global__ void __launch_bounds__(WARPS * 32 + 32, 1) bench(unsigned long long* out, int iters, int mma_iters) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == WARPS) {  // MMA issuer: TS MMAs, A = TMEM cols [0,64), D = cols [256, 384)
    if (MMA && ptx::elect_one()) {
      const uint32_t idesc = ptx::make_idesc(128, 128, 1, 1, false, true, false);
      const uint32_t b_addr = ptx::smem_u32(smem);
      for (int it = 0; it < mma_iters; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          ptx::mma_f16_ts(tmem + 256, tmem + k * 8, ptx::sw128_desc(b_addr + k * 16 * 128, 16384, 1024), idesc, 1);
      ptx::mma_commit(&bar);
      ptx::mbar_wait(&bar, 0);
    }
  } else {
    // reader warps: lanes 32 (warp % 4), columns [128 + 32 (warp / 4) ...) cycling over 128 columns
    const uint32_t lane_base = static_cast<uint32_t>(32 * (warp & 3)) << 16;
    uint32_t acc = 0;
    __syncwarp();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint32_t r[32];
      ptx::tmem_ld32(tmem + lane_base + 128 + ((it + warp / 4) & 3) * 32, r);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i];
    }
    const long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
    if (acc == 0x12345678u) out[1] = acc;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

template <int WARPS, bool MMA>
void run() {
  auto k = bench<WARPS, MMA>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int iters = 4096;
  k<<<148, WARPS * 32 + 32, SMEM>>>(d, iters, 4096);
  k<<<148, WARPS * 32 + 32, SMEM>>>(d, iters, 4096);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double bytes = static_cast<double>(iters) * WARPS * 32 * 32 * 4;
  std::printf("%2d reader warps %-12s %7.1f cyc per ld.x32 per warp, %6.1f B/clk/SM  %s\n", WARPS,
              MMA ? "+ TS-MMA" : "alone", static_cast<double>(h[0]) / iters, bytes / h[0],
              e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<1, false>();
  run<4, false>();
  run<8, false>();
  run<16, false>();
  run<4, true>();
  run<8, true>();
  run<16, true>();
  return 0;
}
