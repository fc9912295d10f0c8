// Microbenchmark: tcgen05.mma issue rate per SM for the operand placements the
// backward kernel can choose between (A from shared memory vs TMEM, N = 64 /
// 128 / 256, K-major vs MN-major operands), optionally with other warps
// streaming STS traffic into shared memory at the same time.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench tools/mma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2407_08608_b200/csrc/sm100_ptx.cuh"

using namespace fa3b;

constexpr int SMEM = 200 * 1024;

template <int N, bool TS, bool MN, bool STS>
__global__ void __launch_bounds__(256, 1) bench(unsigned long long* out, int iters) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
    done = 0;
  }
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  // A: 128 rows x 128 B (16 KB), B: N rows x 128 B at +64 KB; STS scratch at +128 KB
  const uint32_t a_addr = ptx::smem_u32(smem);
  const uint32_t b_addr = ptx::smem_u32(smem + 65536);
  const uint32_t idesc = ptx::make_idesc(128, N, 1, 1, MN && !TS, MN, false);
  if (warp == 0) {
    if (ptx::elect_one()) {
      const long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t off = MN ? k * 16 * 128 : k * 32;
          const uint32_t lbo = MN ? 16384 : 16;
          const uint64_t bd = ptx::sw128_desc(b_addr + off, lbo, 1024);
          if (TS)
            ptx::mma_f16_ts(tmem + 256, tmem + k * 8, bd, idesc, 1);
          else
            ptx::mma_f16_ss(tmem + 256, ptx::sw128_desc(a_addr + off, lbo, 1024), bd, idesc, 1);
        }
      }
      ptx::mma_commit(&bar);
      ptx::mbar_wait(&bar, 0);
      const long long t1 = clock64();
      done = 1;
      if (blockIdx.x == 0) out[0] = t1 - t0;
    }
  } else if (STS && warp >= 4) {
    // 4 warps of 16-byte stores into a private 16 KB region until the MMAs finish
    uint4* dst = reinterpret_cast<uint4*>(smem + 131072) + (threadIdx.x - 128);
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    long long n = 0;
    while (!done) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[i * 128] = v;
      v.x += 1;
      n += 8;
    }
    if (blockIdx.x == 0 && threadIdx.x == 128) out[1] = n;
  }
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

template <int N, bool TS, bool MN, bool STS>
void run(const char* name) {
  auto k = bench<N, TS, MN, STS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  const int iters = 2048;
  k<<<148, 256, SMEM>>>(d, iters);
  k<<<148, 256, SMEM>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double mmas = iters * 4.0;
  const double cyc = h[0] / mmas;
  const double flop_clk = 2.0 * 128 * N * 16 / cyc;
  std::printf("%-28s N=%3d  %6.1f cyc/mma (ideal %5.1f)  %6.0f FLOP/clk/SM  sts_bytes/clk=%.1f  %s\n", name, N,
              cyc, 128.0 * N / 256.0, flop_clk, STS ? h[1] * 16.0 * 128 / h[0] : 0.0,
              e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<64, false, false, false>("SS K-major");
  run<128, false, false, false>("SS K-major");
  run<256, false, false, false>("SS K-major");
  run<64, true, false, false>("TS (A in TMEM)");
  run<128, true, false, false>("TS (A in TMEM)");
  run<256, true, false, false>("TS (A in TMEM)");
  run<64, false, true, false>("SS MN-major");
  run<128, false, true, false>("SS MN-major");
  run<256, false, true, false>("SS MN-major");
  run<64, true, true, false>("TS, B MN-major");
  run<128, true, true, false>("TS, B MN-major");
  run<64, false, false, true>("SS K-major + STS");
  run<128, false, false, true>("SS K-major + STS");
  run<64, true, false, true>("TS + STS");
  run<128, true, false, true>("TS + STS");
  return 0;
}
