// Prints the thread <-> (TMEM lane, column) mapping of tcgen05.ld.sync.aligned.16x256b
// and .16x128b / .16x64b (one warp, lanes 0-31 of warp 0's quarter) by loading a TMEM
// region filled with value = 1000 * lane + column through the 32x32b shape.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tmem_layout tools/tmem_layout.cu
#include <cuda.h>
#include <cstdio>
#include "../paper_2407_08608_b200/csrc/sm100_ptx.cuh"
using namespace fa3b;

__global__ void k(unsigned* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) ptx::tmem_alloc<512>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    uint32_t v[32];
    for (int c0 = 0; c0 < 64; c0 += 32) {
      for (int i = 0; i < 32; ++i) v[i] = 1000u * lane + c0 + i;
      ptx::tmem_st32(tmem + c0, v);
    }
    ptx::tmem_wait_st();
    uint32_t a[4], b[2], c[1];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]) : "r"(tmem));
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(b[0]), "=r"(b[1]) : "r"(tmem));
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(c[0]) : "r"(tmem));
    uint32_t d[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7])
                 : "r"(tmem + (16u << 16)));
    ptx::tmem_wait_ld();
    for (int i = 0; i < 4; ++i) out[lane * 16 + i] = a[i];
    for (int i = 0; i < 2; ++i) out[lane * 16 + 4 + i] = b[i];
    out[lane * 16 + 6] = c[0];
    for (int i = 0; i < 8; ++i) out[lane * 16 + 8 + i] = d[i];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<512>(tmem);
}

int main() {
  unsigned* d;
  cudaMalloc(&d, 32 * 16 * 4);
  k<<<1, 128>>>(d);
  unsigned h[32 * 16];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  printf("thread: 16x256b.x1 (4 regs) | 16x128b.x1 (2) | 16x64b.x1 (1) | 16x256b.x2 at lane 16 (8)   [value = 1000*lane + col]\n");
  for (int t = 0; t < 32; ++t) {
    printf("%2d:", t);
    for (int i = 0; i < 4; ++i) printf(" %5u", h[t * 16 + i]);
    printf(" |");
    for (int i = 4; i < 6; ++i) printf(" %5u", h[t * 16 + i]);
    printf(" | %5u |", h[t * 16 + 6]);
    for (int i = 8; i < 16; ++i) printf(" %5u", h[t * 16 + i]);
    printf("\n");
  }
}
