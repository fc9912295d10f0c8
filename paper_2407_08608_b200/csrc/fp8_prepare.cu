// K5: incoherent processing + e4m3 quantization of one [B, N, H, d] tensor.
//
// Reference: preprocess_incoherent (core/src/fp8_attention.cpp:33-42) ->
// DHTransform::apply = sign flip then normalized FWHT (core/src/hadamard.cpp:11-33)
// with signs from sample_sign_vector (core/src/rng.cpp:73-78); then
// quantize_per_block / quantize_per_tensor (core/src/quantize.cpp:10-60):
// scale = amax / 448 (1 if amax == 0), code = round_to(x * (1 / scale), e4m3)
// (core/src/formats.cpp:45-61, RNE, saturating).
//
// The arithmetic is FP64 with the reference's rounding points (the butterfly
// sums of 16-bit or fp32 inputs are exact in FP64, so their order is free), so
// codes and scales are byte-identical to the reference for the same input
// values (tests/test_fp8_gpu.py). Algorithmic traffic: 2-4 bytes read and 1
// byte written per element.
//
// bf16 input in 128-row blocks (the FP8 forward's case) takes the fast path
// below: d <= 128 one thread per row (fa3b_fp8_prepare_row_kernel), d = 256 the
// lane-split kernel over a TMA ring (fa3b_fp8_prepare_fast_kernel). Otherwise:
// Layout (see Quad): 4 lanes per row at d <= 128 (8 at d = 256), each holding
// d / 4 (d / 8) contiguous elements, so all but the last two (three) butterfly
// stages run in registers; vector loads and stores. 128-row blocks at
// d <= 128 keep the whole transformed block in registers across the amax
// (one read of the input); d = 256 and other block sizes (per tensor) take two
// passes that recompute the transform (the second read hits L2), split over an
// 8-CTA cluster when there are too few blocks to fill the GPU.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstddef>
#include <cstdlib>

#include "../../include/fa3b.h"
#include "fa3b_internal.cuh"
#include "sm100_ptx.cuh"

namespace fa3b {
namespace {

// round_to(x, e4m3) of formats.cpp:45-61 (quantum of the clamped binade,
// ties to even, saturate or NaN past 448), done exactly on the FP64 bits:
// with e = floor(log2|x|) >= -6, k = rint(|x| 2^(3-e)) in [8, 16] is the
// significand in eighths and code = ((e + 7) << 3) + k - 8 (k = 16 carries
// into the exponent); below 2^-6 the quantum is 2^-9 and code = rint(|x| 512).
__device__ __forceinline__ uint8_t e4m3_code(double x, bool saturate) {
  if (isnan(x)) return 0x7F;
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
  const uint8_t sign = (bits >> 63) ? 0x80 : 0x00;
  const double ax = fabs(x);
  int code;
  if (ax < 0.015625) {
    code = __double2int_rn(ax * 512.0);
  } else {
    const int e = static_cast<int>((bits >> 52) & 0x7FF) - 1023;
    if (e > 8) {
      code = 0x7F;  // beyond every finite code
    } else {
      const double up = __longlong_as_double(static_cast<long long>(1023 + 3 - e) << 52);
      code = ((e + 7) << 3) + __double2int_rn(ax * up) - 8;
    }
  }
  if (code > 0x7E) code = saturate ? 0x7E : 0x7F;
  return sign | static_cast<uint8_t>(code);
}

struct PrepArgs {
  const void* src;
  long long s_sb, s_ss, s_sh;
  int src_dtype;
  uint8_t* dst;
  long long d_sb, d_ss, d_sh;
  float* scales;
  int N, H, block_rows, nblk, hadamard, saturate, pow2;
  unsigned long long signs[4];  // bit i set -> sign_i = +1
};

// scale = amax / 448 (1 if amax == 0), quantize.cpp:41-42,54-55; with pow2 the
// smallest power of two >= that value (fa3b_fp8_prepare_params.scale_pow2)
__device__ __forceinline__ double block_scale(const PrepArgs& a, double amax) {
  double scale = amax == 0.0 ? 1.0 : amax / 448.0;
  if (a.pow2) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(scale));
    if (u & 0x000FFFFFFFFFFFFFull)
      scale = __longlong_as_double(static_cast<long long>((u & 0x7FF0000000000000ull) + (1ull << 52)));
  }
  return scale;
}
__device__ __forceinline__ void write_scale(const PrepArgs& a, int b, int h, int blk, double amax,
                                            bool bad) {
  const double scale = block_scale(a, amax);
  // non-finite inputs: the reference throws; the device reports a NaN scale
  a.scales[(static_cast<size_t>(b) * a.H + h) * a.nblk + blk] =
      bad ? __int_as_float(0x7fc00000) : static_cast<float>(scale);
}

// Control flow around the butterflies is kept warp-uniform by construction
// (trip counts from blockIdx / kernel arguments only, row validity applied to
// the loads and stores): shuffles under a thread-dependent branch compile to
// WARPSYNC collectives that cost more than the arithmetic.

// Quad layout: LPR lanes per row (4 at d <= 128, 8 at d = 256). Lane l owns row
// l / LPR of its warp's group and the elements [Q (l % LPR), Q (l % LPR) + Q),
// Q = d / LPR (16 or 32), so log2(Q) butterfly stages run in registers and only
// log2(LPR) cross lanes (64-bit shuffles within the lane group).
template <int D>
struct Quad {
  static constexpr int LPR = D <= 128 ? 4 : 8;
  static constexpr int Q = D / LPR;
  static constexpr int RPW = 32 / LPR;  // rows per warp
};

template <int D>
__device__ __forceinline__ void quad_load(const PrepArgs& a, int b, int h, int row, bool valid, int qd,
                                          double (&v)[Quad<D>::Q]) {
  constexpr int Q = Quad<D>::Q;
  const size_t base = b * a.s_sb + static_cast<size_t>(row) * a.s_ss + h * a.s_sh + qd * Q;
  if (a.src_dtype == FA3B_DTYPE_F32) {
    uint4 raw[Q / 4];
#pragma unroll
    for (int k = 0; k < Q / 4; ++k)
      raw[k] = valid ? __ldg(reinterpret_cast<const uint4*>(static_cast<const float*>(a.src) + base) + k)
                     : make_uint4(0, 0, 0, 0);
    const uint32_t* u = reinterpret_cast<const uint32_t*>(raw);
#pragma unroll
    for (int e = 0; e < Q; ++e) v[e] = __uint_as_float(u[e]);
  } else {
    uint4 raw[Q / 8];
#pragma unroll
    for (int k = 0; k < Q / 8; ++k)
      raw[k] = valid ? __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(a.src) + base) + k)
                     : make_uint4(0, 0, 0, 0);
    const uint32_t* u = reinterpret_cast<const uint32_t*>(raw);
#pragma unroll
    for (int e = 0; e < Q; ++e) {
      const uint16_t bits = static_cast<uint16_t>(u[e >> 1] >> (16 * (e & 1)));
      v[e] = a.src_dtype == FA3B_DTYPE_BF16 ? __uint_as_float(static_cast<uint32_t>(bits) << 16)
                                            : __half2float(__ushort_as_half(bits));
    }
  }
}

template <int D>
__device__ __forceinline__ void quad_transform(const PrepArgs& a, int qd, double (&v)[Quad<D>::Q]) {
  constexpr int Q = Quad<D>::Q, LPR = Quad<D>::LPR;
  if (!a.hadamard) return;
  // sign_i = +1 iff bit i of the sign mask is set (elements qd Q .. qd Q + Q - 1)
  const uint32_t sm = static_cast<uint32_t>(a.signs[(qd * Q) >> 6] >> ((qd * Q) & 63));
#pragma unroll
  for (int e = 0; e < Q; ++e)
    if (!((sm >> e) & 1u)) v[e] = -v[e];
#pragma unroll
  for (int len = 1; len < Q; len <<= 1) {
#pragma unroll
    for (int e = 0; e < Q; ++e) {
      if ((e & len) == 0) {
        const double p = v[e], q = v[e + len];
        v[e] = p + q;
        v[e + len] = p - q;
      }
    }
  }
#pragma unroll
  for (int m = 1; m < LPR; m <<= 1) {  // stages len = Q, 2Q, ...: partners within the lane group
    const double sgn = (qd & m) ? -1.0 : 1.0;
#pragma unroll
    for (int e = 0; e < Q; ++e) {
      const double other = __shfl_xor_sync(0xffffffffu, v[e], m);
      v[e] = fma(sgn, v[e], other);  // exact product: equals a + b / b - a of the reference
    }
  }
  const double norm = 1.0 / sqrt(static_cast<double>(D));
#pragma unroll
  for (int e = 0; e < Q; ++e) v[e] *= norm;
}

template <int D>
__device__ __forceinline__ void quad_store(const PrepArgs& a, int b, int h, int row, int qd,
                                           const double (&v)[Quad<D>::Q], double inv) {
  constexpr int Q = Quad<D>::Q;
  uint32_t packed[Q / 4];
  if (a.saturate) {
#pragma unroll
    for (int e = 0; e < Q; e += 4) {
      float f[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // FP64 -> FP32 round-to-odd, then hardware RNE to e4m3
        const double t = v[e + u] * inv;
        float z = __double2float_rz(t);
        if (static_cast<double>(z) != t) z = __uint_as_float(__float_as_uint(z) | 1u);
        f[u] = z;
      }
      packed[e >> 2] = ptx::pack_e4m3x4_merge(f[0], f[1], f[2], f[3]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < Q; e += 4)
      packed[e >> 2] = e4m3_code(v[e] * inv, false) | (e4m3_code(v[e + 1] * inv, false) << 8) |
                       (e4m3_code(v[e + 2] * inv, false) << 16) |
                       (static_cast<uint32_t>(e4m3_code(v[e + 3] * inv, false)) << 24);
  }
  uint4* dst = reinterpret_cast<uint4*>(a.dst + b * a.d_sb + static_cast<size_t>(row) * a.d_ss + h * a.d_sh +
                                        qd * Q);
#pragma unroll
  for (int k = 0; k < Q / 16; ++k)
    dst[k] = make_uint4(packed[4 * k], packed[4 * k + 1], packed[4 * k + 2], packed[4 * k + 3]);
}

// 128-row blocks, d = 64 / 128: the 16 warps of quad-layout rows hold the whole
// transformed block in registers across the amax (one read of the input).
// Persistent (one CTA per SM walking (block, head, batch) items) with the next
// item's rows streaming into shared memory by cp.async while the current one is
// transformed: a CTA needs all 120 registers of 512 threads, so without the
// prefetch every block's load latency sat exposed in front of its FP64 work.
template <int D, int ESZ>
__global__ void __launch_bounds__(512, 1) fa3b_fp8_prepare_quad_kernel(const PrepArgs a, int items) {
  using QD = Quad<D>;
  constexpr int Q = QD::Q;
  constexpr int NV = Q * ESZ / 16;  // 16-byte vectors per thread and block
  extern __shared__ uint4 stage[];  // [2 stages][NV][512 threads]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, qd = lane % QD::LPR;
  const int rloc = warp * QD::RPW + lane / QD::LPR;
  __shared__ double s_amax[2][16];
  __shared__ int s_bad[2][16];
  auto coords = [&](int item, int& blk, int& h, int& b) {
    blk = item % a.nblk;
    const int hb = item / a.nblk;
    h = hb % a.H;
    b = hb / a.H;
  };
  auto prefetch = [&](int item, int st) {
    if (item < items) {
      int blk, h, b;
      coords(item, blk, h, b);
      const int row = blk * 128 + rloc;
      const bool valid = row < a.N;
      const char* src = static_cast<const char*>(a.src) +
                        (b * a.s_sb + static_cast<long long>(valid ? row : 0) * a.s_ss + h * a.s_sh + qd * Q) * ESZ;
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const uint32_t dst = ptx::smem_u32(&stage[(st * NV + k) * 512 + threadIdx.x]);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src + 16 * k),
                     "r"(valid ? 16 : 0)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int st = 0;
  prefetch(blockIdx.x, 0);
  for (int item = blockIdx.x, it = 0; item < items; item += gridDim.x, ++it, st ^= 1) {
    prefetch(item + gridDim.x, st ^ 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    int blk, h, b;
    coords(item, blk, h, b);
    const int row = blk * 128 + rloc;
    double v[Q];
    {
      uint4 raw[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) raw[k] = stage[(st * NV + k) * 512 + threadIdx.x];
      const uint32_t* u = reinterpret_cast<const uint32_t*>(raw);
#pragma unroll
      for (int e = 0; e < Q; ++e) {
        if constexpr (ESZ == 4) {
          v[e] = __uint_as_float(u[e]);
        } else {
          const uint16_t bits = static_cast<uint16_t>(u[e >> 1] >> (16 * (e & 1)));
          v[e] = a.src_dtype == FA3B_DTYPE_BF16 ? __uint_as_float(static_cast<uint32_t>(bits) << 16)
                                                : __half2float(__ushort_as_half(bits));
        }
      }
    }
    quad_transform<D>(a, qd, v);
    double amax = 0.0;
    bool bad = false;
#pragma unroll
    for (int e = 0; e < Q; ++e) {
      const double x = fabs(v[e]);
      bad |= !isfinite(x);
      amax = fmax(amax, x);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    bad = __any_sync(0xffffffffu, bad);
    const int sb = it & 1;  // two reduction buffers: the next item's writes cannot race these reads
    if (lane == 0) {
      s_amax[sb][warp] = amax;
      s_bad[sb][warp] = bad;
    }
    __syncthreads();
    amax = s_amax[sb][0];
    bad = s_bad[sb][0];
#pragma unroll
    for (int w = 1; w < 16; ++w) {
      amax = fmax(amax, s_amax[sb][w]);
      bad |= s_bad[sb][w] != 0;
    }
    if (threadIdx.x == 0) write_scale(a, b, h, blk, amax, bad);
    const double inv = 1.0 / block_scale(a, amax);  // quantize.cpp:25
    if (row < a.N) quad_store<D>(a, b, h, row, qd, v, inv);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ double ld_cluster_f64(const double* p, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(ptx::smem_u32(p)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
  return v;
}

// Any block size (0 = the whole tensor) and d = 256: two passes over the rows
// (the second recomputes the transform; its reads hit L1/L2). A block is split
// over a cluster of C CTAs whose partial maxima meet through distributed shared
// memory, so even one scale per (batch, head) keeps C x B x H CTAs busy.
template <int D, int C>
__global__ void __launch_bounds__(256) fa3b_fp8_prepare_kernel(const PrepArgs a) {
  using QD = Quad<D>;
  constexpr int WARPS = 8, ROWS = WARPS * QD::RPW;  // rows per CTA iteration
  const int blk = blockIdx.x / C, part = blockIdx.x % C, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, qd = lane % QD::LPR;
  const int rb0 = a.block_rows ? blk * a.block_rows : 0;
  const int rb1 = a.block_rows ? min(a.N, rb0 + a.block_rows) : a.N;
  const int chunk = (rb1 - rb0 + C - 1) / C;
  const int c0 = rb0 + part * chunk, c1 = min(rb1, c0 + chunk);
  const int iters = c1 > c0 ? (c1 - c0 + ROWS - 1) / ROWS : 0;
  const int rsub = warp * QD::RPW + lane / QD::LPR;
  __shared__ double s_amax[WARPS];
  __shared__ int s_bad[WARPS];
  __shared__ double s_cta[2];  // this CTA's (amax, bad) for the cluster
  double amax = 0.0;
  bool bad = false;
  for (int it = 0; it < iters; ++it) {
    const int row = c0 + it * ROWS + rsub;
    double v[QD::Q];
    quad_load<D>(a, b, h, row, row < c1, qd, v);
    quad_transform<D>(a, qd, v);
#pragma unroll
    for (int e = 0; e < QD::Q; ++e) {
      const double x = fabs(v[e]);
      bad |= !isfinite(x);
      amax = fmax(amax, x);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    s_amax[warp] = amax;
    s_bad[warp] = bad;
  }
  __syncthreads();
  amax = s_amax[0];
  bad = s_bad[0];
#pragma unroll
  for (int w = 1; w < WARPS; ++w) {
    amax = fmax(amax, s_amax[w]);
    bad |= s_bad[w] != 0;
  }
  if constexpr (C > 1) {
    if (threadIdx.x == 0) {
      s_cta[0] = amax;
      s_cta[1] = bad ? 1.0 : 0.0;
    }
    cluster_sync();
#pragma unroll
    for (int r = 0; r < C; ++r) {
      amax = fmax(amax, ld_cluster_f64(&s_cta[0], r));
      bad |= ld_cluster_f64(&s_cta[1], r) != 0.0;
    }
    cluster_sync();  // keep every CTA's shared memory alive until all have read it
  }
  if (threadIdx.x == 0 && (C == 1 || cluster_rank() == 0)) write_scale(a, b, h, blk, amax, bad);
  const double inv = 1.0 / block_scale(a, amax);
  for (int it = 0; it < iters; ++it) {
    const int row = c0 + it * ROWS + rsub;
    double v[QD::Q];
    quad_load<D>(a, b, h, row, row < c1, qd, v);
    quad_transform<D>(a, qd, v);
    if (row < c1) quad_store<D>(a, b, h, row, qd, v, inv);
  }
}

template <int D, int C>
cudaError_t launch_two_pass(const PrepArgs& a, dim3 grid, cudaStream_t st) {
  auto kern = fa3b_fp8_prepare_kernel<D, C>;
  grid.x *= C;
  if constexpr (C == 1) {
    kern<<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
  }
}

template <int D>
cudaError_t launch_generic(const PrepArgs& a, dim3 grid, cudaStream_t st) {
  // split each scale block over a cluster when there are too few blocks to fill 148 SMs
  const long long ctas = static_cast<long long>(grid.x) * grid.y * grid.z;
  const int rows = a.block_rows ? a.block_rows : a.N;
  if (ctas < 296 && rows >= 8 * 256) return launch_two_pass<D, 8>(a, grid, st);
  return launch_two_pass<D, 1>(a, grid, st);
}

// ---------------------------------------------------------------- fast path
// bf16 input, 128-row blocks, saturating encode (the FP8 forward's case). The
// same codes and scales as the FP64 kernels above, at a fraction of the work:
//
// * Transform in exact int32 arithmetic. A bf16 value is (128 + m) 2^(E - 134);
//   scaled by 2^k (k = 157 - log2 d - E_max of the row) every entry of a row
//   whose exponents span at most 23 - log2 d binades is an integer below
//   2^(31 - log2 d), so FMUL by 2^k and F2I are exact and the int32 butterflies
//   cannot overflow: the integer FWHT equals the reference's FP64 sums exactly
//   (those sums are exact in FP64 too, so the order of additions is free).
// * amax: max |S| per row is exact (ldexp of an integer), so amax =
//   RN64(max|S| * norm) = max |RN64(S * norm)| is the reference's value bit for
//   bit, and scale / inv follow with the reference's FP64 operations.
// * Encode: t = RN64(RN64(S * norm) * inv) is approximated in FP32 by
//   I2F(I) * RN32(2^-k * norm * inv) (relative error < 3.01 * 2^-24). The code is
//   taken when the e4m3 conversions of t32 (1 -/+ 6 * 2^-24) agree (RNE is
//   monotone, so every value in between, the exact t included, has that code);
//   otherwise (~1e-5 of the entries) t is recomputed exactly in FP64.
// * Rows outside the int32 range (exponent spread, zeros mixed with non-zeros,
//   subnormals, non-finite values) are done by the whole warp in FP64 with the
//   reference's operation order (fast_row_fp64), one row at a time.
// Without the Hadamard (V) the FP32 encode of the exact bf16 value is used
// directly. One CTA per 128-row block; lane group of LPR lanes per row, each
// lane Q = 32 (d = 64: 16) contiguous elements.
template <int D>
struct Fast {
  static constexpr int Q = D == 64 ? 16 : 32;
  static constexpr int LPR = D / Q;           // 4, 4, 8
  static constexpr int RPW = 32 / LPR;        // rows per warp
  static constexpr int THREADS = 128 * LPR;   // 512, 512, 1024
  static constexpr int WARPS = THREADS / 32;
  static constexpr int LOGD = D == 64 ? 6 : (D == 128 ? 7 : 8);
  static constexpr int SPREAD = 23 - LOGD;    // binades an int32 row may span
  // TMA ring: a 128-row block of bf16 as D / 64 boxes of 128 rows x 128 bytes
  // (128-byte swizzle), STAGES blocks in flight per CTA
  static constexpr int CPS = THREADS == 512 ? 2 : 1;  // CTAs per SM
  static constexpr int STAGES = D == 64 ? 4 : 3;
  static constexpr int BOX_BYTES = 128 * 128;
  static constexpr int STAGE_BYTES = 128 * D * 2;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024;  // + alignment slack
};

__device__ __forceinline__ uint32_t vmax_u16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t vmin_u16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ double pow2d(int e) {  // 2^e, |e| <= 1022
  return __longlong_as_double(static_cast<long long>(1023 + e) << 52);
}
// saturating RNE e4m3 code of an FP64 value: FP64 -> FP32 round-to-odd, then the
// hardware RNE (24 >= 4 + 2 bits, so the double rounding is exact)
__device__ __forceinline__ uint32_t e4m3_sat(double t) {
  float z = __double2float_rz(t);
  if (static_cast<double>(z) != t) z = __uint_as_float(__float_as_uint(z) | 1u);
  return ptx::pack_e4m3x4_merge(z, 0.f, 0.f, 0.f) & 0xFFu;
}

// One row by the whole warp in FP64 (lane l holds entries [l M, l M + M)), the
// reference's FWHT order: len = 1, 2, ... with (a + b, a - b) (hadamard.cpp:11-33).
template <int D, bool HAD>
__device__ __forceinline__ void fast_row_fp64(const PrepArgs& a, int b, int h, int row, int lane,
                                              double (&s)[D / 32]) {
  constexpr int M = D / 32;
  const uint16_t* src = static_cast<const uint16_t*>(a.src) + b * a.s_sb +
                        static_cast<size_t>(row) * a.s_ss + h * a.s_sh + lane * M;
  uint16_t v16[M];
  if constexpr (M == 2) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(src);
    v16[0] = u & 0xFFFF; v16[1] = u >> 16;
  } else if constexpr (M == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(src);
    v16[0] = u.x & 0xFFFF; v16[1] = u.x >> 16; v16[2] = u.y & 0xFFFF; v16[3] = u.y >> 16;
  } else {
    const uint4 u = *reinterpret_cast<const uint4*>(src);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) { v16[2 * i] = w[i] & 0xFFFF; v16[2 * i + 1] = w[i] >> 16; }
  }
#pragma unroll
  for (int e = 0; e < M; ++e) s[e] = __uint_as_float(static_cast<uint32_t>(v16[e]) << 16);
  if constexpr (HAD) {
#pragma unroll
    for (int e = 0; e < M; ++e) {
      const int i = lane * M + e;
      if (!((a.signs[i >> 6] >> (i & 63)) & 1ull)) s[e] = -s[e];
    }
#pragma unroll
    for (int len = 1; len < M; len <<= 1)
#pragma unroll
      for (int e = 0; e < M; ++e)
        if ((e & len) == 0) {
          const double p = s[e], q = s[e + len];
          s[e] = p + q;
          s[e + len] = p - q;
        }
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const double sgn = (lane & m) ? -1.0 : 1.0;
#pragma unroll
      for (int e = 0; e < M; ++e) s[e] = fma(sgn, s[e], __shfl_xor_sync(0xffffffffu, s[e], m));
    }
  }
}

// Persistent CTAs (TMA = true, grid = min(blocks, CPS x SMs)) walk the 128-row
// blocks c, c + G, ... (blocks of one head are consecutive); the TMA ring keeps
// the next STAGES - 1 blocks loading while this one is transformed, so the
// block's barriers no longer leave the SM without loads in flight. TMA = false
// is the earlier one-CTA-per-block kernel with direct vector loads (grid = blocks;
// measured and not kept: a persistent variant streaming through cp.async into an
// unswizzled ring, and an L2 prefetch of the next wave, r02i_prep.log, r02l_prep.log).
template <int D, bool HAD, bool TMA>
__global__ void __launch_bounds__(Fast<D>::THREADS, Fast<D>::CPS)
    fa3b_fp8_prepare_fast_kernel(const __grid_constant__ CUtensorMap tm, const PrepArgs a,
                                 const int items) {
  using F = Fast<D>;
  constexpr int Q = F::Q, LPR = F::LPR, NP = Q / 2;
  // t32 = RN(I2F(I) * RN(c kLo|Hi)) brackets the exact RN64(RN64(S norm) inv):
  // relative error of I2F(I) * c is < 3.01 u, the bracket adds 2 u of rounding
  constexpr float kLo = 1.f - 8.f / 16777216.f, kHi = 1.f + 8.f / 16777216.f;
  __shared__ __align__(16) uint32_t s_mask[LPR * NP];  // sign flips per bf16 pair
  __shared__ double s_red[F::WARPS];
  __shared__ int s_bad[F::WARPS];
  __shared__ double s_bc[2];
  __shared__ __align__(8) uint64_t s_full[F::STAGES];
  extern __shared__ uint8_t k5_dyn[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(k5_dyn) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, qd = lane % LPR;
  const int rl = warp * F::RPW + lane / LPR;  // row within the block
  const double norm = HAD ? 1.0 / sqrt(static_cast<double>(D)) : 1.0;
  const int G = static_cast<int>(gridDim.x);
  auto issue = [&](int stage, int it) {  // one elected thread: block `it` -> ring stage
    const int hb = it / a.nblk;
    ptx::mbar_arrive_expect_tx(&s_full[stage], F::STAGE_BYTES);
#pragma unroll
    for (int bx = 0; bx < D / 64; ++bx)
      ptx::tma_load_4d(ring + stage * F::STAGE_BYTES + bx * F::BOX_BYTES, &tm, &s_full[stage], bx * 64,
                       hb % a.H, (it % a.nblk) * 128, hb / a.H, ptx::kEvictFirst);
  };
  if constexpr (HAD) {
    for (int i = tid; i < LPR * NP; i += F::THREADS) {
      const int e0 = (i / NP) * Q + 2 * (i % NP), e1 = e0 + 1;
      const bool f0 = !((a.signs[e0 >> 6] >> (e0 & 63)) & 1ull);
      const bool f1 = !((a.signs[e1 >> 6] >> (e1 & 63)) & 1ull);
      s_mask[i] = (f0 ? 0x8000u : 0u) | (f1 ? 0x80000000u : 0u);
    }
  }
  if constexpr (TMA) {
    if (tid == 0) {
      ptx::prefetch_tmap(&tm);
      for (int st = 0; st < F::STAGES; ++st) ptx::mbar_init(&s_full[st], 1);
      ptx::fence_mbar_init();
      for (int st = 0; st < F::STAGES; ++st)
        if (static_cast<int>(blockIdx.x) + st * G < items) issue(st, blockIdx.x + st * G);
    }
  }
  if constexpr (HAD || TMA) __syncthreads();  // s_mask, barrier init
  int n = 0;
  for (int it = blockIdx.x; it < items; it += G, ++n) {
  const int blk = it % a.nblk, h = (it / a.nblk) % a.H, b = it / a.nblk / a.H;
  const int row = blk * 128 + rl;
  const bool valid = row < a.N;
  uint32_t w[NP];
  if constexpr (TMA) {
    // rows past N arrive as zeros; chunk c (16 bytes) of row rl sits in box c / 8 at
    // swizzled position (c % 8) ^ (rl % 8): 4 lanes per bank group, no conflicts
    const int stage = n % F::STAGES;
    ptx::mbar_wait(&s_full[stage], (n / F::STAGES) & 1);
    const uint8_t* sb = ring + stage * F::STAGE_BYTES + rl * 128;
#pragma unroll
    for (int k = 0; k < Q / 8; ++k) {
      const int c = qd * (Q / 8) + k;
      const uint4 v = *reinterpret_cast<const uint4*>(sb + (c >> 3) * F::BOX_BYTES + (((c & 7) ^ (rl & 7)) << 4));
      w[4 * k] = v.x; w[4 * k + 1] = v.y; w[4 * k + 2] = v.z; w[4 * k + 3] = v.w;
    }
  } else {
    const uint4* src = reinterpret_cast<const uint4*>(
        static_cast<const uint16_t*>(a.src) + b * a.s_sb + static_cast<size_t>(valid ? row : 0) * a.s_ss +
        h * a.s_sh + qd * Q);
#pragma unroll
    for (int k = 0; k < Q / 8; ++k) {
      const uint4 v = valid ? __ldg(src + k) : make_uint4(0, 0, 0, 0);
      w[4 * k] = v.x; w[4 * k + 1] = v.y; w[4 * k + 2] = v.z; w[4 * k + 3] = v.w;
    }
  }
  if constexpr (HAD) {
    const uint4* mk = reinterpret_cast<const uint4*>(s_mask + qd * NP);
#pragma unroll
    for (int k = 0; k < NP / 4; ++k) {
      const uint4 m = mk[k];
      w[4 * k] ^= m.x; w[4 * k + 1] ^= m.y; w[4 * k + 2] ^= m.z; w[4 * k + 3] ^= m.w;
    }
  }
  // exponent range of the row (16-bit magnitudes compare like the values)
  uint32_t mx = 0, mn = 0xFFFFFFFFu;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const uint32_t m = w[p] & 0x7FFF7FFFu;
    mx = vmax_u16x2(mx, m);
    mn = vmin_u16x2(mn, m);
  }
  uint32_t mx16 = max(mx & 0xFFFFu, mx >> 16), mn16 = min(mn & 0xFFFFu, mn >> 16);
#pragma unroll
  for (int o = 1; o < LPR; o <<= 1) {
    mx16 = max(mx16, __shfl_xor_sync(0xffffffffu, mx16, o));
    mn16 = min(mn16, __shfl_xor_sync(0xffffffffu, mn16, o));
  }
  const int emax = static_cast<int>(mx16 >> 7), emin = static_cast<int>(mn16 >> 7);
  const bool allzero = mx16 == 0;
  const int k = 157 - F::LOGD - emax;
  const bool fast = HAD ? (allzero || (emax <= 254 && emin >= 1 && emin >= emax - F::SPREAD && k <= 127))
                        : emax <= 254;
  // ---- transform (fast rows; other rows compute garbage that is never used)
  int I[HAD ? Q : 1];
  double rowS = 0.0;  // max |S| of this row (exact)
  if constexpr (HAD) {
    const float fs = (fast && !allzero) ? __uint_as_float(static_cast<uint32_t>(k + 127) << 23) : 0.f;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const float2 x = __fmul2_rn(make_float2(__uint_as_float(w[p] << 16), __uint_as_float(w[p] & 0xFFFF0000u)),
                                  make_float2(fs, fs));
      I[2 * p] = __float2int_rn(x.x);
      I[2 * p + 1] = __float2int_rn(x.y);
    }
#pragma unroll
    for (int len = 1; len < Q; len <<= 1)
#pragma unroll
      for (int e = 0; e < Q; ++e)
        if ((e & len) == 0) {
          const int p = I[e], q = I[e + len];
          I[e] = p + q;
          I[e + len] = p - q;
        }
#pragma unroll
    for (int m = 1; m < LPR; m <<= 1) {
      // lower lane a + b, upper lane a - b = other - mine: one IMAD with sgn = +-1
      // (written as PTX mad: the compiler would otherwise select between I and -I)
      const int sgn = (qd & m) ? -1 : 1;
#pragma unroll
      for (int e = 0; e < Q; ++e) {
        const int other = __shfl_xor_sync(0xffffffffu, I[e], m);
        asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(I[e]) : "r"(I[e]), "r"(sgn), "r"(other));
      }
    }
    int hi_i = I[0], lo_i = I[0];
#pragma unroll
    for (int e = 1; e + 1 < Q; e += 2) {
      hi_i = max(hi_i, max(I[e], I[e + 1]));
      lo_i = min(lo_i, min(I[e], I[e + 1]));
    }
    hi_i = max(hi_i, I[Q - 1]);
    lo_i = min(lo_i, I[Q - 1]);
    int rm = max(hi_i, -lo_i);  // |I| < 2^31: no overflow
#pragma unroll
    for (int o = 1; o < LPR; o <<= 1) rm = max(rm, __shfl_xor_sync(0xffffffffu, rm, o));
    rowS = fast ? static_cast<double>(rm) * pow2d(-k) : 0.0;
  } else {
    rowS = static_cast<double>(__uint_as_float(mx16 << 16));  // exact max |x| (finite rows)
  }
  // ---- rows outside the fast range: the whole warp, one row at a time, in FP64
  bool bad = false;
  const uint32_t slow_rows = __ballot_sync(0xffffffffu, !fast && valid && qd == 0);
  for (uint32_t sr = slow_rows; sr != 0; sr &= sr - 1) {
    const int src_lane = __ffs(sr) - 1;
    const int r = blk * 128 + warp * F::RPW + src_lane / LPR;
    double s[D / 32];
    fast_row_fp64<D, HAD>(a, b, h, r, lane, s);
    double m = 0.0;
    bool nf = false;
#pragma unroll
    for (int e = 0; e < D / 32; ++e) {
      nf |= !isfinite(s[e]);
      m = fmax(m, fabs(s[e]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    nf = __any_sync(0xffffffffu, nf);
    if (lane / LPR == src_lane / LPR) {
      rowS = m;
      bad |= nf;
    }
  }
  // ---- block amax, scale = amax / 448, inv = 1 / scale (quantize.cpp:25,55)
  double v = rowS;
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    s_red[warp] = v;
    s_bad[warp] = bad;
  }
  __syncthreads();  // also: every thread has read this block's ring stage
  if (tid == 0) {
    if constexpr (TMA)
      if (it + F::STAGES * G < items) issue(n % F::STAGES, it + F::STAGES * G);
    double m = s_red[0];
    int bd = s_bad[0];
#pragma unroll
    for (int i = 1; i < F::WARPS; ++i) {
      m = fmax(m, s_red[i]);
      bd |= s_bad[i];
    }
    const double amax = m * norm;
    write_scale(a, b, h, blk, amax, bd != 0);
    const double inv = 1.0 / block_scale(a, amax);
    s_bc[0] = inv;
    s_bc[1] = norm * inv;
  }
  __syncthreads();
  const double inv = s_bc[0];
  // ---- encode
  uint8_t* dst_row = a.dst + b * a.d_sb + static_cast<size_t>(row) * a.d_ss + h * a.d_sh;
  if (fast && valid) {
    float c;
    if constexpr (HAD)
      c = allzero ? 0.f : static_cast<float>(s_bc[1] * pow2d(-k));
    else
      c = inv < 1e38 ? static_cast<float>(inv) : 0.f;
    const bool huge = !HAD && !(inv < 1e38);  // c would overflow FP32: encode exactly
    // t32 * (1 -/+ 8 u) in one FMUL2 per entry: (x, x) * (c kLo, c kHi)
    const float2 cc = make_float2(c * kLo, c * kHi);
    uint32_t packed[Q / 4];
    uint32_t miss = 0;  // groups of 4 whose bracket straddles an e4m3 rounding boundary
#pragma unroll
    for (int g = 0; g < Q / 4; ++g) {
      float2 t[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float x;
        if constexpr (HAD) {
          x = static_cast<float>(I[4 * g + i]);
        } else {
          const uint32_t wp = w[2 * g + (i >> 1)];
          x = __uint_as_float((i & 1) ? (wp & 0xFFFF0000u) : (wp << 16));
        }
        t[i] = __fmul2_rn(cc, make_float2(x, x));
      }
      const uint32_t lo = ptx::pack_e4m3x4_merge(t[0].x, t[1].x, t[2].x, t[3].x);
      const uint32_t hi = ptx::pack_e4m3x4_merge(t[0].y, t[1].y, t[2].y, t[3].y);
      packed[g] = lo;
      miss |= static_cast<uint32_t>(lo != hi) << g;
    }
    if (huge) miss = ~0u;
    if (miss != 0) {  // ~1e-5 of the entries: the exact FP64 encode for those groups
#pragma unroll
      for (int g = 0; g < Q / 4; ++g) {
        if (!((miss >> g) & 1u)) continue;
        uint32_t code = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double td;
          if constexpr (HAD) {
            td = (static_cast<double>(I[4 * g + i]) * pow2d(-k) * norm) * inv;
          } else {
            const uint32_t wp = w[2 * g + (i >> 1)];
            td = static_cast<double>(__uint_as_float((i & 1) ? (wp & 0xFFFF0000u) : (wp << 16))) * inv;
          }
          code |= e4m3_sat(td) << (8 * i);
        }
        packed[g] = code;
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(dst_row + qd * Q);
#pragma unroll
    for (int k2 = 0; k2 < Q / 16; ++k2)
      dst[k2] = make_uint4(packed[4 * k2], packed[4 * k2 + 1], packed[4 * k2 + 2], packed[4 * k2 + 3]);
  }
  for (uint32_t sr = slow_rows; sr != 0; sr &= sr - 1) {
    const int src_lane = __ffs(sr) - 1;
    const int r = blk * 128 + warp * F::RPW + src_lane / LPR;
    double s[D / 32];
    fast_row_fp64<D, HAD>(a, b, h, r, lane, s);
    uint32_t cw[(D / 32 + 3) / 4] = {};
#pragma unroll
    for (int e = 0; e < D / 32; ++e) cw[e >> 2] |= e4m3_sat((s[e] * norm) * inv) << (8 * (e & 3));
    uint8_t* drow = a.dst + b * a.d_sb + static_cast<size_t>(r) * a.d_ss + h * a.d_sh + lane * (D / 32);
    if constexpr (D / 32 == 2)
      *reinterpret_cast<uint16_t*>(drow) = static_cast<uint16_t>(cw[0]);
    else if constexpr (D / 32 == 4)
      *reinterpret_cast<uint32_t*>(drow) = cw[0];
    else
      *reinterpret_cast<uint2*>(drow) = make_uint2(cw[0], cw[1]);
  }
  }  // blocks of this CTA
}

// Rare paths of the row kernel kept out of line (one copy instead of one per
// unrolled group, which would overflow the instruction cache).
__device__ __noinline__ uint32_t e4m3_group_int(int i0, int i1, int i2, int i3, double pk, double norm,
                                                double inv) {
  const int v[4] = {i0, i1, i2, i3};
  uint32_t code = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) code |= e4m3_sat((static_cast<double>(v[i]) * pk * norm) * inv) << (8 * i);
  return code;
}
__device__ __noinline__ uint32_t e4m3_group_bf16(uint32_t w0, uint32_t w1, double inv) {
  const float x[4] = {__uint_as_float(w0 << 16), __uint_as_float(w0 & 0xFFFF0000u), __uint_as_float(w1 << 16),
                      __uint_as_float(w1 & 0xFFFF0000u)};
  uint32_t code = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) code |= e4m3_sat(static_cast<double>(x[i]) * inv) << (8 * i);
  return code;
}

// Row-per-thread variant of the fast path (d <= 128; FA3B_K5_ROW, default on):
// one CTA of 128 threads per 128-row block, thread r owns row r whole, so the
// FWHT runs entirely in registers (log2 d stages of IADD pairs, no shuffles), the
// block's amax barrier spans 4 warps, and 3-4 CTAs per SM overlap one block's
// TMA load with the others' arithmetic. Same arithmetic as the lane-split kernel
// above: exact int32 transform, FP32 bracketed encode, FP64 rows and groups.
#ifndef FA3B_K5_ISM
#define FA3B_K5_ISM 0
#endif
template <int D, int LPR>
struct RowK {
  static constexpr int LOGD = D == 64 ? 6 : (D == 128 ? 7 : 8);
  static constexpr int SPREAD = 23 - LOGD;
  static constexpr int Q = D / LPR;        // elements per thread
  static constexpr int THREADS = 128 * LPR;
  static constexpr int WARPS = THREADS / 32;
  static constexpr int RPW = 32 / LPR;     // rows per warp
  static constexpr int MINB = THREADS == 512 ? 1 : (Q == 64 ? (LPR == 1 ? 4 : 2) : (THREADS == 256 ? 1 : 3));  // CTAs per SM (registers)
  static constexpr int BOX_BYTES = 128 * 128;
  static constexpr int TILE_BYTES = 128 * D * 2;
  // ISM (with the Hadamard): the transformed int32 row goes to shared memory
  // (half over the thread's own, consumed, tile row, half into a second tile-sized
  // buffer) and the encode runs as a rolled loop over it: one copy of the encode
  // code instead of Q / 16 (d128: 3640 -> 2888 instructions). Measured 10-20 %
  // slower (the second tile-sized buffer costs occupancy; r02bj_prep.log): off
  static constexpr bool ISM = FA3B_K5_ISM != 0;
  static constexpr int SMEM = (ISM ? 2 : 1) * TILE_BYTES + 1024;
};

// One CTA per block (measured: persistent CTAs with a TMA ring of the next tiles
// were 10-30 % slower than letting the block scheduler refill SMs, r02as_prep.log).
template <int D, int LPR, bool HAD>
__global__ void __launch_bounds__(RowK<D, LPR>::THREADS, RowK<D, LPR>::MINB)
    fa3b_fp8_prepare_row_kernel(const __grid_constant__ CUtensorMap tm, const PrepArgs a) {
  using R = RowK<D, LPR>;
  constexpr int Q = R::Q, NP = Q / 2, NC = Q / 8;  // per thread: elements, bf16 pairs, 16-byte chunks
  constexpr float kLo = 1.f - 8.f / 16777216.f, kHi = 1.f + 8.f / 16777216.f;
  __shared__ __align__(16) uint32_t s_mask[D / 2];
  __shared__ double s_red[R::WARPS];
  __shared__ int s_bad[R::WARPS];
  __shared__ double s_bc[2];
  __shared__ __align__(8) uint64_t s_full;
  extern __shared__ uint8_t k5r_dyn[];
  uint8_t* tile = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(k5r_dyn) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rl = tid / LPR, part = tid % LPR;  // row within the block, element range of the row
  const int blk = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int row = blk * 128 + rl;
  const bool valid = row < a.N;
  const double norm = HAD ? 1.0 / sqrt(static_cast<double>(D)) : 1.0;
  if (tid == 0) {
    ptx::mbar_init(&s_full, 1);
    ptx::fence_mbar_init();
    ptx::mbar_arrive_expect_tx(&s_full, R::TILE_BYTES);
#pragma unroll
    for (int bx = 0; bx < D / 64; ++bx)
      ptx::tma_load_4d(tile + bx * R::BOX_BYTES, &tm, &s_full, bx * 64, h, blk * 128, b, ptx::kEvictFirst);
  }
  if constexpr (HAD) {
    for (int i = tid; i < D / 2; i += R::THREADS) {
      const int e0 = 2 * i, e1 = e0 + 1;
      const bool f0 = !((a.signs[e0 >> 6] >> (e0 & 63)) & 1ull);
      const bool f1 = !((a.signs[e1 >> 6] >> (e1 & 63)) & 1ull);
      s_mask[i] = (f0 ? 0x8000u : 0u) | (f1 ? 0x80000000u : 0u);
    }
  }
  __syncthreads();  // barrier init, s_mask
  ptx::mbar_wait(&s_full, 0);
  // chunk c of the row: box c / 8, swizzled slot (c % 8) ^ (row % 8); rows past N are 0
  const uint8_t* trow = tile + rl * 128;
  auto chunk = [&](int c) {
    const int cc = part * NC + c;
    return *reinterpret_cast<const uint4*>(trow + (cc >> 3) * R::BOX_BYTES + (((cc & 7) ^ (rl & 7)) << 4));
  };
  // exponent range of the row (16-bit magnitudes compare like the values)
  uint32_t mx = 0, mn = 0xFFFFFFFFu;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const uint4 v = chunk(c);
    const uint32_t q[4] = {v.x & 0x7FFF7FFFu, v.y & 0x7FFF7FFFu, v.z & 0x7FFF7FFFu, v.w & 0x7FFF7FFFu};
    mx = vmax_u16x2(mx, vmax_u16x2(vmax_u16x2(q[0], q[1]), vmax_u16x2(q[2], q[3])));
    mn = vmin_u16x2(mn, vmin_u16x2(vmin_u16x2(q[0], q[1]), vmin_u16x2(q[2], q[3])));
  }
  uint32_t mx16 = max(mx & 0xFFFFu, mx >> 16), mn16 = min(mn & 0xFFFFu, mn >> 16);
#pragma unroll
  for (int o = 1; o < LPR; o <<= 1) {
    mx16 = max(mx16, __shfl_xor_sync(0xffffffffu, mx16, o));
    mn16 = min(mn16, __shfl_xor_sync(0xffffffffu, mn16, o));
  }
  const int emax = static_cast<int>(mx16 >> 7), emin = static_cast<int>(mn16 >> 7);
  const bool allzero = mx16 == 0;
  const int k = 157 - R::LOGD - emax;
  const bool fast = HAD ? (allzero || (emax <= 254 && emin >= 1 && emin >= emax - R::SPREAD && k <= 127))
                        : emax <= 254;
  int I[HAD ? Q : 1];
  double rowS = 0.0;
  if constexpr (HAD) {
    const float fs = (fast && !allzero) ? __uint_as_float(static_cast<uint32_t>(k + 127) << 23) : 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const uint4 v = chunk(c);
      const uint4 m = *reinterpret_cast<const uint4*>(s_mask + part * NP + 4 * c);
      const uint32_t wv[4] = {v.x ^ m.x, v.y ^ m.y, v.z ^ m.z, v.w ^ m.w};
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const float2 x = __fmul2_rn(
            make_float2(__uint_as_float(wv[p] << 16), __uint_as_float(wv[p] & 0xFFFF0000u)), make_float2(fs, fs));
        I[8 * c + 2 * p] = __float2int_rn(x.x);
        I[8 * c + 2 * p + 1] = __float2int_rn(x.y);
      }
    }
#pragma unroll
    for (int len = 1; len < Q; len <<= 1)
#pragma unroll
      for (int e = 0; e < Q; ++e)
        if ((e & len) == 0) {
          const int p = I[e], q = I[e + len];
          I[e] = p + q;
          I[e + len] = p - q;
        }
#pragma unroll
    for (int m = 1; m < LPR; m <<= 1) {
      // lower part a + b, upper part a - b = other - mine: one IMAD with sgn = +-1
      const int sgn = (part & m) ? -1 : 1;
#pragma unroll
      for (int e = 0; e < Q; ++e) {
        const int other = __shfl_xor_sync(0xffffffffu, I[e], m);
        asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(I[e]) : "r"(I[e]), "r"(sgn), "r"(other));
      }
    }
    int hi_i = I[0], lo_i = I[0];
#pragma unroll
    for (int e = 1; e + 1 < Q; e += 2) {
      hi_i = max(hi_i, max(I[e], I[e + 1]));
      lo_i = min(lo_i, min(I[e], I[e + 1]));
    }
    hi_i = max(hi_i, I[Q - 1]);
    lo_i = min(lo_i, I[Q - 1]);
    int rm = max(hi_i, -lo_i);
#pragma unroll
    for (int o = 1; o < LPR; o <<= 1) rm = max(rm, __shfl_xor_sync(0xffffffffu, rm, o));
    rowS = fast ? static_cast<double>(rm) * pow2d(-k) : 0.0;
    if constexpr (R::ISM) {
      // int chunk c (4 values): chunks [0, NC) over this thread's own tile chunks
      // (read above, not needed again), [NC, 2 NC) at the same places one tile on
#pragma unroll
      for (int c = 0; c < Q / 4; ++c) {
        const int cc = part * NC + (c % NC);
        *reinterpret_cast<uint4*>(const_cast<uint8_t*>(trow) + (c / NC) * R::TILE_BYTES +
                                  (cc >> 3) * R::BOX_BYTES + (((cc & 7) ^ (rl & 7)) << 4)) =
            make_uint4(I[4 * c], I[4 * c + 1], I[4 * c + 2], I[4 * c + 3]);
      }
    }
  } else {
    rowS = static_cast<double>(__uint_as_float(mx16 << 16));
  }
  // rows outside the fast range: the whole warp, one row at a time, in FP64
  bool bad = false;
  const uint32_t slow_rows = __ballot_sync(0xffffffffu, !fast && valid && part == 0);
  for (uint32_t sr = slow_rows; sr != 0; sr &= sr - 1) {
    const int src_lane = __ffs(sr) - 1;
    double sv[D / 32];
    fast_row_fp64<D, HAD>(a, b, h, blk * 128 + warp * R::RPW + src_lane / LPR, lane, sv);
    double m = 0.0;
    bool nf = false;
#pragma unroll
    for (int e = 0; e < D / 32; ++e) {
      nf |= !isfinite(sv[e]);
      m = fmax(m, fabs(sv[e]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    nf = __any_sync(0xffffffffu, nf);
    if (lane / LPR == src_lane / LPR) {
      rowS = m;
      bad = nf;
    }
  }
  // block amax, scale = amax / 448, inv = 1 / scale (quantize.cpp:25,55)
  double v = rowS;
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    s_red[warp] = v;
    s_bad[warp] = bad;
  }
  __syncthreads();
  if (tid == 0) {
    double m = s_red[0];
    int bd = s_bad[0];
#pragma unroll
    for (int i = 1; i < R::WARPS; ++i) {
      m = fmax(m, s_red[i]);
      bd |= s_bad[i];
    }
    const double amax = m * norm;
    write_scale(a, b, h, blk, amax, bd != 0);
    const double inv = 1.0 / block_scale(a, amax);
    s_bc[0] = inv;
    s_bc[1] = norm * inv;
  }
  __syncthreads();
  const double inv = s_bc[0];
  uint8_t* dst_row = a.dst + b * a.d_sb + static_cast<size_t>(row) * a.d_ss + h * a.d_sh + part * Q;
  if (fast && valid) {
    float c;
    if constexpr (HAD)
      c = allzero ? 0.f : static_cast<float>(s_bc[1] * pow2d(-k));
    else
      c = inv < 1e38 ? static_cast<float>(inv) : 0.f;
    const bool huge = !HAD && !(inv < 1e38);
    const float2 cc = make_float2(c * kLo, c * kHi);
    if constexpr (HAD && R::ISM) {
      // 16 codes per iteration from the staged int32 row, one copy of the code
#pragma unroll 1
      for (int s16 = 0; s16 < Q / 16; ++s16) {
        int J[16];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int c = 4 * s16 + q4, cc2 = part * NC + (c % NC);
          const uint4 u = *reinterpret_cast<const uint4*>(trow + (c / NC) * R::TILE_BYTES + (cc2 >> 3) * R::BOX_BYTES +
                                                          (((cc2 & 7) ^ (rl & 7)) << 4));
          J[4 * q4] = static_cast<int>(u.x); J[4 * q4 + 1] = static_cast<int>(u.y);
          J[4 * q4 + 2] = static_cast<int>(u.z); J[4 * q4 + 3] = static_cast<int>(u.w);
        }
        uint32_t packed[4];
        uint32_t miss = 0;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float2 t[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float x = static_cast<float>(J[4 * g + i]);
            t[i] = __fmul2_rn(cc, make_float2(x, x));
          }
          const uint32_t lo = ptx::pack_e4m3x4_merge(t[0].x, t[1].x, t[2].x, t[3].x);
          const uint32_t hi = ptx::pack_e4m3x4_merge(t[0].y, t[1].y, t[2].y, t[3].y);
          packed[g] = lo;
          miss |= static_cast<uint32_t>(lo != hi) << g;
        }
        if (miss != 0) {
#pragma unroll
          for (int g = 0; g < 4; ++g)
            if ((miss >> g) & 1u)
              packed[g] = e4m3_group_int(J[4 * g], J[4 * g + 1], J[4 * g + 2], J[4 * g + 3], pow2d(-k), norm, inv);
        }
        reinterpret_cast<uint4*>(dst_row)[s16] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      }
    } else
    // 16 codes (one 16-byte store) at a time
#pragma unroll
    for (int s16 = 0; s16 < Q / 16; ++s16) {
      uint32_t packed[4];
      uint32_t miss = 0;
      uint4 raw[2];
      if constexpr (!HAD) {
        raw[0] = chunk(2 * s16);
        raw[1] = chunk(2 * s16 + 1);
      }
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float2 t[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float x;
          if constexpr (HAD) {
            x = static_cast<float>(I[16 * s16 + 4 * g + i]);
          } else {
            const uint32_t* rw = reinterpret_cast<const uint32_t*>(raw);
            const uint32_t wp = rw[2 * g + (i >> 1)];
            x = __uint_as_float((i & 1) ? (wp & 0xFFFF0000u) : (wp << 16));
          }
          t[i] = __fmul2_rn(cc, make_float2(x, x));
        }
        const uint32_t lo = ptx::pack_e4m3x4_merge(t[0].x, t[1].x, t[2].x, t[3].x);
        const uint32_t hi = ptx::pack_e4m3x4_merge(t[0].y, t[1].y, t[2].y, t[3].y);
        packed[g] = lo;
        miss |= static_cast<uint32_t>(lo != hi) << g;
      }
      if (huge) miss = 0xFu;
      if (miss != 0) {  // rare: the exact FP64 encode for those groups
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          if (!((miss >> g) & 1u)) continue;
          if constexpr (HAD) {
            const int* ig = I + 16 * s16 + 4 * g;
            packed[g] = e4m3_group_int(ig[0], ig[1], ig[2], ig[3], pow2d(-k), norm, inv);
          } else {
            const uint32_t* rw = reinterpret_cast<const uint32_t*>(raw);
            packed[g] = e4m3_group_bf16(rw[2 * g], rw[2 * g + 1], inv);
          }
        }
      }
      reinterpret_cast<uint4*>(dst_row)[s16] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    }
  }
  for (uint32_t sr = slow_rows; sr != 0; sr &= sr - 1) {
    const int src_lane = __ffs(sr) - 1;
    const int r = blk * 128 + warp * R::RPW + src_lane / LPR;
    double sv[D / 32];
    fast_row_fp64<D, HAD>(a, b, h, r, lane, sv);
    uint32_t cw[(D / 32 + 3) / 4] = {};
#pragma unroll
    for (int e = 0; e < D / 32; ++e) cw[e >> 2] |= e4m3_sat((sv[e] * norm) * inv) << (8 * (e & 3));
    uint8_t* drow = a.dst + b * a.d_sb + static_cast<size_t>(r) * a.d_ss + h * a.d_sh + lane * (D / 32);
    if constexpr (D / 32 == 2)
      *reinterpret_cast<uint16_t*>(drow) = static_cast<uint16_t>(cw[0]);
    else if constexpr (D / 32 == 4)
      *reinterpret_cast<uint32_t*>(drow) = cw[0];
    else
      *reinterpret_cast<uint2*>(drow) = make_uint2(cw[0], cw[1]);
  }
}

uint64_t mix64(uint64_t z) {  // rng.cpp:15-19
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace
}  // namespace fa3b

using namespace fa3b;

extern "C" int fa3b_fp8_prepare(const fa3b_fp8_prepare_params* pp) {
  g_last_launch_count = 0;
  if (pp == nullptr) return FA3B_ERR_NULL;
  // ABI 1 callers pass the struct without scale_pow2
  if (pp->struct_size != sizeof(fa3b_fp8_prepare_params) &&
      pp->struct_size != offsetof(fa3b_fp8_prepare_params, scale_pow2))
    return FA3B_ERR_STRUCT;
  const auto& p = *pp;
  if (p.batch <= 0 || p.heads <= 0 || p.seqlen <= 0 || p.head_dim <= 0) return FA3B_ERR_EMPTY;
  if (p.hadamard && (p.head_dim & (p.head_dim - 1))) return FA3B_ERR_NOT_POW2;
  if (p.head_dim != 64 && p.head_dim != 128 && p.head_dim != 256) return FA3B_ERR_HEAD_DIM;
  if (p.block_rows < 0) return FA3B_ERR_TILE;
  if (!p.src.ptr || !p.dst.ptr || !p.scales) return FA3B_ERR_NULL;
  if (p.src_dtype != FA3B_DTYPE_BF16 && p.src_dtype != FA3B_DTYPE_F16 && p.src_dtype != FA3B_DTYPE_F32)
    return FA3B_ERR_DTYPE;
  const int sb = p.src_dtype == FA3B_DTYPE_F32 ? 4 : 2;
  if (!strides_ok(p.src, sb, p.batch, p.seqlen, p.heads) || !strides_ok(p.dst, 1, p.batch, p.seqlen, p.heads))
    return FA3B_ERR_ALIGNMENT;
  if (const int rc = check_device(); rc != FA3B_OK) return rc;  // sm_100 current device
  PrepArgs a{};
  a.src = p.src.ptr;
  a.s_sb = p.src.stride_batch;
  a.s_ss = p.src.stride_seq;
  a.s_sh = p.src.stride_head;
  a.src_dtype = p.src_dtype;
  a.dst = static_cast<uint8_t*>(p.dst.ptr);
  a.d_sb = p.dst.stride_batch;
  a.d_ss = p.dst.stride_seq;
  a.d_sh = p.dst.stride_head;
  a.scales = p.scales;
  a.N = p.seqlen;
  a.H = p.heads;
  a.block_rows = p.block_rows;
  a.nblk = p.block_rows ? (p.seqlen + p.block_rows - 1) / p.block_rows : 1;
  a.hadamard = p.hadamard;
  a.saturate = p.saturate;
  a.pow2 = p.struct_size == sizeof(fa3b_fp8_prepare_params) && p.scale_pow2 != 0;
  // sample_sign_vector(d, seed): sign_i = +1 iff word(i) = mix64(seed + (i+1) gamma) is odd
  for (int i = 0; i < p.head_dim; ++i)
    if (mix64(p.seed + static_cast<uint64_t>(i + 1) * 0x9E3779B97F4A7C15ull) & 1ull)
      a.signs[i >> 6] |= 1ull << (i & 63);
  dim3 grid(a.nblk, p.heads, p.batch);
  cudaStream_t st = static_cast<cudaStream_t>(p.stream);
  cudaError_t e = cudaSuccess;
  static const bool fast_env = [] {
    const char* e = std::getenv("FA3B_K5_FAST");
    return e == nullptr || std::atoi(e) != 0;
  }();
  if (fast_env && p.block_rows == 128 && p.src_dtype == FA3B_DTYPE_BF16 && p.saturate) {
    static const bool tma_env = [] {
      const char* e = std::getenv("FA3B_K5_TMA");
      return e == nullptr || std::atoi(e) != 0;
    }();
    const int items = a.nblk * p.heads * p.batch;
    CUtensorMap tm{};
    if (tma_env) {
      const int rc = make_tmap_4d(&tm, p.src, 2, p.head_dim, p.heads, p.seqlen, p.batch, 64, 128);
      if (rc != FA3B_OK) return rc;
    }
    auto go = [&](auto tma_kern, auto direct_kern, int threads, int smem, int cps) {
      if (!tma_env) {
        direct_kern<<<items, threads, 0, st>>>(tm, a, items);
        return cudaGetLastError();
      }
      const int rc = ensure_smem_attr(reinterpret_cast<const void*>(tma_kern), smem);
      if (rc != FA3B_OK) return cudaErrorInvalidValue;
      const int grid = items < cps * num_sms() ? items : cps * num_sms();
      tma_kern<<<grid, threads, smem, st>>>(tm, a, items);
      return cudaGetLastError();
    };
#define FA3B_K5_GO(D, HAD) \
  go(fa3b_fp8_prepare_fast_kernel<D, HAD, true>, fa3b_fp8_prepare_fast_kernel<D, HAD, false>, \
     Fast<D>::THREADS, Fast<D>::SMEM, Fast<D>::CPS)
    static const bool row_env = [] {
      const char* e = std::getenv("FA3B_K5_ROW");
      return e == nullptr || std::atoi(e) != 0;
    }();
    auto go_row = [&](auto kern, int threads, int smem, int mb) {
      const int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
      if (rc != FA3B_OK) return cudaErrorInvalidValue;
      (void)mb;
      kern<<<grid, threads, smem, st>>>(tm, a);
      return cudaGetLastError();
    };
    if (row_env && !tma_env) {
      const int rc = make_tmap_4d(&tm, p.src, 2, p.head_dim, p.heads, p.seqlen, p.batch, 64, 128);
      if (rc != FA3B_OK) return rc;
    }
    static const int row_lpr = [] {  // lanes per row at d = 128 (A/B: FA3B_K5_LPR=1|2)
      const char* e = std::getenv("FA3B_K5_LPR");
      return e != nullptr && std::atoi(e) == 2 ? 2 : 1;
    }();
    static const int row_lpr256 = [] {  // d = 256: 0 = lane-split TMA-ring kernel, else lanes per row
      const char* e = std::getenv("FA3B_K5_LPR256");
      return e != nullptr ? std::atoi(e) : 2;
    }();
    if (row_env && p.head_dim == 64) {
      e = p.hadamard ? go_row(fa3b_fp8_prepare_row_kernel<64, 1, true>, RowK<64, 1>::THREADS, RowK<64, 1>::SMEM, RowK<64, 1>::MINB)
                     : go_row(fa3b_fp8_prepare_row_kernel<64, 1, false>, RowK<64, 1>::THREADS, RowK<64, 1>::SMEM, RowK<64, 1>::MINB);
    } else if (row_env && p.head_dim == 128 && row_lpr == 1) {
      e = p.hadamard ? go_row(fa3b_fp8_prepare_row_kernel<128, 1, true>, RowK<128, 1>::THREADS, RowK<128, 1>::SMEM, RowK<128, 1>::MINB)
                     : go_row(fa3b_fp8_prepare_row_kernel<128, 1, false>, RowK<128, 1>::THREADS, RowK<128, 1>::SMEM, RowK<128, 1>::MINB);
    } else if (row_env && p.head_dim == 128) {
      e = p.hadamard ? go_row(fa3b_fp8_prepare_row_kernel<128, 2, true>, RowK<128, 2>::THREADS, RowK<128, 2>::SMEM, RowK<128, 2>::MINB)
                     : go_row(fa3b_fp8_prepare_row_kernel<128, 2, false>, RowK<128, 2>::THREADS, RowK<128, 2>::SMEM, RowK<128, 2>::MINB);
    } else if (row_env && p.head_dim == 256 && row_lpr256 == 2) {
      e = p.hadamard ? go_row(fa3b_fp8_prepare_row_kernel<256, 2, true>, RowK<256, 2>::THREADS, RowK<256, 2>::SMEM, RowK<256, 2>::MINB)
                     : go_row(fa3b_fp8_prepare_row_kernel<256, 2, false>, RowK<256, 2>::THREADS, RowK<256, 2>::SMEM, RowK<256, 2>::MINB);
    } else if (row_env && p.head_dim == 256 && row_lpr256 == 4) {
      e = p.hadamard ? go_row(fa3b_fp8_prepare_row_kernel<256, 4, true>, RowK<256, 4>::THREADS, RowK<256, 4>::SMEM, RowK<256, 4>::MINB)
                     : go_row(fa3b_fp8_prepare_row_kernel<256, 4, false>, RowK<256, 4>::THREADS, RowK<256, 4>::SMEM, RowK<256, 4>::MINB);
    } else {
      switch (p.head_dim) {
        case 64: e = p.hadamard ? FA3B_K5_GO(64, true) : FA3B_K5_GO(64, false); break;
        case 128: e = p.hadamard ? FA3B_K5_GO(128, true) : FA3B_K5_GO(128, false); break;
        default: e = p.hadamard ? FA3B_K5_GO(256, true) : FA3B_K5_GO(256, false); break;
      }
    }
#undef FA3B_K5_GO
    if (e != cudaSuccess) return cuda_fail(e);
  } else if (p.block_rows == 128 && p.head_dim <= 128) {
    // d = 256 would hold 64 doubles per thread; it takes the two-pass kernel instead
    const int items = a.nblk * p.heads * p.batch;
    // persistent at d = 128 (+7 %); d = 64 (half the FP64 work per block) was faster
    // with one CTA per item (1334 vs 1073 GB/s), where the prefetch is a no-op
    const int pgrid = (p.head_dim == 64 || items < num_sms()) ? items : num_sms();
    const bool f32 = p.src_dtype == FA3B_DTYPE_F32;
    const int smem = 2 * 512 * (p.head_dim / 4) * (f32 ? 4 : 2);
    auto go = [&](auto kern) {
      const int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
      if (rc == FA3B_OK) kern<<<pgrid, 512, smem, st>>>(a, items);
      return rc;
    };
    const int rc = p.head_dim == 64
                       ? (f32 ? go(fa3b_fp8_prepare_quad_kernel<64, 4>) : go(fa3b_fp8_prepare_quad_kernel<64, 2>))
                       : (f32 ? go(fa3b_fp8_prepare_quad_kernel<128, 4>) : go(fa3b_fp8_prepare_quad_kernel<128, 2>));
    if (rc != FA3B_OK) return rc;
  } else {
    switch (p.head_dim) {
      case 64: e = launch_generic<64>(a, grid, st); break;
      case 128: e = launch_generic<128>(a, grid, st); break;
      default: e = launch_generic<256>(a, grid, st); break;
    }
    if (e != cudaSuccess) return cuda_fail(e);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launch_count = 1;
  return FA3B_OK;
}
