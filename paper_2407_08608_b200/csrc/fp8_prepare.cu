// K5: incoherent processing + e4m3 quantization of one [B, N, H, d] tensor.
//
// Reference: preprocess_incoherent (core/src/fp8_attention.cpp:33-42) ->
// DHTransform::apply = sign flip then normalized FWHT (core/src/hadamard.cpp:11-33)
// with signs from sample_sign_vector (core/src/rng.cpp:73-78); then
// quantize_per_block / quantize_per_tensor (core/src/quantize.cpp:10-60):
// scale = amax / 448 (1 if amax == 0), code = round_to(x * (1 / scale), e4m3)
// (core/src/formats.cpp:45-61, RNE, saturating).
//
// The arithmetic is FP64 with the reference's butterfly and rounding order, so
// codes and scales are byte-identical to the reference for the same input
// values (tests/test_fp8_gpu.py). The kernel is HBM-bound (2-4 bytes read,
// 1 byte written per element); FP64 costs ~7 flop/element, well under the
// B200 FP64 rate needed to stay memory-bound.
//
// Layout: one CTA per (row block, head, batch); one warp per row, lane l
// holds the E = d/32 contiguous elements [l E, l E + E). Butterfly stages with
// len < E stay in the thread, larger ones exchange with lane l ^ (len / E)
// through shuffles. Each lane's E source elements arrive in one or two vector
// loads, all rows of a warp in flight together. 128-row blocks at d <= 128 keep
// the whole transformed block in registers (16 warps x 8 rows) across the amax
// reduction; d = 256 and other block sizes (per tensor) take two passes that
// recompute the transform (the second read hits L2).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>

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

template <int E>
__device__ __forceinline__ void fwht_warp(double (&v)[E], int lane) {
  constexpr int D = 32 * E;
#pragma unroll
  for (int len = 1; len < D; len <<= 1) {
    if (len < E) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if ((e & len) == 0) {
          const double a = v[e], b = v[e + len];
          v[e] = a + b;
          v[e + len] = a - b;
        }
      }
    } else {
      const int lmask = len / E;
      // lower lane: v + other; upper lane: other - v; one exact-product DFMA either way
      // (IEEE addition commutes, so the rounding equals the reference's a + b / a - b)
      const double sgn = (lane & lmask) ? -1.0 : 1.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double other = __shfl_xor_sync(0xffffffffu, v[e], lmask);
        v[e] = fma(sgn, v[e], other);
      }
    }
  }
  const double norm = 1.0 / sqrt(static_cast<double>(D));
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] *= norm;
}

struct PrepArgs {
  const void* src;
  long long s_sb, s_ss, s_sh;
  int src_dtype;
  uint8_t* dst;
  long long d_sb, d_ss, d_sh;
  float* scales;
  int N, H, block_rows, nblk, hadamard, saturate;
  unsigned long long signs[4];  // bit i set -> sign_i = +1
};

// The E contiguous source elements of one lane as raw words: E x 16-bit (4-16 B)
// or E x fp32 (8-32 B), one or two vector loads.
template <int E>
struct RawRow {
  uint4 w[E / 2 > 2 ? E / 2 : 2];
};

template <int E>
__device__ __forceinline__ void load_raw(const PrepArgs& a, int b, int h, int row, int lane,
                                         RawRow<E>& r) {
  const size_t base = b * a.s_sb + static_cast<size_t>(row) * a.s_ss + h * a.s_sh + lane * E;
  if (a.src_dtype == FA3B_DTYPE_F32) {
    const float* p = static_cast<const float*>(a.src) + base;
    if constexpr (E == 2) {
      const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
      r.w[0] = make_uint4(t.x, t.y, 0, 0);
    } else {
#pragma unroll
      for (int i = 0; i < E / 4; ++i) r.w[i] = __ldg(reinterpret_cast<const uint4*>(p) + i);
    }
  } else {
    const uint16_t* p = static_cast<const uint16_t*>(a.src) + base;
    if constexpr (E == 2) {
      r.w[0].x = __ldg(reinterpret_cast<const unsigned int*>(p));
    } else if constexpr (E == 4) {
      const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
      r.w[0] = make_uint4(t.x, t.y, 0, 0);
    } else {
      r.w[0] = __ldg(reinterpret_cast<const uint4*>(p));
    }
  }
}

template <int E>
__device__ __forceinline__ void unpack_raw(const PrepArgs& a, const RawRow<E>& r, double (&v)[E]) {
  const uint32_t* u = reinterpret_cast<const uint32_t*>(&r.w[0]);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (a.src_dtype == FA3B_DTYPE_F32) {
      v[e] = __uint_as_float(u[e]);
    } else {
      const uint16_t bits = static_cast<uint16_t>(u[e >> 1] >> (16 * (e & 1)));
      v[e] = a.src_dtype == FA3B_DTYPE_BF16 ? __uint_as_float(static_cast<uint32_t>(bits) << 16)
                                            : __half2float(__ushort_as_half(bits));
    }
  }
}

template <int E>
__device__ __forceinline__ void transform_row(const PrepArgs& a, int lane, double (&v)[E]) {
  if (a.hadamard) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = lane * E + e;
      if (!((a.signs[i >> 6] >> (i & 63)) & 1ull)) v[e] = -v[e];
    }
    fwht_warp<E>(v, lane);
  }
}

template <int E>
__device__ __forceinline__ void load_row(const PrepArgs& a, int b, int h, int row, int lane,
                                         double (&v)[E]) {
  RawRow<E> r;
  load_raw<E>(a, b, h, row, lane, r);
  unpack_raw<E>(a, r, v);
  transform_row<E>(a, lane, v);
}

template <int E>
__device__ __forceinline__ void store_codes(const PrepArgs& a, int b, int h, int row, int lane,
                                            const double (&v)[E], double inv) {
  uint8_t c[E];
  if (a.saturate) {
    // FP64 -> FP32 with round-to-odd (truncate, then set the last bit if inexact),
    // then the hardware RNE saturating e4m3 conversion: rounding to odd at 24
    // bits before rounding to 4 bits equals rounding the FP64 value directly.
#pragma unroll
    for (int e = 0; e < E; e += 2) {
      float f[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double t = v[e + u] * inv;
        float z = __double2float_rz(t);
        if (static_cast<double>(z) != t) z = __uint_as_float(__float_as_uint(z) | 1u);
        f[u] = z;
      }
      uint16_t pr;
      asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(pr) : "f"(f[1]), "f"(f[0]));
      c[e] = static_cast<uint8_t>(pr & 0xFF);
      c[e + 1] = static_cast<uint8_t>(pr >> 8);
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) c[e] = e4m3_code(v[e] * inv, false);
  }
  uint8_t* dst = a.dst + b * a.d_sb + static_cast<size_t>(row) * a.d_ss + h * a.d_sh + lane * E;
  if constexpr (E == 2) {
    *reinterpret_cast<uint16_t*>(dst) = c[0] | (c[1] << 8);
  } else {
#pragma unroll
    for (int e = 0; e < E; e += 4)
      *reinterpret_cast<uint32_t*>(dst + e) = c[e] | (c[e + 1] << 8) | (c[e + 2] << 16) | (c[e + 3] << 24);
  }
}

__device__ __forceinline__ void write_scale(const PrepArgs& a, int b, int h, int blk, double amax,
                                            bool bad) {
  const double scale = amax == 0.0 ? 1.0 : amax / 448.0;
  // non-finite inputs: the reference throws; the device reports a NaN scale
  a.scales[(static_cast<size_t>(b) * a.H + h) * a.nblk + blk] =
      bad ? __int_as_float(0x7fc00000) : static_cast<float>(scale);
}

// Control flow around the butterflies is kept warp-uniform by construction
// (trip counts from blockIdx / kernel arguments only, row validity applied to
// the loads and stores): shuffles under a thread-dependent branch compile to
// WARPSYNC collectives that cost more than the arithmetic.

// 128-row blocks, d <= 128: 16 warps x 8 rows, the transformed block stays in
// registers between the amax reduction and the encode (one read of the input).
template <int E>
__global__ void __launch_bounds__(512) fa3b_fp8_prepare_block128_kernel(const PrepArgs a) {
  constexpr int RPW = 8;
  const int blk = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blk * 128 + warp * RPW;
  __shared__ double s_amax[16];
  __shared__ int s_bad[16];
  double v[RPW][E];
  double amax = 0.0;
  bool bad = false;
  // every row's loads are in flight before any arithmetic; rows past N read as zero
  RawRow<E> raw[RPW];
#pragma unroll
  for (int rr = 0; rr < RPW; ++rr) {
    raw[rr] = RawRow<E>{};
    if (r0 + rr < a.N) load_raw<E>(a, b, h, r0 + rr, lane, raw[rr]);
  }
#pragma unroll
  for (int rr = 0; rr < RPW; ++rr) {
    unpack_raw<E>(a, raw[rr], v[rr]);
    transform_row<E>(a, lane, v[rr]);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double x = fabs(v[rr][e]);
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
  for (int w = 1; w < 16; ++w) {
    amax = fmax(amax, s_amax[w]);
    bad |= s_bad[w] != 0;
  }
  if (threadIdx.x == 0) write_scale(a, b, h, blk, amax, bad);
  const double inv = 1.0 / (amax == 0.0 ? 1.0 : amax / 448.0);  // quantize.cpp:25
#pragma unroll
  for (int rr = 0; rr < RPW; ++rr)
    if (r0 + rr < a.N) store_codes<E>(a, b, h, r0 + rr, lane, v[rr], inv);
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
template <int E, int C>
__global__ void __launch_bounds__(256) fa3b_fp8_prepare_kernel(const PrepArgs a) {
  constexpr int WARPS = 8, RPI = 2;  // rows per warp per iteration
  const int blk = blockIdx.x / C, part = blockIdx.x % C, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb0 = a.block_rows ? blk * a.block_rows : 0;
  const int rb1 = a.block_rows ? min(a.N, rb0 + a.block_rows) : a.N;
  const int chunk = (rb1 - rb0 + C - 1) / C;
  const int c0 = rb0 + part * chunk, c1 = min(rb1, c0 + chunk);
  const int iters = c1 > c0 ? (c1 - c0 + WARPS * RPI - 1) / (WARPS * RPI) : 0;
  __shared__ double s_amax[WARPS];
  __shared__ int s_bad[WARPS];
  __shared__ double s_cta[2];  // this CTA's (amax, bad) for the cluster
  double amax = 0.0;
  bool bad = false;
  for (int it = 0; it < iters; ++it) {
    RawRow<E> raw[RPI];
#pragma unroll
    for (int u = 0; u < RPI; ++u) {
      const int row = c0 + (it * RPI + u) * WARPS + warp;
      raw[u] = RawRow<E>{};
      if (row < c1) load_raw<E>(a, b, h, row, lane, raw[u]);
    }
#pragma unroll
    for (int u = 0; u < RPI; ++u) {
      double v[E];
      unpack_raw<E>(a, raw[u], v);
      transform_row<E>(a, lane, v);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double x = fabs(v[e]);
        bad |= !isfinite(x);
        amax = fmax(amax, x);
      }
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
  const double inv = 1.0 / (amax == 0.0 ? 1.0 : amax / 448.0);
  for (int it = 0; it < iters; ++it) {
    RawRow<E> raw[RPI];
#pragma unroll
    for (int u = 0; u < RPI; ++u) {
      const int row = c0 + (it * RPI + u) * WARPS + warp;
      raw[u] = RawRow<E>{};
      if (row < c1) load_raw<E>(a, b, h, row, lane, raw[u]);
    }
#pragma unroll
    for (int u = 0; u < RPI; ++u) {
      const int row = c0 + (it * RPI + u) * WARPS + warp;
      double v[E];
      unpack_raw<E>(a, raw[u], v);
      transform_row<E>(a, lane, v);
      if (row < c1) store_codes<E>(a, b, h, row, lane, v, inv);
    }
  }
}

template <int E, int C>
cudaError_t launch_two_pass(const PrepArgs& a, dim3 grid, cudaStream_t st) {
  auto kern = fa3b_fp8_prepare_kernel<E, C>;
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

template <int E>
cudaError_t launch_generic(const PrepArgs& a, dim3 grid, cudaStream_t st) {
  // split each scale block over a cluster when there are too few blocks to fill 148 SMs
  const long long ctas = static_cast<long long>(grid.x) * grid.y * grid.z;
  const int rows = a.block_rows ? a.block_rows : a.N;
  if (ctas < 296 && rows >= 8 * 256) return launch_two_pass<E, 8>(a, grid, st);
  return launch_two_pass<E, 1>(a, grid, st);
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
  if (pp->struct_size != sizeof(fa3b_fp8_prepare_params)) return FA3B_ERR_STRUCT;
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
  // sample_sign_vector(d, seed): sign_i = +1 iff word(i) = mix64(seed + (i+1) gamma) is odd
  for (int i = 0; i < p.head_dim; ++i)
    if (mix64(p.seed + static_cast<uint64_t>(i + 1) * 0x9E3779B97F4A7C15ull) & 1ull)
      a.signs[i >> 6] |= 1ull << (i & 63);
  dim3 grid(a.nblk, p.heads, p.batch);
  cudaStream_t st = static_cast<cudaStream_t>(p.stream);
  cudaError_t e = cudaSuccess;
  if (p.block_rows == 128 && p.head_dim <= 128) {
    // d = 256 would hold 64 doubles per thread; it takes the two-pass kernel instead
    switch (p.head_dim) {
      case 64: fa3b_fp8_prepare_block128_kernel<2><<<grid, 512, 0, st>>>(a); break;
      default: fa3b_fp8_prepare_block128_kernel<4><<<grid, 512, 0, st>>>(a); break;
    }
  } else {
    switch (p.head_dim) {
      case 64: e = launch_generic<2>(a, grid, st); break;
      case 128: e = launch_generic<4>(a, grid, st); break;
      default: e = launch_generic<8>(a, grid, st); break;
    }
    if (e != cudaSuccess) return cuda_fail(e);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);
  g_last_launch_count = 1;
  return FA3B_OK;
}
