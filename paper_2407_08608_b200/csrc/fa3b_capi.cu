// C-ABI entry points (include/fa3b.h): argument validation with the
// reference's error semantics, TMA descriptor construction, and dispatch to
// the sm_100a kernels. No device allocation happens here.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/fa3b.h"
#include "fa3b_internal.cuh"

namespace fa3b {

thread_local int g_last_cuda_error = 0;
thread_local int g_last_launch_count = 0;

int cuda_fail(cudaError_t e) {
  g_last_cuda_error = static_cast<int>(e);
  return FA3B_ERR_CUDA;
}

namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// Ping-pong pairing choice; FA3B_FWD_PAIRING=cta|warp overrides the measured default.
bool fwd_pairing_impl(int head_dim, bool causal, bool fp8, int seqlen) {
  static const int forced = [] {
    const char* e = std::getenv("FA3B_FWD_PAIRING");
    if (e == nullptr) return -1;
    return std::strcmp(e, "cta") == 0 ? 1 : (std::strcmp(e, "warp") == 0 ? 0 : -1);
  }();
  (void)causal;
  if (head_dim > 128) return false;
  if (forced >= 0) return forced == 1;
  // Warp pairing (two tiles per CTA) measured faster on every C2/C3/C5 shape at
  // N 8k (profiles/r01m_pairing_ab.log) and for bf16 at every length; at short
  // sequences (N <= 512) the FP8 forward gains 5-10 % from two one-tile CTAs per SM, whose item
  // boundaries overlap; at N 1024 it loses 1-3 % (profiles/r02/r02af_pairing_short.log,
  // r02aj_short.log)
  return fp8 && head_dim == 128 && seqlen <= 512;
}

}  // namespace

// sm_100 check, cached per device (a process may drive several GPUs) and made by
// every entry point that launches kernels.
int check_device() {
  static std::mutex mu;
  static std::vector<int> cache;  // 0 unknown, 1 ok, 2 unsupported
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FA3B_ERR_DEVICE;
  std::lock_guard<std::mutex> lock(mu);
  if (dev >= static_cast<int>(cache.size())) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cache[dev] = (major == 10 && minor == 0) ? 1 : 2;
  }
  return cache[dev] == 1 ? FA3B_OK : FA3B_ERR_DEVICE;
}

bool fwd_pairing(int head_dim, bool causal, bool fp8, int seqlen) {
  return fwd_pairing_impl(head_dim, causal, fp8, seqlen);
}

int num_sms() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lock(mu);
  if (dev >= static_cast<int>(cache.size())) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

int ensure_smem_attr(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;  // (kernel, device)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first == kernel && d.second == dev) return FA3B_OK;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return cuda_fail(e);
  done.emplace_back(kernel, dev);
  return FA3B_OK;
}

// [batch, seq, head, dim] tensor -> 4D map (dim, head, seq, batch) with a box
// of (inner_elems, 1, rows, 1) and 128B swizzle. OOB rows read as zero.
int make_tmap_4d(CUtensorMap* map, const fa3b_tensor4& t, int elem_bytes, int dim, int heads,
                 int seqlen, int batch, int inner_elems, int rows, int swizzle_bytes) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return cuda_fail(cudaErrorNotSupported);
  CUtensorMapDataType dt = elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                           : (elem_bytes == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                                              : CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(dim), static_cast<cuuint64_t>(heads),
                        static_cast<cuuint64_t>(seqlen), static_cast<cuuint64_t>(batch)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(t.stride_head) * elem_bytes,
                           static_cast<cuuint64_t>(t.stride_seq) * elem_bytes,
                           static_cast<cuuint64_t>(t.stride_batch) * elem_bytes};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(inner_elems), 1u, static_cast<cuuint32_t>(rows),
                       1u};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, dt, 4, t.ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cuda_fail(cudaErrorInvalidValue);
  return FA3B_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Strides (elements) must keep every row 16-byte aligned for TMA and the
// vectorized epilogue.
bool strides_ok(const fa3b_tensor4& t, int elem_bytes, int batch, int seqlen, int heads) {
  auto ok = [&](int64_t s, int extent) {
    return extent <= 1 || (s > 0 && (s * elem_bytes) % 16 == 0);
  };
  return aligned16(t.ptr) && ok(t.stride_batch, batch) && ok(t.stride_seq, seqlen) &&
         ok(t.stride_head, heads);
}

// Shared validation of the attention problem (reference validate_inputs,
// attention_ref.cpp:20-29, plus gqa_head_map :130-137 and the head_dim set).
int validate_problem(int batch, int heads_q, int heads_kv, int seqlen, int head_dim,
                     double alpha) {
  if (batch <= 0 || heads_q <= 0 || heads_kv <= 0 || seqlen <= 0 || head_dim <= 0)
    return FA3B_ERR_EMPTY;
  if (!std::isfinite(alpha) || alpha == 0.0) return FA3B_ERR_ALPHA;
  if (heads_q % heads_kv != 0) return FA3B_ERR_GQA;
  if (head_dim != 64 && head_dim != 128 && head_dim != 256) return FA3B_ERR_HEAD_DIM;
  return FA3B_OK;
}

}  // namespace fa3b

using namespace fa3b;

extern "C" {

int fa3b_abi_version(void) { return FA3B_ABI_VERSION; }

int fa3b_last_cuda_error(void) { return g_last_cuda_error; }
int fa3b_last_launch_count(void) { return g_last_launch_count; }

uint64_t fa3b_flops_forward(uint64_t seqlen, uint64_t headdim, uint64_t heads, int32_t causal) {
  const uint64_t f = 4ull * seqlen * seqlen * headdim * heads;
  return causal ? f / 2 : f;
}
uint64_t fa3b_flops_backward(uint64_t seqlen, uint64_t headdim, uint64_t heads,
                             int32_t causal) {
  return fa3b_flops_forward(seqlen, headdim, heads, causal) * 5 / 2;
}

const char* fa3b_error_string(int status) {
  switch (status) {
    case FA3B_OK: return "ok";
    case FA3B_ERR_EMPTY: return "attention: empty inputs";
    case FA3B_ERR_HEAD_DIM_MISMATCH: return "attention: head dimension mismatch";
    case FA3B_ERR_SEQLEN_MISMATCH: return "attention: sequence length mismatch";
    case FA3B_ERR_ALPHA: return "attention: alpha must be finite and nonzero";
    case FA3B_ERR_HEAD_DIM: return "fa3b: head dimension must be 64, 128 or 256";
    case FA3B_ERR_GQA: return "gqa_head_map: heads must be a multiple of kv_heads";
    case FA3B_ERR_ALIGNMENT:
      return "fa3b: pointers must be 16-byte aligned and row strides multiples of 16 bytes";
    case FA3B_ERR_DTYPE: return "fa3b: unsupported dtype combination";
    case FA3B_ERR_NULL: return "fa3b: required pointer is NULL";
    case FA3B_ERR_DO_SHAPE: return "flash_bwd: dO shape mismatch";
    case FA3B_ERR_FWD_SHAPE: return "flash_bwd: forward output shape mismatch";
    case FA3B_ERR_NOT_POW2: return "random_dh_transform: dim must be a power of two";
    case FA3B_ERR_TILE: return "TileConfig: block sizes must be positive";
    case FA3B_ERR_WORKSPACE: return "fa3b: workspace missing or too small";
    case FA3B_ERR_STRUCT: return "fa3b: parameter struct size mismatch (ABI)";
    case FA3B_ERR_BLOCK: return "fa3b: fp8 quantization block must be 0 (per tensor) or 128 rows";
    case FA3B_ERR_SCHEDULE: return "fa3b: unknown schedule, or schedule unsupported for this dtype";
    case FA3B_ERR_SCALES: return "fa3b: fp8 scale arrays do not match the quantization blocks";
    case FA3B_ERR_CUDA: return "fa3b: CUDA error (see fa3b_last_cuda_error)";
    case FA3B_ERR_DEVICE: return "fa3b: requires an sm_100 (B200) device";
    default: return "fa3b: unknown status";
  }
}

int fa3b_fwd(const fa3b_fwd_params* pp) {
  g_last_launch_count = 0;
  if (pp == nullptr) return FA3B_ERR_NULL;
  if (pp->struct_size != sizeof(fa3b_fwd_params)) return FA3B_ERR_STRUCT;
  const fa3b_fwd_params& p = *pp;
  int rc = validate_problem(p.batch, p.heads_q, p.heads_kv, p.seqlen, p.head_dim, p.alpha);
  if (rc != FA3B_OK) return rc;
  if (!p.q.ptr || !p.k.ptr || !p.v.ptr || !p.o.ptr) return FA3B_ERR_NULL;
  if (p.schedule < FA3B_SCHED_PINGPONG || p.schedule > FA3B_SCHED_LAST) return FA3B_ERR_SCHEDULE;
  const bool fp8 = p.in_dtype == FA3B_DTYPE_E4M3;
  if (p.in_dtype != FA3B_DTYPE_F16 && p.in_dtype != FA3B_DTYPE_BF16 && !fp8)
    return FA3B_ERR_DTYPE;
  if (!fp8 && p.out_dtype != p.in_dtype && p.out_dtype != FA3B_DTYPE_F32) return FA3B_ERR_DTYPE;
  if (fp8 && p.out_dtype != FA3B_DTYPE_BF16 && p.out_dtype != FA3B_DTYPE_F32)
    return FA3B_ERR_DTYPE;
  const int in_b = fp8 ? 1 : 2;
  const int out_b = p.out_dtype == FA3B_DTYPE_F32 ? 4 : 2;
  if (!strides_ok(p.q, in_b, p.batch, p.seqlen, p.heads_q) ||
      !strides_ok(p.k, in_b, p.batch, p.seqlen, p.heads_kv) ||
      !strides_ok(p.v, in_b, p.batch, p.seqlen, p.heads_kv) ||
      !strides_ok(p.o, out_b, p.batch, p.seqlen, p.heads_q))
    return FA3B_ERR_ALIGNMENT;
  if ((rc = check_device()) != FA3B_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(p.stream);
  if (fp8) return launch_fwd_fp8(p, s);
  if (p.schedule != FA3B_SCHED_PINGPONG) {
    // the one-tile schedule variants (the reference's basic / 2-stage / 3-stage and
    // the no-warp-specialization ablation); at d = 256 the default is already 3-stage
    if (p.head_dim == 256 && p.schedule == FA3B_SCHED_3STAGE)
      return launch_fwd16_default_d256(p, s, false);
    const bool bf16 = p.in_dtype == FA3B_DTYPE_BF16;
    if (p.causal) return bf16 ? launch_fwd16_sched_bf16_c1(p, s) : launch_fwd16_sched_f16_c1(p, s);
    return bf16 ? launch_fwd16_sched_bf16_c0(p, s) : launch_fwd16_sched_f16_c0(p, s);
  }
  // Ping-pong pairs: two query tiles of one CTA (warp pairing, the default) or
  // one tile in each of two CTAs per SM (CTA pairing, FA3B_FWD_PAIRING=cta);
  // A/B in profiles/r01m_pairing_ab.log.
  const bool cta_pairs = fwd_pairing(p.head_dim, p.causal != 0, false, p.seqlen);
  switch (p.head_dim) {
    case 64: return launch_fwd16_default_d64(p, s, cta_pairs);
    case 128: return launch_fwd16_default_d128(p, s, cta_pairs);
    case 256: return launch_fwd16_default_d256(p, s, false);
  }
  return FA3B_ERR_HEAD_DIM;
}

}  // extern "C"
