/*
 * fa3b — B200-native (sm_100a) FlashAttention-3 hot path behind a C ABI.
 *
 * This is the drop-in boundary for the attention entry points of the
 * reference library "flashlab" (proj/core). Each entry point below names the
 * reference function it replaces (paths relative to the reference tree):
 *
 *   fa3b_fwd            flash_fwd_basic / flash_fwd_2stage / flash_fwd_3stage
 *                       (core/include/flashlab/flash_fwd.hpp:54-65,
 *                        core/src/flash_fwd.cpp:219-232), and with
 *                       in_dtype = FA3B_DTYPE_E4M3 the main loop of
 *                       fp8_flash_fwd (core/include/flashlab/fp8_attention.hpp:46,
 *                        core/src/fp8_attention.cpp:77-181)
 *   fa3b_fp8_prepare    preprocess_incoherent + quantize_per_block /
 *                       quantize_per_tensor as called by fp8_flash_fwd
 *                       (core/src/fp8_attention.cpp:33-42,88-96;
 *                        core/src/hadamard.cpp:11-64; core/src/quantize.cpp:35-60)
 *   fa3b_bwd_preprocess bwd_preprocess (core/include/flashlab/flash_bwd.hpp:15,
 *                        core/src/flash_bwd.cpp:29-41)
 *   fa3b_bwd            flash_bwd (core/include/flashlab/flash_bwd.hpp:20-21,
 *                        core/src/flash_bwd.cpp:43-126)
 *
 * Differences from the reference contract, all deliberate:
 *   - the reference computes one head per call on an FP64 row-major N x d
 *     matrix; here one call covers [batch, seq, head, dim] device tensors in
 *     f16/bf16/e4m3 (head dim contiguous) with fp32 accumulation;
 *   - head_dim must be 64, 128 or 256 (reference: any d);
 *   - TileConfig has no equivalent: results are block-size invariant up to
 *     rounding (reference test_flash_fwd.cpp:120-137).
 * Error codes map 1:1 to the reference's std::invalid_argument cases; the
 * message for each code is what fa3b_error_string returns (the reference's
 * wording where one exists).
 *
 * Threading: every call is reentrant, allocates nothing on the device and
 * launches on the caller's stream; results are ready when that stream is.
 */
#ifndef FA3B_H_
#define FA3B_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FA3B_ABI_VERSION 2

#if defined(__GNUC__)
#define FA3B_API __attribute__((visibility("default")))
#else
#define FA3B_API
#endif

typedef enum fa3b_dtype {
  FA3B_DTYPE_F16 = 0,
  FA3B_DTYPE_BF16 = 1,
  FA3B_DTYPE_E4M3 = 2, /* OCP FN e4m3, max finite 448 */
  FA3B_DTYPE_F32 = 3
} fa3b_dtype;

/* Kernel schedule, the device analogue of the reference's three forward
 * schedules (flash_fwd.cpp:142-191) plus the paper's ablation variants
 * (PAPER.md:748-765). All give results equal within rounding; the default is
 * the fastest. "Tile" = 128 query rows; "S" = the QK^T block in TMEM. */
typedef enum fa3b_schedule {
  FA3B_SCHED_PINGPONG = 0, /* default (flash_fwd_2stage): d <= 128 runs 2 query tiles per
                              CTA whose softmax and GEMMs alternate on the tensor core
                              (inter-warpgroup ping-pong); d = 256 runs
                              the 3STAGE schedule (two tiles do not fit TMEM) */
  FA3B_SCHED_BASIC = 1,    /* flash_fwd_basic: one tile per SM, strictly serial
                              S_j -> softmax_j -> PV_j (flash_fwd.cpp:142-147); warp
                              specialized, no GEMM-softmax overlap */
  FA3B_SCHED_3STAGE = 2,   /* flash_fwd_3stage: one tile, S_{j+1} in flight during softmax_j,
                              which also overlaps PV_{j-1}; the O rescale is deferred to
                              just before PV_j (two live P blocks, flash_fwd.cpp:170-191) */
  FA3B_SCHED_2STAGE = 3,   /* the reference's 2-stage order on one tile: S_{j+1} in flight
                              during softmax_j, softmax_j starts after PV_{j-1} completes
                              (one pending score, one live P block, flash_fwd.cpp:148-169) */
  FA3B_SCHED_NO_WS = 4,    /* ablation: GEMM-softmax pipelining (S_{j+1} during softmax_j)
                              without warp specialization: the softmax warps issue the TMA
                              loads and MMAs themselves; f16/bf16 only */
  FA3B_SCHED_LAST = FA3B_SCHED_NO_WS
} fa3b_schedule;

typedef enum fa3b_status {
  FA3B_OK = 0,
  FA3B_ERR_EMPTY = -1,             /* attention: empty inputs */
  FA3B_ERR_HEAD_DIM_MISMATCH = -2, /* attention: head dimension mismatch */
  FA3B_ERR_SEQLEN_MISMATCH = -3,   /* attention: sequence length mismatch */
  FA3B_ERR_ALPHA = -4,             /* attention: alpha must be finite and nonzero */
  FA3B_ERR_HEAD_DIM = -5,          /* head_dim must be 64, 128 or 256 */
  FA3B_ERR_GQA = -6,               /* gqa_head_map: heads must be a multiple of kv_heads */
  FA3B_ERR_ALIGNMENT = -7,         /* 16-byte aligned pointers, strides multiple of 16 B */
  FA3B_ERR_DTYPE = -8,             /* unsupported dtype combination */
  FA3B_ERR_NULL = -9,              /* required pointer is NULL */
  FA3B_ERR_DO_SHAPE = -10,         /* flash_bwd: dO shape mismatch */
  FA3B_ERR_FWD_SHAPE = -11,        /* flash_bwd: forward output shape mismatch */
  FA3B_ERR_NOT_POW2 = -12,         /* random_dh_transform: dim must be a power of two */
  FA3B_ERR_TILE = -13,             /* TileConfig: block sizes must be positive */
  FA3B_ERR_WORKSPACE = -14,        /* workspace missing or too small */
  FA3B_ERR_STRUCT = -15,           /* struct_size does not match this library */
  FA3B_ERR_BLOCK = -16,            /* fp8 quantization block size unsupported */
  FA3B_ERR_SCHEDULE = -17,         /* schedule value unknown or unsupported for the dtype */
  FA3B_ERR_SCALES = -18,           /* fp8 scale arrays do not match the block sizes */
  FA3B_ERR_CUDA = -100,            /* CUDA error; see fa3b_last_cuda_error() */
  FA3B_ERR_DEVICE = -101           /* device is not sm_100 */
} fa3b_status;

/* A [batch, seq, head, dim] tensor with the dim axis contiguous. Strides are
 * in elements. */
typedef struct fa3b_tensor4 {
  void* ptr;
  int64_t stride_batch;
  int64_t stride_seq;
  int64_t stride_head;
} fa3b_tensor4;

typedef struct fa3b_fwd_params {
  uint32_t struct_size; /* = sizeof(fa3b_fwd_params) */
  int32_t batch, heads_q, heads_kv, seqlen, head_dim;
  int32_t in_dtype;     /* F16, BF16 or E4M3 */
  int32_t out_dtype;    /* F16/BF16 (must equal in_dtype for 16-bit input; BF16 for
                           E4M3 input) or F32 */
  fa3b_tensor4 q, k, v; /* heads_q / heads_kv / heads_kv heads */
  fa3b_tensor4 o;       /* heads_q heads */
  float* lse;           /* [batch, heads_q, seqlen] natural-log logsumexp; may be NULL.
                           -inf (and O = 0) for a row with no unmasked column. */
  double alpha;         /* score scale; finite, nonzero, may be negative */
  int32_t causal;       /* key j hidden from query i when j > i */
  int32_t schedule;     /* fa3b_schedule */
  /* E4M3 only: dequantization scales as written by fa3b_fp8_prepare,
   * [batch, heads, ceil(seqlen / block_rows)] (or [batch, heads] when the
   * block size is 0 = per tensor). */
  const float* q_scale;
  const float* k_scale;
  const float* v_scale;
  int32_t q_block_rows;  /* 0 (per tensor) or 128 */
  int32_t kv_block_rows; /* 0 (per tensor) or 128 */
  void* stream;          /* cudaStream_t; NULL = legacy default stream */
} fa3b_fwd_params;

typedef struct fa3b_fp8_prepare_params {
  uint32_t struct_size; /* = sizeof(fa3b_fp8_prepare_params) */
  int32_t batch, heads, seqlen, head_dim;
  int32_t src_dtype;    /* F16, BF16 or F32 */
  fa3b_tensor4 src;
  fa3b_tensor4 dst;     /* E4M3 codes, same shape as src */
  float* scales;        /* out: [batch, heads, nblocks]; amax/448, or 1 if amax == 0 */
  int32_t block_rows;   /* rows per scale; 0 = one scale per (batch, head) */
  int32_t hadamard;     /* apply diag(signs) * H / sqrt(d) to each row first */
  uint64_t seed;        /* sign vector seed: sign_i = +1 iff word(i) is odd */
  int32_t saturate;     /* 1: clamp |code| to 448 (reference default); 0: overflow to NaN */
  void* stream;
  /* Added in ABI 2 (an ABI 1 struct_size, without it, reads as 0). 1: scale = the smallest
     power of two >= amax / 448 (codes of a block's maximum land in (224, 448]).
     Not a reference mode: the FP8 forward quantizes V this way so that K6 can
     carry V's per-block scale in the P codes exactly (an exponent shift). */
  int32_t scale_pow2;
} fa3b_fp8_prepare_params;

typedef struct fa3b_bwd_params {
  uint32_t struct_size; /* = sizeof(fa3b_bwd_params) */
  int32_t batch, heads_q, heads_kv, seqlen, head_dim;
  int32_t dtype;        /* F16 or BF16 for q, k, v, o, dout, dq, dk, dv */
  fa3b_tensor4 q, k, v, o, dout;
  fa3b_tensor4 dq, dk, dv;
  const float* lse;     /* [batch, heads_q, seqlen] from fa3b_fwd */
  double alpha;
  int32_t causal;
  int32_t deterministic; /* 0: dQ tiles summed in arrival order (fastest);
                            1: in ascending KV-tile order, the reference's
                            (flash_bwd.cpp:58-61): reruns are bitwise identical */
  void* workspace;       /* >= fa3b_bwd_workspace_bytes(...) bytes, 256-byte aligned */
  size_t workspace_bytes;
  void* stream;
} fa3b_bwd_params;

typedef struct fa3b_bwd_preprocess_params {
  uint32_t struct_size;
  int32_t batch, heads, seqlen, head_dim;
  int32_t dtype;        /* F16, BF16 or F32 */
  fa3b_tensor4 o, dout;
  float* delta;         /* out: [batch, heads, seqlen], D_i = sum_j dO_ij * O_ij */
  void* stream;
} fa3b_bwd_preprocess_params;

FA3B_API int fa3b_fwd(const fa3b_fwd_params* p);
FA3B_API int fa3b_fp8_prepare(const fa3b_fp8_prepare_params* p);
FA3B_API int fa3b_bwd_preprocess(const fa3b_bwd_preprocess_params* p);
FA3B_API int fa3b_bwd(const fa3b_bwd_params* p);
FA3B_API size_t fa3b_bwd_workspace_bytes(int32_t batch, int32_t heads_q, int32_t heads_kv,
                                int32_t seqlen, int32_t head_dim);

/* Closed-form model FLOPs (reference flash_fwd.hpp:69-77). */
FA3B_API uint64_t fa3b_flops_forward(uint64_t seqlen, uint64_t headdim, uint64_t heads, int32_t causal);
FA3B_API uint64_t fa3b_flops_backward(uint64_t seqlen, uint64_t headdim, uint64_t heads,
                             int32_t causal);

FA3B_API const char* fa3b_error_string(int status);
FA3B_API int fa3b_last_cuda_error(void); /* cudaError_t of the most recent FA3B_ERR_CUDA, per thread */
FA3B_API int fa3b_abi_version(void);
/* Number of kernels the most recent successful call on this thread launched. */
FA3B_API int fa3b_last_launch_count(void);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* FA3B_H_ */
