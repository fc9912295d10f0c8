/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the fa3b hot path.
 *
 * A plain-C restatement of the reference library's attention algorithms
 * (flashlab, proj/core), one head per call on row-major FP64 arrays. Each
 * function cites the reference file:line it follows. It is pinned against the
 * reference compiled from its own sources (oracle/_ref, see Makefile) and
 * against the reference tests' golden values (tests/golden/). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it.
 *
 * Status returns: 0 ok, negative = the reference's std::invalid_argument case
 * (fa3b_oracle_last_error() gives the reference's message).
 */
#ifndef FA3B_ORACLE_H_
#define FA3B_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_FP64 = 0, ORC_FP32 = 1, ORC_FP16 = 2, ORC_BF16 = 3, ORC_E4M3 = 4 };

const char* fa3b_oracle_last_error(void);

/* rng.cpp:13-78 */
uint64_t orc_substream(uint64_t seed, uint64_t salt);
uint64_t orc_word(uint64_t seed, uint64_t counter);
double orc_gaussian(uint64_t seed, uint64_t counter);
void orc_sample_gaussian(size_t rows, size_t cols, uint64_t seed, double* out);
int orc_sample_outlier(size_t rows, size_t cols, uint64_t seed, double p, double* out);
void orc_sign_vector(size_t n, uint64_t seed, double* out);

/* formats.cpp:45-61 */
double orc_round_to(double x, int fmt, int overflow_infinite);
void orc_round_array(const double* in, size_t n, int fmt, double* out);

/* hadamard.cpp:11-64, fp8_attention.cpp:33-42 */
int orc_fwht(double* v, size_t n);
int orc_preprocess_incoherent(const double* q, const double* k, size_t n, size_t d,
                              uint64_t seed, double* qo, double* ko);

/* quantize.cpp:35-60 (block_rows 0 = per tensor) */
int orc_quantize(const double* m, size_t rows, size_t cols, size_t block_rows,
                 int overflow_infinite, double* codes, double* scales);

/* flash_fwd.cpp:18-215 (basic schedule; all schedules are bit-identical) */
int orc_flash_fwd(const double* q, const double* k, const double* v, size_t n, size_t d,
                  double alpha, int causal, size_t br, size_t bc, double* o, double* lse,
                  uint64_t* visited, uint64_t* skipped);

/* flash_bwd.cpp:29-126 */
int orc_bwd_preprocess(const double* dO, const double* o, size_t n, size_t d, double* out);
int orc_flash_bwd(const double* q, const double* k, const double* v, const double* dO,
                  const double* o, const double* lse, size_t n, size_t d, double alpha,
                  int causal, size_t br, size_t bc, double* dq, double* dk, double* dv);

/* lowprec.cpp:166-240 generalized to fmt in {ORC_FP16, ORC_BF16}: 16-bit
 * operands, fp32 scores / online softmax / accumulator, P rounded to fmt. */
int orc_lowprec_flash_fwd(const double* q, const double* k, const double* v, size_t n,
                          size_t d, double alpha, int causal, size_t br, size_t bc, int fmt,
                          double* o, double* lse);

/* Backward with the tensor-core rounding points: inputs in fmt, P and dS
 * rounded to fmt before their GEMMs, fp32 accumulation (the yardstick for
 * the device backward; the reference has no low-precision backward). */
int orc_lowprec_flash_bwd(const double* q, const double* k, const double* v,
                          const double* dO, const double* o, const double* lse, size_t n,
                          size_t d, double alpha, int causal, size_t br, size_t bc, int fmt,
                          double* dq, double* dk, double* dv);

/* fp8_attention.cpp:77-181 (permuted_value_layout = false) */
int orc_fp8_flash_fwd(const double* q, const double* k, const double* v, size_t n, size_t d,
                      double alpha, int causal, int per_block, int incoherent, uint64_t seed,
                      size_t br, size_t bc, double* o, double* lse);

/* reference_attention_o (attention_ref.cpp:116-128): exact FP64 standard
 * attention streamed over row blocks. */
int orc_reference_attention(const double* q, const double* k, const double* v, size_t n,
                            size_t d, double alpha, int causal, double* o, double* lse);

#ifdef __cplusplus
}
#endif
#endif
