// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the reference library (flashlab proj/core), compiled
// from the sources where they lie under /root/reference by oracle/Makefile
// into oracle/_ref/libflashlab_ref.so. It lets the Python tests run the
// reference itself on the same inputs as the CUDA path, pin the C
// restatement (oracle/fa3b_oracle.c) against it, and time it as the CPU
// baseline. Every function handles one head: row-major FP64 n x d arrays,
// exactly the reference's Matrix carrier (matrix.hpp:17-40).
//
// Status: 0 ok, -1 std::invalid_argument (message via flref_last_error()).
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "flashlab/attention_ref.hpp"
#include "flashlab/flash_bwd.hpp"
#include "flashlab/flash_fwd.hpp"
#include "flashlab/formats.hpp"
#include "flashlab/fp8_attention.hpp"
#include "flashlab/hadamard.hpp"
#include "flashlab/lowprec.hpp"
#include "flashlab/matrix.hpp"
#include "flashlab/quantize.hpp"
#include "flashlab/rng.hpp"

using namespace flashlab;

namespace {

thread_local std::string g_err;

Matrix to_matrix(const double* p, std::size_t r, std::size_t c) {
  Matrix m(r, c);
  if (r * c) std::memcpy(m.data(), p, sizeof(double) * r * c);
  return m;
}
void from_matrix(const Matrix& m, double* out) {
  if (out && m.size()) std::memcpy(out, m.data(), sizeof(double) * m.size());
}
void from_vec(const std::vector<double>& v, double* out) {
  if (out && !v.empty()) std::memcpy(out, v.data(), sizeof(double) * v.size());
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

AttentionInputs inputs(const double* q, const double* k, const double* v, std::size_t n,
                       std::size_t d, double alpha, int causal) {
  return AttentionInputs{to_matrix(q, n, d), to_matrix(k, n, d), to_matrix(v, n, d), alpha,
                         causal != 0};
}

}  // namespace

extern "C" {

const char* flref_last_error() { return g_err.c_str(); }

uint64_t flref_substream(uint64_t seed, uint64_t salt) { return substream(seed, salt); }
uint64_t flref_word(uint64_t seed, uint64_t counter) { return CounterRng(seed).word(counter); }
double flref_gaussian(uint64_t seed, uint64_t counter) {
  return CounterRng(seed).gaussian(counter);
}

int flref_sample_gaussian(std::size_t rows, std::size_t cols, uint64_t seed, double* out) {
  return guarded([&] { from_matrix(sample_gaussian_matrix(rows, cols, seed), out); });
}
int flref_sample_outlier(std::size_t rows, std::size_t cols, uint64_t seed, double p,
                         double* out) {
  return guarded([&] { from_matrix(sample_outlier_matrix(rows, cols, seed, p), out); });
}
int flref_sign_vector(std::size_t n, uint64_t seed, double* out) {
  return guarded([&] { from_vec(sample_sign_vector(n, seed), out); });
}

// fmt: 0 fp64, 1 fp32, 2 fp16, 3 bf16, 4 e4m3 (FloatFormatId order)
double flref_round_to(double x, int fmt, int overflow_infinite) {
  return round_to(x, static_cast<FloatFormatId>(fmt),
                  overflow_infinite ? OverflowPolicy::infinite : OverflowPolicy::saturate);
}
int flref_round_array(const double* in, std::size_t n, int fmt, double* out) {
  for (std::size_t i = 0; i < n; ++i) out[i] = round_to(in[i], static_cast<FloatFormatId>(fmt));
  return 0;
}

uint64_t flref_flops_forward(uint64_t n, uint64_t d, uint64_t h, int causal) {
  return flops_forward(n, d, h, causal != 0);
}
uint64_t flref_flops_backward(uint64_t n, uint64_t d, uint64_t h, int causal) {
  return flops_backward(n, d, h, causal != 0);
}
int flref_gqa_head_map(std::size_t heads, std::size_t kv_heads, uint64_t* out) {
  return guarded([&] {
    const auto m = gqa_head_map(heads, kv_heads);
    for (std::size_t i = 0; i < m.size(); ++i) out[i] = m[i];
  });
}

// sched: 0 basic, 1 2-stage, 2 3-stage. stats[6] = visited, skipped,
// max_pending_scores, max_live_probs, deferred_output_scale, fell_back.
int flref_flash_fwd(int sched, const double* q, const double* k, const double* v,
                    std::size_t n, std::size_t d, double alpha, int causal, std::size_t br,
                    std::size_t bc, double* o, double* lse, uint64_t* stats) {
  return guarded([&] {
    const AttentionInputs in = inputs(q, k, v, n, d, alpha, causal);
    FlashFwdStats st;
    const TileConfig cfg{br, bc};
    ForwardOutput out = sched == 0   ? flash_fwd_basic(in, cfg, &st)
                        : sched == 1 ? flash_fwd_2stage(in, cfg, &st)
                                     : flash_fwd_3stage(in, cfg, &st);
    from_matrix(out.o, o);
    from_vec(out.logsumexp, lse);
    if (stats) {
      stats[0] = st.blocks_visited;
      stats[1] = st.blocks_skipped;
      stats[2] = st.max_pending_scores;
      stats[3] = st.max_live_probs;
      stats[4] = st.deferred_output_scale;
      stats[5] = st.fell_back_to_basic;
    }
  });
}

int flref_reference_attention(const double* q, const double* k, const double* v,
                              std::size_t n, std::size_t d, double alpha, int causal,
                              double* o, double* lse) {
  return guarded([&] {
    ForwardOutput out = reference_attention_o(inputs(q, k, v, n, d, alpha, causal));
    from_matrix(out.o, o);
    from_vec(out.logsumexp, lse);
  });
}

int flref_std_attention_bwd(const double* q, const double* k, const double* v,
                            const double* dO, std::size_t n, std::size_t d, double alpha,
                            int causal, double* dq, double* dk, double* dv) {
  return guarded([&] {
    const AttentionInputs in = inputs(q, k, v, n, d, alpha, causal);
    const StdForward f = std_attention_fwd(in);
    AttentionGrads g = std_attention_bwd(in, f.p, to_matrix(dO, n, d));
    from_matrix(g.dq, dq);
    from_matrix(g.dk, dk);
    from_matrix(g.dv, dv);
  });
}

int flref_bwd_preprocess(const double* dO, const double* o, std::size_t n, std::size_t d,
                         double* out) {
  return guarded([&] { from_vec(bwd_preprocess(to_matrix(dO, n, d), to_matrix(o, n, d)), out); });
}

int flref_flash_bwd(const double* q, const double* k, const double* v, const double* dO,
                    const double* o, const double* lse, std::size_t n, std::size_t d,
                    double alpha, int causal, std::size_t br, std::size_t bc, double* dq,
                    double* dk, double* dv) {
  return guarded([&] {
    const AttentionInputs in = inputs(q, k, v, n, d, alpha, causal);
    ForwardOutput fwd{to_matrix(o, n, d), std::vector<double>(lse, lse + n)};
    AttentionGrads g = flash_bwd(in, to_matrix(dO, n, d), fwd, TileConfig{br, bc});
    from_matrix(g.dq, dq);
    from_matrix(g.dk, dk);
    from_matrix(g.dv, dv);
  });
}

int flref_preprocess_incoherent(const double* q, const double* k, std::size_t n,
                                std::size_t d, uint64_t seed, double* qo, double* ko) {
  return guarded([&] {
    auto pr = preprocess_incoherent(to_matrix(q, n, d), to_matrix(k, n, d), seed);
    from_matrix(pr.first, qo);
    from_matrix(pr.second, ko);
  });
}

int flref_fwht(double* v, std::size_t n) {
  return guarded([&] { fwht(std::span<double>(v, n)); });
}

// block_rows 0 = per tensor. scales has ceil(rows/block_rows) (or 1) entries.
int flref_quantize(const double* m, std::size_t rows, std::size_t cols, std::size_t block_rows,
                   int overflow_infinite, double* codes, double* scales) {
  return guarded([&] {
    const auto ov = overflow_infinite ? OverflowPolicy::infinite : OverflowPolicy::saturate;
    QuantizedTensor t =
        block_rows == 0
            ? quantize_per_tensor(to_matrix(m, rows, cols), FloatFormatId::fp8e4m3, ov)
            : quantize_per_block(to_matrix(m, rows, cols), block_rows, FloatFormatId::fp8e4m3,
                                 ov);
    from_matrix(t.codes, codes);
    from_vec(t.scales, scales);
  });
}

// granularity: 0 per tensor, 1 per block.
int flref_fp8_flash_fwd(const double* q, const double* k, const double* v, std::size_t n,
                        std::size_t d, double alpha, int causal, int granularity,
                        int incoherent, uint64_t seed, std::size_t br, std::size_t bc,
                        int permuted, double* o, double* lse) {
  return guarded([&] {
    Fp8AttentionConfig cfg;
    cfg.granularity = granularity ? QuantGranularity::per_block : QuantGranularity::per_tensor;
    cfg.incoherent = incoherent != 0;
    cfg.seed = seed;
    cfg.tile = TileConfig{br, bc};
    cfg.permuted_value_layout = permuted != 0;
    ForwardOutput out = fp8_flash_fwd(inputs(q, k, v, n, d, alpha, causal), cfg);
    from_matrix(out.o, o);
    from_vec(out.logsumexp, lse);
  });
}

// fmt 2 = fp16, 4 = e4m3.
int flref_baseline_lowprec(const double* q, const double* k, const double* v, std::size_t n,
                           std::size_t d, double alpha, int causal, int fmt,
                           std::size_t block_rows, double* o, double* lse) {
  return guarded([&] {
    ForwardOutput out = baseline_lowprec_attention(inputs(q, k, v, n, d, alpha, causal),
                                                   static_cast<FloatFormatId>(fmt), block_rows);
    from_matrix(out.o, o);
    from_vec(out.logsumexp, lse);
  });
}

int flref_fp16_flash_fwd(const double* q, const double* k, const double* v, std::size_t n,
                         std::size_t d, double alpha, int causal, std::size_t br,
                         std::size_t bc, double* o, double* lse) {
  return guarded([&] {
    ForwardOutput out =
        fp16_flash_fwd(inputs(q, k, v, n, d, alpha, causal), TileConfig{br, bc});
    from_matrix(out.o, o);
    from_vec(out.logsumexp, lse);
  });
}

// Accumulator permutation / value-tile transpose (fp8_attention.cpp:44-75).
int flref_accumulator_permutation(std::size_t width, uint64_t* out) {
  return guarded([&] {
    const auto p = accumulator_permutation(width);
    for (std::size_t i = 0; i < p.size(); ++i) out[i] = p[i];
  });
}

}  // extern "C"
