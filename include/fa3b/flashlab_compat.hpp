#pragma once
// fa3b::flashlab — the reference library's attention API (flashlab, proj/core)
// served by the B200 kernels behind include/fa3b.h.
//
// A caller of the reference switches by namespace: flashlab::flash_fwd_2stage
// -> fa3b::flashlab::flash_fwd_2stage, same types, same signatures, same
// std::invalid_argument messages. Mirrored declarations (reference file:line):
//   AttentionInputs / attention_inputs / validate_inputs  attention_ref.hpp:15-26
//   ForwardOutput / AttentionGrads                         attention_ref.hpp:28-44
//   gqa_head_map                                           attention_ref.hpp:57
//   TileConfig / FlashFwdStats                             flash_fwd.hpp:21-52
//   flash_fwd_basic / _2stage / _3stage                    flash_fwd.hpp:54-65
//   flops_forward / flops_backward                         flash_fwd.hpp:69-77
//   bwd_preprocess / flash_bwd                             flash_bwd.hpp:15-21
//   QuantGranularity / Fp8AttentionConfig                  fp8_attention.hpp:27-38
//   preprocess_incoherent / fp8_flash_fwd                  fp8_attention.hpp:41-46
//   SoftmaxState / SoftmaxStep / online_softmax_step       flash_fwd.hpp:26-41
//   accumulator_permutation / permute_accumulator /
//     vtile_transpose                                      fp8_attention.hpp:50-57
// A link-level drop-in built against the reference's own headers (no namespace
// switch at all) is paper_2407_08608_b200/dropin/ (INTEGRATION.md).
//
// Semantics that differ, by design:
//   - FP64 inputs are rounded to the device format (bf16 by default, see
//     set_device_format) and the kernels compute with fp32 accumulation; O
//     and L come back as fp32 values on the FP64 carrier. Results match the
//     reference within the tolerances stated in tests/, not bit for bit.
//   - TileConfig is validated (zero sizes throw as in the reference) and
//     drives FlashFwdStats, but the device tiles are always 128 x 128.
//   - head dims are 64, 128, 256 (backward: 64, 128; FP8: 128, 256).
//   - fp8_flash_fwd quantizes in 128-row blocks regardless of cfg.tile and
//     needs no permuted value layout on sm_100a (the flag is validated only).
// Each call copies one head to the device, runs, and copies back; batch many
// heads through include/fa3b.h directly for throughput.

#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <utility>
#include <vector>

namespace fa3b {
namespace flashlab {

class Matrix {
 public:
  Matrix() = default;
  Matrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), data_(rows * cols, 0.0) {}
  Matrix(std::size_t rows, std::size_t cols, std::initializer_list<double> vals);
  static Matrix identity(std::size_t n);

  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  std::size_t size() const { return data_.size(); }
  bool empty() const { return data_.empty(); }
  double operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
  double& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
  double* row_ptr(std::size_t i) { return data_.data() + i * cols_; }
  const double* row_ptr(std::size_t i) const { return data_.data() + i * cols_; }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  bool same_shape(const Matrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

struct AttentionInputs {
  Matrix q, k, v;
  double alpha = 0.0;
  bool causal = false;
};
AttentionInputs attention_inputs(Matrix q, Matrix k, Matrix v, bool causal = false);
void validate_inputs(const AttentionInputs& in);

struct ForwardOutput {
  Matrix o;
  std::vector<double> logsumexp;
};
struct AttentionGrads {
  Matrix dq, dk, dv;
};
std::vector<std::size_t> gqa_head_map(std::size_t heads, std::size_t kv_heads);

struct TileConfig {
  std::size_t block_rows = 64;
  std::size_t block_cols = 64;
};
// flash_fwd.hpp:26-41: the online-softmax state and one block step, the
// reference's host building block (the device kernels fuse it).
struct SoftmaxState {
  std::vector<double> row_max;
  std::vector<double> row_sum;
  explicit SoftmaxState(std::size_t rows);
};
struct SoftmaxStep {
  Matrix p_tilde;
  std::vector<double> rescale;
};
SoftmaxStep online_softmax_step(SoftmaxState& state, const Matrix& s_block);

struct FlashFwdStats {
  std::size_t blocks_visited = 0;
  std::size_t blocks_skipped = 0;
  std::size_t max_pending_scores = 0;
  std::size_t max_live_probs = 0;
  bool deferred_output_scale = false;
  bool fell_back_to_basic = false;
};

ForwardOutput flash_fwd_basic(const AttentionInputs& in, const TileConfig& cfg,
                              FlashFwdStats* stats = nullptr);
ForwardOutput flash_fwd_2stage(const AttentionInputs& in, const TileConfig& cfg,
                               FlashFwdStats* stats = nullptr);
ForwardOutput flash_fwd_3stage(const AttentionInputs& in, const TileConfig& cfg,
                               FlashFwdStats* stats = nullptr);

constexpr std::uint64_t flops_forward(std::uint64_t seqlen, std::uint64_t headdim,
                                      std::uint64_t heads, bool causal) {
  const std::uint64_t f = 4ull * seqlen * seqlen * headdim * heads;
  return causal ? f / 2 : f;
}
constexpr std::uint64_t flops_backward(std::uint64_t seqlen, std::uint64_t headdim,
                                       std::uint64_t heads, bool causal) {
  return flops_forward(seqlen, headdim, heads, causal) * 5 / 2;
}

std::vector<double> bwd_preprocess(const Matrix& dO, const Matrix& o);
AttentionGrads flash_bwd(const AttentionInputs& in, const Matrix& dO, const ForwardOutput& fwd,
                         const TileConfig& cfg);

enum class QuantGranularity { per_tensor, per_block };
enum class OverflowPolicy { saturate, infinite };
struct Fp8AttentionConfig {
  QuantGranularity granularity = QuantGranularity::per_block;
  bool incoherent = true;
  std::uint64_t seed = 0;
  TileConfig tile{64, 64};
  OverflowPolicy overflow = OverflowPolicy::saturate;
  bool permuted_value_layout = false;
};
std::pair<Matrix, Matrix> preprocess_incoherent(const Matrix& q, const Matrix& k,
                                                std::uint64_t seed);
ForwardOutput fp8_flash_fwd(const AttentionInputs& in, const Fp8AttentionConfig& cfg);
// fp8_attention.hpp:50-57: the Hopper accumulator layout helpers (host only;
// sm_100a consumes V MN-major, so the device needs neither).
std::vector<std::size_t> accumulator_permutation(std::size_t width);
Matrix permute_accumulator(const Matrix& block);
Matrix vtile_transpose(const Matrix& vblock, bool permute_rows = false);

// Device format the FP64 inputs are rounded to (f16 or bf16; default bf16).
enum class DeviceFormat { f16, bf16 };
void set_device_format(DeviceFormat f);
DeviceFormat device_format();

}  // namespace flashlab
}  // namespace fa3b
