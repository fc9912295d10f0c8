// fa3b::flashlab — the reference attention API over the fa3b C ABI, as a
// source-level mirror (include/fa3b/flashlab_compat.hpp: the same types in
// namespace fa3b::flashlab). The entry points themselves are flashlab_core.inc,
// shared with the link-level drop-in (flashlab_dropin.cpp).
#include "fa3b/flashlab_compat.hpp"

#include <cuda_runtime_api.h>

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>

#include "fa3b.h"

namespace fa3b {
namespace flashlab {

namespace {
DeviceFormat g_format = DeviceFormat::bf16;
bool fmt_is_bf16() { return g_format == DeviceFormat::bf16; }
}  // namespace

Matrix::Matrix(std::size_t rows, std::size_t cols, std::initializer_list<double> vals)
    : rows_(rows), cols_(cols), data_(vals) {
  if (data_.size() != rows * cols)
    throw std::invalid_argument("Matrix: initializer size " + std::to_string(data_.size()) +
                                " does not match " + std::to_string(rows) + "x" +
                                std::to_string(cols));
}

Matrix Matrix::identity(std::size_t n) {
  Matrix m(n, n);
  for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
  return m;
}

void set_device_format(DeviceFormat f) { g_format = f; }
DeviceFormat device_format() { return g_format; }

AttentionInputs attention_inputs(Matrix q, Matrix k, Matrix v, bool causal) {
  const double alpha = 1.0 / std::sqrt(static_cast<double>(q.cols()));
  return AttentionInputs{std::move(q), std::move(k), std::move(v), alpha, causal};
}

void validate_inputs(const AttentionInputs& in) {  // attention_ref.cpp:20-29
  if (in.q.rows() == 0 || in.q.cols() == 0) throw std::invalid_argument("attention: empty inputs");
  if (in.q.cols() != in.k.cols() || in.k.cols() != in.v.cols())
    throw std::invalid_argument("attention: head dimension mismatch");
  if (in.q.rows() != in.k.rows() || in.k.rows() != in.v.rows())
    throw std::invalid_argument("attention: sequence length mismatch");
  if (!std::isfinite(in.alpha) || in.alpha == 0.0)
    throw std::invalid_argument("attention: alpha must be finite and nonzero");
}

std::vector<std::size_t> gqa_head_map(std::size_t heads, std::size_t kv_heads) {
  if (heads == 0 || kv_heads == 0 || heads % kv_heads != 0)
    throw std::invalid_argument("gqa_head_map: heads must be a multiple of kv_heads");
  std::vector<std::size_t> map(heads);
  for (std::size_t h = 0; h < heads; ++h) map[h] = h / (heads / kv_heads);
  return map;
}

#include "flashlab_core.inc"

}  // namespace flashlab
}  // namespace fa3b
