// fa3b::flashlab — the reference attention API over the fa3b C ABI.
// See include/fa3b/flashlab_compat.hpp for the contract and deviations.
#include "fa3b/flashlab_compat.hpp"

#include <cuda_runtime_api.h>

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

// Status codes that are the reference's std::invalid_argument cases.
[[noreturn]] void throw_status(int rc) {
  const std::string msg = fa3b_error_string(rc);
  if (rc == FA3B_ERR_CUDA || rc == FA3B_ERR_DEVICE)
    throw std::runtime_error(msg + " (cudaError " + std::to_string(fa3b_last_cuda_error()) + ")");
  throw std::invalid_argument(msg);
}
void check(int rc) {
  if (rc != FA3B_OK) throw_status(rc);
}
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("fa3b::flashlab: ") + what + ": " + cudaGetErrorString(e));
}

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(std::size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc"); }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// Round-to-nearest-even onto a 16-bit format (formats.cpp:45-61 semantics,
// saturating); the result is exact in float, whose top bits give the code.
double round16(double x, int mant, int min_exp, double max_finite) {
  if (std::isnan(x) || x == 0.0 || std::isinf(x)) return x;
  const double ax = std::fabs(x);
  int e = std::ilogb(ax);
  if (e < min_exp) e = min_exp;
  const double q = std::ldexp(1.0, e - mant);
  double r = std::nearbyint(ax / q) * q;
  if (r > max_finite) r = max_finite;
  return std::copysign(r, x);
}
uint16_t to_bf16(double x) {
  const float f = static_cast<float>(round16(x, 7, -126, 0x1.FEp127));
  return static_cast<uint16_t>(std::bit_cast<uint32_t>(f) >> 16);
}
uint16_t to_f16(double x) {
  const _Float16 h = static_cast<_Float16>(static_cast<float>(round16(x, 10, -14, 65504.0)));
  return std::bit_cast<uint16_t>(h);
}

std::vector<uint16_t> pack16(const Matrix& m) {
  std::vector<uint16_t> out(m.size());
  const bool bf = g_format == DeviceFormat::bf16;
  for (std::size_t i = 0; i < m.size(); ++i) out[i] = bf ? to_bf16(m.data()[i]) : to_f16(m.data()[i]);
  return out;
}
int fmt_code() { return g_format == DeviceFormat::bf16 ? FA3B_DTYPE_BF16 : FA3B_DTYPE_F16; }

// one head, [1, n, 1, d] contiguous
fa3b_tensor4 t4(void* p, std::size_t n, std::size_t d) {
  return fa3b_tensor4{p, static_cast<int64_t>(n * d), static_cast<int64_t>(d), static_cast<int64_t>(d)};
}

template <class T>
void upload(void* dst, const std::vector<T>& v) {
  cuda_check(cudaMemcpy(dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
}
template <class T>
std::vector<T> download(const void* src, std::size_t n) {
  std::vector<T> v(n);
  cuda_check(cudaMemcpy(v.data(), src, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
  return v;
}

void check_tile(const TileConfig& cfg) {  // flash_fwd.cpp:127-129
  if (cfg.block_rows == 0 || cfg.block_cols == 0)
    throw std::invalid_argument("TileConfig: block sizes must be positive");
}

enum class Schedule { basic, two_stage, three_stage };

// FlashFwdStats as the reference's schedules report them (flash_fwd.cpp:110-215):
// pure functions of (n, tile, causal, schedule).
FlashFwdStats analytic_stats(std::size_t n, bool causal, const TileConfig& cfg, Schedule sched) {
  FlashFwdStats st;
  const std::size_t t_c = (n + cfg.block_cols - 1) / cfg.block_cols;
  Schedule eff = sched;
  if ((sched == Schedule::two_stage && t_c < 2) || (sched == Schedule::three_stage && t_c < 4)) {
    eff = Schedule::basic;
    st.fell_back_to_basic = true;
  }
  for (std::size_t r0 = 0; r0 < n; r0 += cfg.block_rows) {
    const std::size_t nr = std::min(cfg.block_rows, n - r0);
    std::size_t cnt = 0;
    for (std::size_t c0 = 0; c0 < n; c0 += cfg.block_cols) {
      if (causal && c0 > r0 + nr - 1) {
        ++st.blocks_skipped;
        continue;
      }
      ++cnt;
    }
    st.blocks_visited += cnt;
    if (eff == Schedule::two_stage && cnt >= 2) st.max_pending_scores = 1;
    if (eff == Schedule::three_stage && cnt >= 2) {
      st.deferred_output_scale = true;
      st.max_pending_scores = 1;
      if (cnt >= 3) st.max_live_probs = 2;
    }
  }
  return st;
}

ForwardOutput run_fwd(const AttentionInputs& in, const TileConfig& cfg, Schedule sched,
                      FlashFwdStats* stats) {
  validate_inputs(in);
  check_tile(cfg);
  const std::size_t n = in.q.rows(), d = in.q.cols();
  DevBuf q(n * d * 2), k(n * d * 2), v(n * d * 2), o(n * d * 4), lse(n * 4);
  upload(q.p, pack16(in.q));
  upload(k.p, pack16(in.k));
  upload(v.p, pack16(in.v));
  fa3b_fwd_params p{};
  p.struct_size = sizeof(p);
  p.batch = p.heads_q = p.heads_kv = 1;
  p.seqlen = static_cast<int32_t>(n);
  p.head_dim = static_cast<int32_t>(d);
  p.in_dtype = fmt_code();
  p.out_dtype = FA3B_DTYPE_F32;
  p.q = t4(q.p, n, d);
  p.k = t4(k.p, n, d);
  p.v = t4(v.p, n, d);
  p.o = t4(o.p, n, d);
  p.lse = static_cast<float*>(lse.p);
  p.alpha = in.alpha;
  p.causal = in.causal;
  p.schedule = sched == Schedule::basic ? FA3B_SCHED_BASIC
                                        : (sched == Schedule::two_stage ? FA3B_SCHED_PINGPONG
                                                                        : FA3B_SCHED_3STAGE);
  check(fa3b_fwd(&p));
  const auto of = download<float>(o.p, n * d);
  const auto lf = download<float>(lse.p, n);
  ForwardOutput out{Matrix(n, d), std::vector<double>(n)};
  for (std::size_t i = 0; i < n * d; ++i) out.o.data()[i] = of[i];
  for (std::size_t i = 0; i < n; ++i) out.logsumexp[i] = lf[i];
  if (stats) *stats = analytic_stats(n, in.causal, cfg, sched);
  return out;
}

bool pow2(std::size_t x) { return x != 0 && (x & (x - 1)) == 0; }

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

ForwardOutput flash_fwd_basic(const AttentionInputs& in, const TileConfig& cfg,
                              FlashFwdStats* stats) {
  return run_fwd(in, cfg, Schedule::basic, stats);
}
ForwardOutput flash_fwd_2stage(const AttentionInputs& in, const TileConfig& cfg,
                               FlashFwdStats* stats) {
  return run_fwd(in, cfg, Schedule::two_stage, stats);
}
ForwardOutput flash_fwd_3stage(const AttentionInputs& in, const TileConfig& cfg,
                               FlashFwdStats* stats) {
  return run_fwd(in, cfg, Schedule::three_stage, stats);
}

std::vector<double> bwd_preprocess(const Matrix& dO, const Matrix& o) {
  if (!dO.same_shape(o)) throw std::invalid_argument("bwd_preprocess: shape mismatch");
  const std::size_t n = o.rows(), d = o.cols();
  if (n == 0 || d == 0) return {};
  std::vector<float> of(n * d), gf(n * d);
  for (std::size_t i = 0; i < n * d; ++i) {
    of[i] = static_cast<float>(o.data()[i]);
    gf[i] = static_cast<float>(dO.data()[i]);
  }
  DevBuf od(n * d * 4), gd(n * d * 4), dd(n * 4);
  upload(od.p, of);
  upload(gd.p, gf);
  fa3b_bwd_preprocess_params p{};
  p.struct_size = sizeof(p);
  p.batch = p.heads = 1;
  p.seqlen = static_cast<int32_t>(n);
  p.head_dim = static_cast<int32_t>(d);
  p.dtype = FA3B_DTYPE_F32;
  p.o = t4(od.p, n, d);
  p.dout = t4(gd.p, n, d);
  p.delta = static_cast<float*>(dd.p);
  check(fa3b_bwd_preprocess(&p));
  const auto df = download<float>(dd.p, n);
  return std::vector<double>(df.begin(), df.end());
}

AttentionGrads flash_bwd(const AttentionInputs& in, const Matrix& dO, const ForwardOutput& fwd,
                         const TileConfig& cfg) {
  validate_inputs(in);  // flash_bwd.cpp:45-50
  check_tile(cfg);
  if (!dO.same_shape(in.q)) throw std::invalid_argument("flash_bwd: dO shape mismatch");
  if (!fwd.o.same_shape(dO) || fwd.logsumexp.size() != dO.rows())
    throw std::invalid_argument("flash_bwd: forward output shape mismatch");
  const std::size_t n = in.q.rows(), d = in.q.cols();
  DevBuf q(n * d * 2), k(n * d * 2), v(n * d * 2), o(n * d * 2), g(n * d * 2), lse(n * 4);
  DevBuf dq(n * d * 2), dk(n * d * 2), dv(n * d * 2);
  upload(q.p, pack16(in.q));
  upload(k.p, pack16(in.k));
  upload(v.p, pack16(in.v));
  upload(o.p, pack16(fwd.o));
  upload(g.p, pack16(dO));
  std::vector<float> lf(fwd.logsumexp.begin(), fwd.logsumexp.end());
  upload(lse.p, lf);
  const std::size_t wsb = fa3b_bwd_workspace_bytes(1, 1, 1, static_cast<int32_t>(n),
                                                   static_cast<int32_t>(d));
  DevBuf ws(wsb);
  fa3b_bwd_params p{};
  p.struct_size = sizeof(p);
  p.batch = p.heads_q = p.heads_kv = 1;
  p.seqlen = static_cast<int32_t>(n);
  p.head_dim = static_cast<int32_t>(d);
  p.dtype = fmt_code();
  p.q = t4(q.p, n, d);
  p.k = t4(k.p, n, d);
  p.v = t4(v.p, n, d);
  p.o = t4(o.p, n, d);
  p.dout = t4(g.p, n, d);
  p.dq = t4(dq.p, n, d);
  p.dk = t4(dk.p, n, d);
  p.dv = t4(dv.p, n, d);
  p.lse = static_cast<const float*>(lse.p);
  p.alpha = in.alpha;
  p.causal = in.causal;
  p.workspace = ws.p;
  p.workspace_bytes = wsb;
  check(fa3b_bwd(&p));
  AttentionGrads out{Matrix(n, d), Matrix(n, d), Matrix(n, d)};
  const bool bf = g_format == DeviceFormat::bf16;
  auto widen = [&](const void* src, Matrix& m) {
    const auto h = download<uint16_t>(src, n * d);
    for (std::size_t i = 0; i < n * d; ++i) {
      m.data()[i] = bf ? static_cast<double>(std::bit_cast<float>(static_cast<uint32_t>(h[i]) << 16))
                       : static_cast<double>(std::bit_cast<_Float16>(h[i]));
    }
  };
  widen(dq.p, out.dq);
  widen(dk.p, out.dk);
  widen(dv.p, out.dv);
  return out;
}

std::pair<Matrix, Matrix> preprocess_incoherent(const Matrix& q, const Matrix& k,
                                                std::uint64_t seed) {
  // fp8_attention.cpp:33-42. A host utility with the reference's FP64
  // arithmetic; on the FP8 hot path the same transform runs fused into the
  // device quantizer (fa3b_fp8_prepare).
  if (q.cols() != k.cols()) throw std::invalid_argument("preprocess_incoherent: column mismatch");
  const std::size_t d = q.cols();
  if (!pow2(d)) throw std::invalid_argument("random_dh_transform: dim must be a power of two");
  std::vector<double> signs(d);
  for (std::size_t i = 0; i < d; ++i) {  // rng.cpp:13-27,73-78
    std::uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    signs[i] = (z & 1ull) ? 1.0 : -1.0;
  }
  auto apply = [&](const Matrix& src) {
    Matrix m = src;
    const double norm = 1.0 / std::sqrt(static_cast<double>(d));
    for (std::size_t r = 0; r < m.rows(); ++r) {
      double* v = m.row_ptr(r);
      for (std::size_t i = 0; i < d; ++i) v[i] *= signs[i];
      for (std::size_t len = 1; len < d; len <<= 1)  // hadamard.cpp:11-27
        for (std::size_t i = 0; i < d; i += len << 1)
          for (std::size_t j = i; j < i + len; ++j) {
            const double a = v[j], b = v[j + len];
            v[j] = a + b;
            v[j + len] = a - b;
          }
      for (std::size_t i = 0; i < d; ++i) v[i] *= norm;
    }
    return m;
  };
  return {apply(q), apply(k)};
}

ForwardOutput fp8_flash_fwd(const AttentionInputs& in, const Fp8AttentionConfig& cfg) {
  validate_inputs(in);  // fp8_attention.cpp:77-86
  if (cfg.tile.block_rows == 0 || cfg.tile.block_cols == 0)
    throw std::invalid_argument("fp8_flash_fwd: tile sizes must be positive");
  const std::size_t n = in.q.rows(), d = in.q.cols();
  if (cfg.permuted_value_layout && (cfg.tile.block_cols % 16 != 0 || n % 16 != 0))
    throw std::invalid_argument(
        "fp8_flash_fwd: permuted layout needs block_cols and N divisible by 16");
  if (cfg.incoherent && !pow2(d))
    throw std::invalid_argument("random_dh_transform: dim must be a power of two");
  for (const Matrix* m : {&in.q, &in.k, &in.v})
    for (std::size_t i = 0; i < m->size(); ++i)
      if (!std::isfinite(m->data()[i])) throw std::invalid_argument("quantize: non-finite input entry");
  const int blk = cfg.granularity == QuantGranularity::per_block ? 128 : 0;
  const int nblk = blk ? static_cast<int>((n + 127) / 128) : 1;
  DevBuf src(n * d * 4), q8(n * d), k8(n * d), v8(n * d), o(n * d * 4), lse(n * 4);
  DevBuf sq(nblk * 4), sk(nblk * 4), sv(nblk * 4);
  auto prep = [&](const Matrix& m, void* dst, void* scales, bool hadamard) {
    std::vector<float> f(m.size());
    for (std::size_t i = 0; i < m.size(); ++i) f[i] = static_cast<float>(m.data()[i]);
    upload(src.p, f);
    fa3b_fp8_prepare_params p{};
    p.struct_size = sizeof(p);
    p.batch = p.heads = 1;
    p.seqlen = static_cast<int32_t>(n);
    p.head_dim = static_cast<int32_t>(d);
    p.src_dtype = FA3B_DTYPE_F32;
    p.src = t4(src.p, n, d);
    p.dst = t4(dst, n, d);
    p.scales = static_cast<float*>(scales);
    p.block_rows = blk;
    p.hadamard = hadamard;
    p.seed = cfg.seed;
    p.saturate = cfg.overflow == OverflowPolicy::saturate;
    check(fa3b_fp8_prepare(&p));
    cuda_check(cudaDeviceSynchronize(), "prepare");
  };
  prep(in.q, q8.p, sq.p, cfg.incoherent);
  prep(in.k, k8.p, sk.p, cfg.incoherent);
  prep(in.v, v8.p, sv.p, false);
  fa3b_fwd_params p{};
  p.struct_size = sizeof(p);
  p.batch = p.heads_q = p.heads_kv = 1;
  p.seqlen = static_cast<int32_t>(n);
  p.head_dim = static_cast<int32_t>(d);
  p.in_dtype = FA3B_DTYPE_E4M3;
  p.out_dtype = FA3B_DTYPE_F32;
  p.q = t4(q8.p, n, d);
  p.k = t4(k8.p, n, d);
  p.v = t4(v8.p, n, d);
  p.o = t4(o.p, n, d);
  p.lse = static_cast<float*>(lse.p);
  p.alpha = in.alpha;
  p.causal = in.causal;
  p.q_scale = static_cast<const float*>(sq.p);
  p.k_scale = static_cast<const float*>(sk.p);
  p.v_scale = static_cast<const float*>(sv.p);
  p.q_block_rows = p.kv_block_rows = blk;
  check(fa3b_fwd(&p));
  const auto of = download<float>(o.p, n * d);
  const auto lf = download<float>(lse.p, n);
  ForwardOutput out{Matrix(n, d), std::vector<double>(n)};
  for (std::size_t i = 0; i < n * d; ++i) out.o.data()[i] = of[i];
  for (std::size_t i = 0; i < n; ++i) out.logsumexp[i] = lf[i];
  return out;
}

}  // namespace flashlab
}  // namespace fa3b
