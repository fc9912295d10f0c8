// Tests of fa3b::flashlab, the reference API over the B200 kernels, written
// like the reference's own suites (proj/tests/test_flash_fwd.cpp,
// test_flash_bwd.cpp, test_fp8_attention.cpp) but with device tolerances.
// The FP64 oracle here is a naive dense attention (independent of the oracle
// library, like the reference's test_util.hpp matmul_oracle).
//
//   test_flashlab_compat --validation-only   argument checks, no device
//   test_flashlab_compat                     everything (needs the B200)
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>

#include "fa3b/flashlab_compat.hpp"

namespace fl = fa3b::flashlab;

static int g_fail = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
      ++g_fail;                                                            \
    }                                                                      \
  } while (0)

template <class F>
static void check_throws(F&& f, const char* msg) {
  try {
    f();
  } catch (const std::invalid_argument& e) {
    if (std::string(e.what()).find(msg) == std::string::npos) {
      std::fprintf(stderr, "wrong message: '%s' (want '%s')\n", e.what(), msg);
      ++g_fail;
    }
    return;
  }
  std::fprintf(stderr, "no std::invalid_argument for '%s'\n", msg);
  ++g_fail;
}

static fl::Matrix gaussian(std::size_t r, std::size_t c, unsigned seed) {
  std::mt19937_64 g(seed);
  std::normal_distribution<double> n(0.0, 1.0);
  fl::Matrix m(r, c);
  for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] = n(g);
  return m;
}

// RNE to bf16 (the default device format), so the FP64 oracle sees exactly the
// values the kernels see (the reference's tests round with round_to the same way)
static fl::Matrix bf16_rounded(fl::Matrix m) {
  for (std::size_t i = 0; i < m.size(); ++i) {
    float f = static_cast<float>(m.data()[i]);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    std::memcpy(&f, &u, 4);
    m.data()[i] = f;
  }
  return m;
}

struct Dense {
  fl::Matrix o, p;
  std::vector<double> lse;
};
static Dense dense_fwd(const fl::AttentionInputs& in) {
  const std::size_t n = in.q.rows(), d = in.q.cols();
  Dense r{fl::Matrix(n, d), fl::Matrix(n, n), std::vector<double>(n)};
  for (std::size_t i = 0; i < n; ++i) {
    double m = -INFINITY;
    for (std::size_t j = 0; j < n; ++j) {
      double s = 0;
      for (std::size_t t = 0; t < d; ++t) s += in.q(i, t) * in.k(j, t);
      s = (in.causal && j > i) ? -INFINITY : s * in.alpha;
      r.p(i, j) = s;
      m = std::max(m, s);
    }
    double l = 0;
    for (std::size_t j = 0; j < n; ++j) l += (r.p(i, j) = std::exp(r.p(i, j) - m));
    for (std::size_t j = 0; j < n; ++j) r.p(i, j) /= l;
    r.lse[i] = m + std::log(l);
    for (std::size_t j = 0; j < n; ++j)
      for (std::size_t t = 0; t < d; ++t) r.o(i, t) += r.p(i, j) * in.v(j, t);
  }
  return r;
}
static double rel_rms(const fl::Matrix& a, const fl::Matrix& b) {
  double e = 0, s = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    e += (a.data()[i] - b.data()[i]) * (a.data()[i] - b.data()[i]);
    s += b.data()[i] * b.data()[i];
  }
  return std::sqrt(e / s);
}

static void validation_tests() {
  const fl::Matrix a = gaussian(8, 4, 1);
  auto in = fl::attention_inputs(a, a, a);
  CHECK(std::fabs(in.alpha - 0.5) < 1e-15);
  check_throws([&] { fl::flash_fwd_basic(fl::AttentionInputs{}, {}); }, "attention: empty inputs");
  check_throws([&] { fl::flash_fwd_2stage(fl::attention_inputs(a, gaussian(8, 3, 2), a), {}); },
               "attention: head dimension mismatch");
  check_throws([&] { fl::flash_fwd_3stage(fl::attention_inputs(a, gaussian(7, 4, 2), a), {}); },
               "attention: sequence length mismatch");
  auto bad = in;
  bad.alpha = 0.0;
  check_throws([&] { fl::flash_fwd_basic(bad, {}); }, "alpha must be finite and nonzero");
  check_throws([&] { fl::flash_fwd_basic(in, {0, 8}); }, "TileConfig: block sizes must be positive");
  const fl::ForwardOutput fake{a, std::vector<double>(8)};
  check_throws([&] { fl::flash_bwd(in, gaussian(7, 4, 3), fake, {}); }, "flash_bwd: dO shape mismatch");
  fl::ForwardOutput trimmed = fake;
  trimmed.logsumexp.pop_back();
  check_throws([&] { fl::flash_bwd(in, a, trimmed, {}); }, "flash_bwd: forward output shape mismatch");
  check_throws([&] { fl::gqa_head_map(6, 4); }, "gqa_head_map: heads must be a multiple of kv_heads");
  CHECK(fl::gqa_head_map(16, 4)[5] == 1);
  fl::Fp8AttentionConfig cfg;
  cfg.permuted_value_layout = true;
  cfg.tile = {16, 24};
  check_throws([&] { fl::fp8_flash_fwd(in, cfg); }, "permuted layout needs block_cols");
  fl::Fp8AttentionConfig c2;
  check_throws([&] { fl::fp8_flash_fwd(fl::attention_inputs(gaussian(8, 24, 1), gaussian(8, 24, 2),
                                                            gaussian(8, 24, 3)), c2); },
               "random_dh_transform: dim must be a power of two");
  static_assert(fl::flops_forward(512, 64, 32, false) == 2147483648ull);
  static_assert(fl::flops_forward(512, 64, 32, true) == 1073741824ull);
  static_assert(fl::flops_backward(512, 64, 32, false) == 2147483648ull * 5 / 2);
  // incoherent preprocessing preserves QK^T (test_fp8_attention.cpp:46-55)
  const fl::Matrix q = gaussian(16, 64, 5), k = gaussian(16, 64, 6);
  auto [qp, kp] = fl::preprocess_incoherent(q, k, 11);
  double worst = 0;
  for (std::size_t i = 0; i < 16; ++i)
    for (std::size_t j = 0; j < 16; ++j) {
      double s0 = 0, s1 = 0;
      for (std::size_t t = 0; t < 64; ++t) s0 += q(i, t) * k(j, t), s1 += qp(i, t) * kp(j, t);
      worst = std::max(worst, std::fabs(s0 - s1));
    }
  CHECK(worst <= 1e-10);
}

static void device_tests() {
  // forward, three schedules, causal + ragged (test_flash_fwd.cpp:106-118)
  for (bool causal : {false, true}) {
    auto in = fl::attention_inputs(bf16_rounded(gaussian(300, 64, 10)), bf16_rounded(gaussian(300, 64, 11)),
                                   bf16_rounded(gaussian(300, 64, 12)), causal);
    const Dense ref = dense_fwd(in);
    for (int sched = 0; sched < 3; ++sched) {
      const fl::ForwardOutput out = sched == 0   ? fl::flash_fwd_basic(in, {64, 64})
                                    : sched == 1 ? fl::flash_fwd_2stage(in, {64, 64})
                                                 : fl::flash_fwd_3stage(in, {64, 64});
      CHECK(rel_rms(out.o, ref.o) < 1e-2);
      double lerr = 0;
      for (std::size_t i = 0; i < 300; ++i) lerr = std::max(lerr, std::fabs(out.logsumexp[i] - ref.lse[i]));
      CHECK(lerr < 1e-3);
      if (lerr >= 1e-3) std::fprintf(stderr, "  causal=%d sched=%d max|dLSE|=%g\n", causal, sched, lerr);
    }
  }
  // structural probes (test_flash_fwd.cpp:139-150)
  {
    auto in = fl::attention_inputs(gaussian(128, 64, 1), gaussian(128, 64, 2), gaussian(128, 64, 3), true);
    fl::FlashFwdStats st;
    fl::flash_fwd_basic(in, {32, 32}, &st);
    CHECK(st.blocks_visited == 10 && st.blocks_skipped == 6);
    fl::flash_fwd_2stage(in, {32, 32}, &st);
    CHECK(st.max_pending_scores == 1 && !st.fell_back_to_basic);
    fl::flash_fwd_3stage(in, {32, 32}, &st);
    CHECK(st.deferred_output_scale && st.max_live_probs == 2);
    fl::flash_fwd_2stage(fl::attention_inputs(gaussian(16, 64, 1), gaussian(16, 64, 2), gaussian(16, 64, 3)),
                         {16, 32}, &st);
    CHECK(st.fell_back_to_basic);
  }
  // backward vs dense gradients (test_flash_bwd.cpp:68-80), zero dO (:56-66)
  for (bool causal : {false, true}) {
    const std::size_t n = 200, d = 128;
    auto in = fl::attention_inputs(gaussian(n, d, 20), gaussian(n, d, 21), gaussian(n, d, 22), causal);
    const fl::Matrix dO = gaussian(n, d, 23);
    const Dense ref = dense_fwd(in);
    fl::Matrix dv(n, d), dq(n, d), dk(n, d), dp(n, n), ds(n, n);
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = 0; j < n; ++j)
        for (std::size_t t = 0; t < d; ++t) dp(i, j) += dO(i, t) * in.v(j, t);
    for (std::size_t i = 0; i < n; ++i) {
      double dot = 0;
      for (std::size_t j = 0; j < n; ++j) dot += ref.p(i, j) * dp(i, j);
      for (std::size_t j = 0; j < n; ++j) ds(i, j) = ref.p(i, j) * (dp(i, j) - dot);
    }
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = 0; j < n; ++j)
        for (std::size_t t = 0; t < d; ++t) {
          dv(j, t) += ref.p(i, j) * dO(i, t);
          dq(i, t) += in.alpha * ds(i, j) * in.k(j, t);
          dk(j, t) += in.alpha * ds(i, j) * in.q(i, t);
        }
    const fl::ForwardOutput fwd = fl::flash_fwd_2stage(in, {});
    const fl::AttentionGrads g = fl::flash_bwd(in, dO, fwd, {});
    CHECK(rel_rms(g.dq, dq) < 2e-2);
    CHECK(rel_rms(g.dk, dk) < 2e-2);
    CHECK(rel_rms(g.dv, dv) < 2e-2);
    const fl::AttentionGrads z = fl::flash_bwd(in, fl::Matrix(n, d), fwd, {});
    for (std::size_t i = 0; i < n * d; ++i) CHECK(z.dq.data()[i] == 0 && z.dk.data()[i] == 0 && z.dv.data()[i] == 0);
    const auto D = fl::bwd_preprocess(dO, fwd.o);
    double dmax = 0;
    for (std::size_t i = 0; i < n; ++i) {
      double acc = 0;
      for (std::size_t t = 0; t < d; ++t) acc += dO(i, t) * fwd.o(i, t);
      dmax = std::max(dmax, std::fabs(acc - D[i]));
    }
    CHECK(dmax < 1e-3);
  }
  // fp8 forward within an 8-bit error band (test_fp8_attention.cpp:118-143)
  {
    auto in = fl::attention_inputs(gaussian(512, 128, 30), gaussian(512, 128, 31), gaussian(512, 128, 32));
    const Dense ref = dense_fwd(in);
    fl::Fp8AttentionConfig cfg;
    cfg.seed = 7;
    const fl::ForwardOutput out = fl::fp8_flash_fwd(in, cfg);
    const double e = rel_rms(out.o, ref.o);
    CHECK(e > 1e-3 && e < 1e-1);
  }
  // fp16 device format
  fl::set_device_format(fl::DeviceFormat::f16);
  {
    auto in = fl::attention_inputs(gaussian(256, 64, 40), gaussian(256, 64, 41), gaussian(256, 64, 42), true);
    CHECK(rel_rms(fl::flash_fwd_basic(in, {}).o, dense_fwd(in).o) < 5e-3);
  }
  fl::set_device_format(fl::DeviceFormat::bf16);
}

int main(int argc, char** argv) {
  const bool validation_only = argc > 1 && std::strcmp(argv[1], "--validation-only") == 0;
  validation_tests();
  if (!validation_only) device_tests();
  std::printf("%s: %d failure(s)\n", validation_only ? "validation" : "all", g_fail);
  return g_fail ? 1 : 0;
}
