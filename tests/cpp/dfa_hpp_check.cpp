// C++ drop-in check for include/dfa.hpp, written like the reference's own
// tests (test_attention.cpp).  Host part runs anywhere (no kernel launch);
// `gpu <dir>` also runs dfa::dilated_attention on host tensors and dumps
// q, k, v, out (float32, raw) into <dir> for tests/test_cpp_api.py to check
// against the oracle.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "dfa.hpp"

// Minimal stand-in with attnkit::Tensor<double>'s rank-2 surface (f64 mode).
struct TensorD {
  std::vector<dfa::Index> shape;
  std::vector<double> buf;
  explicit TensorD(std::vector<dfa::Index> s) : shape(std::move(s)), buf(static_cast<size_t>(shape[0] * shape[1])) {}
  dfa::Index rows() const { return shape[0]; }
  dfa::Index cols() const { return shape[1]; }
  double* data() { return buf.data(); }
  const double* data() const { return buf.data(); }
};

// Minimal stand-in with attnkit::Tensor's rank-2 surface.
struct Tensor {
  std::vector<dfa::Index> shape;
  std::vector<float> buf;
  explicit Tensor(std::vector<dfa::Index> s) : shape(std::move(s)), buf(static_cast<size_t>(shape[0] * shape[1])) {}
  dfa::Index rank() const { return static_cast<dfa::Index>(shape.size()); }
  dfa::Index rows() const { return shape[0]; }
  dfa::Index cols() const { return shape[1]; }
  float* data() { return buf.data(); }
  const float* data() const { return buf.data(); }
};

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      ++failures;                                                     \
    }                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, T)        \
  do {                                  \
    bool ok = false;                    \
    try {                               \
      expr;                             \
    } catch (const T&) {                \
      ok = true;                        \
    } catch (...) {                     \
    }                                   \
    CHECK(ok && #expr " throws " #T);   \
  } while (0)

static dfa::AttentionConfig basic_cfg(dfa::Index n, dfa::Index w, dfa::Index r, int h = 1, dfa::Index d = 4) {
  dfa::AttentionConfig cfg;
  cfg.seq_len = n;
  cfg.segment_len = w;
  cfg.interval = r;
  cfg.num_heads = h;
  cfg.head_dim = d;
  cfg.head_offsets = dfa::AttentionConfig::spread_offsets(h, r);
  return cfg;
}

static void host_checks() {
  // test_attention.cpp:36-54
  CHECK_THROWS_AS(basic_cfg(8, 9, 1).validate(), dfa::config_error);
  CHECK_THROWS_AS(basic_cfg(8, 4, 5).validate(), dfa::config_error);
  CHECK_THROWS_AS(basic_cfg(0, 4, 2).validate(), dfa::config_error);
  auto cfg = basic_cfg(8, 4, 2);
  cfg.head_offsets = {2};
  CHECK_THROWS_AS(cfg.validate(), dfa::config_error);
  cfg.head_offsets = {0, 0};
  CHECK_THROWS_AS(cfg.validate(), dfa::config_error);
  auto cov = basic_cfg(8, 4, 2, 2);
  cov.head_offsets = {0, 0};
  cov.validate(false);
  CHECK_THROWS_AS(cov.validate(true), dfa::config_error);
  // test_attention.cpp:148-210
  CHECK((dfa::make_segment_view(8, 4, 2, 1, 0).row_indices == std::vector<dfa::Index>{4, 6}));
  CHECK((dfa::make_segment_view(8, 4, 1, 0, 0).row_indices == std::vector<dfa::Index>{0, 1, 2, 3}));
  CHECK((dfa::make_segment_view(10, 4, 2, 2, 1).row_indices == std::vector<dfa::Index>{9}));
  CHECK_THROWS_AS(dfa::make_segment_view(8, 4, 2, 2, 0), std::out_of_range);
  CHECK_THROWS_AS(dfa::make_segment_view(8, 4, 2, -1, 0), std::out_of_range);
  CHECK_THROWS_AS(dfa::make_segment_view(8, 4, 2, 0, 2), std::out_of_range);
  // test_attention.cpp:444-482
  auto fc = dfa::flop_count(basic_cfg(4096, 512, 2, 1, 64));
  CHECK(fc.dense_mults == 2ull * 4096 * 4096 * 64);
  CHECK(fc.dilated_mults == 8ull * 2 * 256 * 256 * 64);
  CHECK(fc.ratio == 32.0);
  CHECK(dfa::flop_count(basic_cfg(4096, 2048, 2, 1, 64)).ratio == 8.0);
  CHECK(dfa::flop_csv_header() == "N,w,r,h,d,dense_mults,dilated_mults,ratio");
  CHECK(dfa::flop_csv_row(basic_cfg(4096, 512, 2, 1, 64), fc) == "4096,512,2,1,64,2147483648,67108864,32");
}

static void dump(const std::string& path, const Tensor& t) {
  FILE* f = std::fopen(path.c_str(), "wb");
  std::fwrite(t.data(), sizeof(float), t.buf.size(), f);
  std::fclose(f);
}

static void gpu_checks(const std::string& dir) {
  std::mt19937_64 rng(901);
  std::normal_distribution<double> nd;
  auto randn = [&](dfa::Index r, dfa::Index c) {
    Tensor t({r, c});
    for (auto& x : t.buf) x = static_cast<float>(nd(rng));
    return t;
  };
  const auto cfg = basic_cfg(4096, 512, 2, 1, 64);
  auto q = randn(4096, 64), k = randn(4096, 64), v = randn(4096, 64);
  Tensor out = dfa::dilated_attention(q, k, v, cfg, 1);
  dump(dir + "/q.f32", q);
  dump(dir + "/k.f32", k);
  dump(dir + "/v.f32", v);
  dump(dir + "/o.f32", out);
  // rows of the other offset class are exact zeros (attention.hpp:243-245)
  for (dfa::Index i = 0; i < 4096; i += 2)
    for (dfa::Index c = 0; c < 64; ++c) CHECK(out.buf[static_cast<size_t>(i * 64 + c)] == 0.0f);
  // f64 tensors (the reference's double mode) run the f64 kernel: same
  // result as the fp32 call within fp32's resolution
  {
    TensorD qd({4096, 64}), kd({4096, 64}), vd({4096, 64});
    for (size_t i = 0; i < qd.buf.size(); ++i) {
      qd.buf[i] = q.buf[i];
      kd.buf[i] = k.buf[i];
      vd.buf[i] = v.buf[i];
    }
    TensorD od = dfa::dilated_attention(qd, kd, vd, cfg, 1);
    double worst = 0;
    for (size_t i = 0; i < od.buf.size(); ++i) worst = std::fmax(worst, std::fabs(od.buf[i] - out.buf[i]));
    CHECK(worst <= 1e-4);
    for (dfa::Index i = 0; i < 4096; i += 2)
      for (dfa::Index c = 0; c < 64; ++c) CHECK(od.buf[static_cast<size_t>(i * 64 + c)] == 0.0);
  }
  // error paths keep the reference's exception types
  CHECK_THROWS_AS(dfa::dilated_attention(q, k, v, cfg, 2), std::out_of_range);
  Tensor bad({4095, 64});
  CHECK_THROWS_AS(dfa::dilated_attention(bad, k, v, cfg, 0), dfa::dimension_error);
  // fault hook demonstrably perturbs the output
  {
    dfa::fault::ScopedPerturb armed;
    Tensor p = dfa::dilated_attention(q, k, v, cfg, 1);
    CHECK(p.buf[0] != out.buf[0]);
  }

  // multi_head_dilated (attention.hpp:340-360) with MultiHeadWeights' shape:
  // N = 256, D = 128, h = 2 (d = 64), (w, r) = (64, 2); dumped for the test
  struct Weights {
    std::vector<Tensor> wq, wk, wv;
    Tensor wo{{128, 128}};
  } w;
  const auto mcfg = basic_cfg(256, 64, 2, 2, 64);
  for (int j = 0; j < 2; ++j) {
    w.wq.push_back(randn(128, 64));
    w.wk.push_back(randn(128, 64));
    w.wv.push_back(randn(128, 64));
  }
  w.wo = randn(128, 128);
  for (auto* t : {&w.wo}) for (auto& x : t->buf) x /= std::sqrt(128.0f);
  for (auto& vec : {&w.wq, &w.wk, &w.wv})
    for (auto& t : *vec) for (auto& x : t.buf) x /= std::sqrt(128.0f);
  auto x = randn(256, 128);
  Tensor y = dfa::multi_head_dilated(x, w, mcfg);
  dump(dir + "/mh_x.f32", x);
  for (int j = 0; j < 2; ++j) {
    dump(dir + "/mh_wq" + std::to_string(j) + ".f32", w.wq[j]);
    dump(dir + "/mh_wk" + std::to_string(j) + ".f32", w.wk[j]);
    dump(dir + "/mh_wv" + std::to_string(j) + ".f32", w.wv[j]);
  }
  dump(dir + "/mh_wo.f32", w.wo);
  dump(dir + "/mh_y.f32", y);
  // full coverage is required, as in the reference (attention.hpp:343)
  auto partial = basic_cfg(256, 64, 4, 2, 64);
  CHECK_THROWS_AS(dfa::multi_head_dilated(x, w, partial), dfa::config_error);
  Tensor badx({255, 128});
  CHECK_THROWS_AS(dfa::multi_head_dilated(badx, w, mcfg), dfa::dimension_error);
}

// ---------------------------------------------------------------------------
// The reference's acceptance gates 1, 3 and 8 (proj/tests/acceptance.cpp:57-84,
// :119-138, :398-416) with every dilated_attention call routed through
// dfa::dilated_attention -- the swap INTEGRATION.md describes.  Same seeds,
// loops, draws (tensor.hpp:369-376 randn: normal_distribution<double> on
// mt19937_64, cast to Scalar) and tolerances; the comparison oracles are
// restated from oracles.hpp:67-107 (masked_dense_dilated) and
// attention.hpp:119-127 (naive_attention via tensor.hpp matmul / softmax_rows).
template <class T, class S>
static T ref_randn(dfa::Index r, dfa::Index c, std::mt19937_64& rng) {
  T t({r, c});
  std::normal_distribution<double> dist(0.0, 1.0);
  for (auto& x : t.buf) x = static_cast<S>(dist(rng));
  return t;
}

static dfa::AttentionConfig attn_cfg(dfa::Index n, dfa::Index w, dfa::Index r, dfa::Index d, dfa::Index gamma) {
  dfa::AttentionConfig cfg;
  cfg.seq_len = n;
  cfg.segment_len = w;
  cfg.interval = r;
  cfg.num_heads = 1;
  cfg.head_dim = d;
  cfg.head_offsets = {gamma};
  return cfg;
}

// oracles.hpp:67-107
static TensorD masked_dense(const TensorD& q, const TensorD& k, const TensorD& v, const dfa::AttentionConfig& cfg,
                            dfa::Index gamma) {
  const dfa::Index n = cfg.seq_len, d = q.cols(), dv = v.cols();
  std::vector<dfa::Index> group(static_cast<size_t>(n), -1);
  for (dfa::Index i = 0; i < cfg.num_segments(); ++i)
    for (dfa::Index r : dfa::make_segment_view(n, cfg.segment_len, cfg.interval, i, gamma).row_indices)
      group[static_cast<size_t>(r)] = i;
  const double sc = 1.0 / std::sqrt(static_cast<double>(d));
  TensorD out({n, dv});
  for (dfa::Index i = 0; i < n; ++i) {
    if (group[static_cast<size_t>(i)] < 0) continue;
    std::vector<double> s(static_cast<size_t>(n), -INFINITY);
    double m = -INFINITY;
    for (dfa::Index j = 0; j < n; ++j) {
      if (group[static_cast<size_t>(j)] != group[static_cast<size_t>(i)]) continue;
      double acc = 0;
      for (dfa::Index c = 0; c < d; ++c) acc += q.buf[static_cast<size_t>(i * d + c)] * k.buf[static_cast<size_t>(j * d + c)];
      s[static_cast<size_t>(j)] = acc * sc;
      m = std::max(m, s[static_cast<size_t>(j)]);
    }
    double z = 0;
    for (dfa::Index j = 0; j < n; ++j) {
      if (s[static_cast<size_t>(j)] == -INFINITY) {
        s[static_cast<size_t>(j)] = 0;
        continue;
      }
      s[static_cast<size_t>(j)] = std::exp(s[static_cast<size_t>(j)] - m);
      z += s[static_cast<size_t>(j)];
    }
    for (dfa::Index c = 0; c < dv; ++c) {
      double acc = 0;
      for (dfa::Index j = 0; j < n; ++j) acc += s[static_cast<size_t>(j)] * v.buf[static_cast<size_t>(j * dv + c)];
      out.buf[static_cast<size_t>(i * dv + c)] = acc / z;
    }
  }
  return out;
}

// attention.hpp:119-127 in float: S = q k^T (i-k-j matmul), *= 1/sqrt(d), softmax_rows, P v
static Tensor naive_f32(const Tensor& q, const Tensor& k, const Tensor& v) {
  const dfa::Index m = q.rows(), d = q.cols(), dv = v.cols();
  std::vector<float> s(static_cast<size_t>(m * m), 0.0f);
  for (dfa::Index i = 0; i < m; ++i)
    for (dfa::Index kk = 0; kk < d; ++kk) {
      const float a = q.buf[static_cast<size_t>(i * d + kk)];
      for (dfa::Index j = 0; j < m; ++j) s[static_cast<size_t>(i * m + j)] += a * k.buf[static_cast<size_t>(j * d + kk)];
    }
  const float sc = 1.0f / std::sqrt(static_cast<float>(d));
  for (auto& x : s) x *= sc;
  for (dfa::Index i = 0; i < m; ++i) {
    float* row = &s[static_cast<size_t>(i * m)];
    float mx = row[0];
    for (dfa::Index j = 1; j < m; ++j) mx = std::max(mx, row[j]);
    float sum = 0;
    for (dfa::Index j = 0; j < m; ++j) {
      row[j] = std::exp(row[j] - mx);
      sum += row[j];
    }
    for (dfa::Index j = 0; j < m; ++j) row[j] /= sum;
  }
  Tensor o({m, dv});
  for (dfa::Index i = 0; i < m; ++i)
    for (dfa::Index kk = 0; kk < m; ++kk) {
      const float a = s[static_cast<size_t>(i * m + kk)];
      for (dfa::Index c = 0; c < dv; ++c) o.buf[static_cast<size_t>(i * dv + c)] += a * v.buf[static_cast<size_t>(kk * dv + c)];
    }
  return o;
}

template <class T>
static double max_abs_diff(const T& a, const T& b) {
  double w = 0;
  for (size_t i = 0; i < a.buf.size(); ++i) w = std::fmax(w, std::fabs((double)a.buf[i] - (double)b.buf[i]));
  return w;
}

static void acceptance_gates() {
  {  // gate 1: masked-oracle equivalence, f64, tol 1e-10 (acceptance.cpp:57-84)
    std::mt19937_64 rng(101);
    double worst = 0;
    int configs = 0;
    for (dfa::Index n : {8, 16, 32})
      for (dfa::Index w : {2, 4, 8}) {
        if (w > n || n % w != 0) continue;
        for (dfa::Index r : {1, 2, 4}) {
          if (r > w || w % r != 0) continue;
          for (dfa::Index gamma = 0; gamma < r; ++gamma) {
            const auto cfg = attn_cfg(n, w, r, 8, gamma);
            const auto q = ref_randn<TensorD, double>(n, 8, rng);
            const auto k = ref_randn<TensorD, double>(n, 8, rng);
            const auto v = ref_randn<TensorD, double>(n, 8, rng);
            worst = std::fmax(worst, max_abs_diff(dfa::dilated_attention(q, k, v, cfg, gamma),
                                                  masked_dense(q, k, v, cfg, gamma)));
            ++configs;
          }
        }
      }
    const bool pass = worst <= 1e-10 && configs >= 27;
    std::printf("GATE 1 masked-oracle-equivalence %s: max|err| %.3g over %d configs (tol 1e-10)\n",
                pass ? "PASS" : "FAIL", worst, configs);
    CHECK(pass);
  }
  {  // gate 3: collapse w = N, r = 1 equals dense, f32, tol 1e-6 (acceptance.cpp:119-138)
    double worst = 0;
    for (std::uint64_t seed = 0; seed < 20; ++seed) {
      std::mt19937_64 rng(300 + seed);
      const dfa::Index n = 8 + static_cast<dfa::Index>(rng() % 57), d = 8;
      const auto cfg = attn_cfg(n, n, 1, d, 0);
      const auto q = ref_randn<Tensor, float>(n, d, rng);
      const auto k = ref_randn<Tensor, float>(n, d, rng);
      const auto v = ref_randn<Tensor, float>(n, d, rng);
      worst = std::fmax(worst, max_abs_diff(dfa::dilated_attention(q, k, v, cfg, 0), naive_f32(q, k, v)));
    }
    const bool pass = worst <= 1e-6;
    std::printf("GATE 3 collapse-property %s: 20 seeds, f32 max|err| %.3g (tol 1e-6)\n", pass ? "PASS" : "FAIL",
                worst);
    CHECK(pass);
  }
  {  // gate 8: worker count changes no output bit, f64 (acceptance.cpp:398-416)
    bool all = true;
    for (std::uint64_t seed = 0; seed < 10; ++seed) {
      std::mt19937_64 rng(800 + seed);
      const dfa::Index n = 64, d = 8, gamma = static_cast<dfa::Index>(seed % 2);
      const auto cfg = attn_cfg(n, 16, 2, d, gamma);
      const auto q = ref_randn<TensorD, double>(n, d, rng);
      const auto k = ref_randn<TensorD, double>(n, d, rng);
      const auto v = ref_randn<TensorD, double>(n, d, rng);
      const auto a = dfa::dilated_attention(q, k, v, cfg, gamma, 1), b = dfa::dilated_attention(q, k, v, cfg, gamma, 4);
      all = all && std::memcmp(a.buf.data(), b.buf.data(), a.buf.size() * sizeof(double)) == 0;
    }
    std::printf("GATE 8 parallel-determinism %s: 10 seeds at N=64, 1 vs 4 workers %s\n", all ? "PASS" : "FAIL",
                all ? "bitwise identical" : "DIFFER");
    CHECK(all);
  }
}

int main(int argc, char** argv) {
  host_checks();
  if (argc > 2 && std::string(argv[1]) == "gpu") gpu_checks(argv[2]);
  if (argc > 1 && std::string(argv[1]) == "gates") acceptance_gates();
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "PASS", failures);
  return failures ? 1 : 0;
}
