// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points around the UNMODIFIED reference headers
// (/root/reference/proj/include/attnkit/*.hpp), compiled by oracle/Makefile
// into oracle/_ref/libattnkit_ref.so.  Nothing here re-implements the
// algorithm: every function forwards to the reference symbol named beside it.
// Used (a) to pin the C restatement in oracle/dfa_oracle.c bit-for-bit,
// (b) to generate tests/golden/ fixtures, and (c) as the CPU baseline that
// bench.py --impl reference times on the GPU box's host cores.
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
// legs may load it; the product path (paper_2403_09195_b200) never does.

#include <atomic>
#include <cstdio>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "attnkit/attention.hpp"
#include "attnkit/autodiff.hpp"
#include "attnkit/bench.hpp"
#include "attnkit/encoder.hpp"
#include "attnkit/oracles.hpp"
#include "attnkit/tensor.hpp"
#include "attnkit/tensor_io.hpp"

using namespace attnkit;

namespace {

thread_local std::string g_err;

// Status codes shared with include/dfa.h (DFA_OK .. DFA_ERR_CONTRACT).
enum : int { OK = 0, ERR_CONFIG = 1, ERR_DIMENSION = 2, ERR_OUT_OF_RANGE = 3, ERR_CONTRACT = 4, ERR_IO = 7,
             ERR_OTHER = 9 };

template <class F>
int guarded(F&& f) {
  try {
    f();
    return OK;
  } catch (const config_error& e) {
    g_err = e.what();
    return ERR_CONFIG;
  } catch (const dimension_error& e) {
    g_err = e.what();
    return ERR_DIMENSION;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return ERR_OUT_OF_RANGE;
  } catch (const contract_error& e) {
    g_err = e.what();
    return ERR_CONTRACT;
  } catch (const io_error& e) {
    g_err = e.what();
    return ERR_IO;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ERR_OTHER;
  }
}

AttentionConfig make_cfg(int64_t n, int64_t w, int64_t r, int64_t h, int64_t d, const int64_t* offsets,
                         int32_t kernel, int64_t tile, int32_t scale_scores) {
  AttentionConfig cfg;
  cfg.seq_len = n;
  cfg.segment_len = w;
  cfg.interval = r;
  cfg.num_heads = static_cast<int>(h);
  cfg.head_dim = d;
  if (offsets && h > 0) cfg.head_offsets.assign(offsets, offsets + h);
  cfg.kernel = kernel ? Kernel::tiled : Kernel::naive;
  cfg.tile_size = tile;
  cfg.scale_scores = scale_scores != 0;
  return cfg;
}

template <class S>
Tensor<S> wrap(const S* p, int64_t rows, int64_t cols) {
  return Tensor<S>({rows, cols}, std::vector<S>(p, p + rows * cols));
}

template <class S>
int dilated(const S* q, const S* k, const S* v, int64_t n, int64_t d, int64_t dv, int64_t w, int64_t r,
            int64_t gamma, int32_t scale_scores, int32_t kernel, int64_t tile, int32_t workers, S* out) {
  return guarded([&] {
    const int64_t off = gamma;
    auto cfg = make_cfg(n, w, r, 1, d, &off, kernel, tile, scale_scores);
    auto o = dilated_attention(wrap(q, n, d), wrap(k, n, d), wrap(v, n, dv), cfg, gamma, workers);
    std::memcpy(out, o.data(), sizeof(S) * static_cast<size_t>(o.numel()));
  });
}

// attention.hpp:340-360 multi_head_dilated: x [N x D], wq/wk/wv [h x D x d],
// wo [D x D] -> out [N x D]; offsets spread_offsets(h, r).
template <class S>
int multi_head(const S* x, const S* wq, const S* wk, const S* wv, const S* wo, int64_t n, int64_t dm, int64_t h,
               int64_t w, int64_t r, const int64_t* offsets, S* out) {
  return guarded([&] {
    AttentionConfig cfg = make_cfg(n, w, r, h, dm / h, offsets, 0, 1, 1);
    MultiHeadWeights<S> mw;
    const int64_t d = dm / h;
    for (int64_t j = 0; j < h; ++j) {
      mw.wq.push_back(wrap(wq + j * dm * d, dm, d));
      mw.wk.push_back(wrap(wk + j * dm * d, dm, d));
      mw.wv.push_back(wrap(wv + j * dm * d, dm, d));
    }
    mw.wo = wrap(wo, dm, dm);
    auto o = multi_head_dilated(wrap(x, n, dm), mw, cfg, 1);
    std::memcpy(out, o.data(), sizeof(S) * static_cast<size_t>(o.numel()));
  });
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// attention.hpp:280-301 dilated_attention<float>
int ref_dilated_attention_f32(const float* q, const float* k, const float* v, int64_t n, int64_t d, int64_t dv,
                              int64_t w, int64_t r, int64_t gamma, int32_t scale_scores, int32_t kernel,
                              int64_t tile, int32_t workers, float* out) {
  return dilated(q, k, v, n, d, dv, w, r, gamma, scale_scores, kernel, tile, workers, out);
}

// attention.hpp:280-301 dilated_attention<double>
int ref_dilated_attention_f64(const double* q, const double* k, const double* v, int64_t n, int64_t d, int64_t dv,
                              int64_t w, int64_t r, int64_t gamma, int32_t scale_scores, int32_t kernel,
                              int64_t tile, int32_t workers, double* out) {
  return dilated(q, k, v, n, d, dv, w, r, gamma, scale_scores, kernel, tile, workers, out);
}

// oracles.hpp:67-107 masked_dense_dilated<double>
int ref_masked_dense_dilated_f64(const double* q, const double* k, const double* v, int64_t n, int64_t d,
                                 int64_t dv, int64_t w, int64_t r, int64_t gamma, int32_t scale_scores,
                                 double* out) {
  return guarded([&] {
    const int64_t off = gamma;
    auto cfg = make_cfg(n, w, r, 1, d, &off, 0, 1, scale_scores);
    auto o = oracle::masked_dense_dilated(wrap(q, n, d), wrap(k, n, d), wrap(v, n, dv), cfg, gamma);
    std::memcpy(out, o.data(), sizeof(double) * static_cast<size_t>(o.numel()));
  });
}

// attention.hpp:119-127 naive_attention (dense, whole input)
int ref_naive_attention_f64(const double* q, const double* k, const double* v, int64_t nq, int64_t nk, int64_t d,
                            int64_t dv, int32_t scale_scores, double* out) {
  return guarded([&] {
    auto o = naive_attention(wrap(q, nq, d), wrap(k, nk, d), wrap(v, nk, dv), scale_scores != 0);
    std::memcpy(out, o.data(), sizeof(double) * static_cast<size_t>(o.numel()));
  });
}
int ref_naive_attention_f32(const float* q, const float* k, const float* v, int64_t nq, int64_t nk, int64_t d,
                            int64_t dv, int32_t scale_scores, float* out) {
  return guarded([&] {
    auto o = naive_attention(wrap(q, nq, d), wrap(k, nk, d), wrap(v, nk, dv), scale_scores != 0);
    std::memcpy(out, o.data(), sizeof(float) * static_cast<size_t>(o.numel()));
  });
}

// attention.hpp:84-98 make_segment_view; writes up to cap indices.
int ref_segment_view(int64_t n, int64_t w, int64_t r, int64_t i, int64_t gamma, int64_t* rows, int64_t cap,
                     int64_t* count) {
  return guarded([&] {
    auto view = make_segment_view(n, w, r, i, gamma);
    *count = static_cast<int64_t>(view.row_indices.size());
    for (int64_t t = 0; t < *count && t < cap; ++t) rows[t] = view.row_indices[static_cast<size_t>(t)];
  });
}

// attention.hpp:44-65 AttentionConfig::validate
int ref_validate(int64_t n, int64_t w, int64_t r, int64_t h, int64_t d, const int64_t* offsets, int64_t n_offsets,
                 int32_t kernel, int64_t tile, int32_t full_coverage) {
  return guarded([&] {
    auto cfg = make_cfg(n, w, r, h, d, nullptr, kernel, tile, 1);
    if (offsets && n_offsets > 0) cfg.head_offsets.assign(offsets, offsets + n_offsets);
    cfg.validate(full_coverage != 0);
  });
}

// attention.hpp:370-387 flop_count and :389-394 flop_csv_row
int ref_flop_count(int64_t n, int64_t w, int64_t r, int64_t h, int64_t d, const int64_t* offsets,
                   uint64_t* dense_mults, uint64_t* dilated_mults, double* ratio, char* csv, int64_t csv_cap) {
  return guarded([&] {
    auto cfg = make_cfg(n, w, r, h, d, offsets, 0, 1, 1);
    auto fc = flop_count(cfg);
    *dense_mults = fc.dense_mults;
    *dilated_mults = fc.dilated_mults;
    *ratio = fc.ratio;
    if (csv && csv_cap > 0) {
      std::string row = flop_csv_row(cfg, fc);
      std::strncpy(csv, row.c_str(), static_cast<size_t>(csv_cap - 1));
      csv[csv_cap - 1] = 0;
    }
  });
}

// tensor.hpp:369-376 randn over common.hpp:47 Rng (mt19937_64); draws n values.
void ref_randn_f64(uint64_t seed, int64_t n, double* out) {
  Rng rng(seed);
  auto t = randn<double>({n}, rng);
  std::memcpy(out, t.data(), sizeof(double) * static_cast<size_t>(n));
}
void ref_randn_f32(uint64_t seed, int64_t n, float* out) {
  Rng rng(seed);
  auto t = randn<float>({n}, rng);
  std::memcpy(out, t.data(), sizeof(float) * static_cast<size_t>(n));
}

// CPU baseline timing: `units` independent (image, head) forwards of
// dilated_attention<float>(N, w, r, d, gamma = unit % r), spread over
// `threads` std::threads with workers=1 each -- the reference's own
// per-call path (bench.hpp:125-133) driven unit-parallel across host cores.
// Inputs are `distinct` randn-drawn unit tensors cycled over; returns the
// wall-clock seconds for all units (inputs prepared before timing).
double ref_time_dilated_f32(int64_t n, int64_t w, int64_t r, int64_t d, int64_t units, int32_t threads,
                            int32_t distinct, uint64_t seed) {
  if (distinct < 1) distinct = 1;
  Rng rng(seed ^ 0x9e3779b97f4a7c15ull);
  std::vector<Tensor<float>> q, k, v;
  for (int j = 0; j < distinct; ++j) {
    q.push_back(randn<float>({n, d}, rng));
    k.push_back(randn<float>({n, d}, rng));
    v.push_back(randn<float>({n, d}, rng));
  }
  AttentionConfig cfg;
  cfg.seq_len = n;
  cfg.segment_len = w;
  cfg.interval = r;
  cfg.num_heads = 1;
  cfg.head_dim = d;
  cfg.head_offsets = {0};
  std::atomic<int64_t> next{0};
  std::atomic<double> sink{0};
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, threads); ++t) {
    pool.emplace_back([&] {
      double local = 0;
      for (;;) {
        const int64_t u = next.fetch_add(1);
        if (u >= units) break;
        const auto s = static_cast<size_t>(u % distinct);
        auto o = dilated_attention(q[s], k[s], v[s], cfg, u % r, 1);
        local += o[(u % r) * d];
      }
      double cur = sink.load();
      while (!sink.compare_exchange_weak(cur, cur + local)) {
      }
    });
  }
  for (auto& th : pool) th.join();
  auto t1 = std::chrono::steady_clock::now();
  volatile double keep = sink.load();
  (void)keep;
  return std::chrono::duration<double>(t1 - t0).count();
}

// ---------------------------------------------------------------- §8(f) rows

// tensor_io.hpp:86-91 save_tensor / :147-153 load_tensor (DTNSR1).
int ref_save_tensor(const char* path, int32_t dtype, int32_t rank, const int64_t* dims, const void* data) {
  return guarded([&] {
    Shape shape(dims, dims + rank);
    int64_t n = 1;
    for (int i = 0; i < rank; ++i) n *= dims[i];
    if (dtype == 0) {
      const float* f = static_cast<const float*>(data);
      save_tensor(path, Tensor<float>(shape, std::vector<float>(f, f + n)));
    } else {
      const double* f = static_cast<const double*>(data);
      save_tensor(path, Tensor<double>(shape, std::vector<double>(f, f + n)));
    }
  });
}
int ref_load_tensor_f64(const char* path, double* out, int64_t cap, int32_t* rank, int64_t* dims) {
  return guarded([&] {
    auto t = load_tensor<double>(path);
    if (t.numel() > cap) throw dimension_error("ref_load_tensor_f64: buffer too small");
    *rank = static_cast<int32_t>(t.rank());
    for (Index i = 0; i < t.rank(); ++i) dims[i] = t.dim(i);
    std::memcpy(out, t.data(), sizeof(double) * static_cast<size_t>(t.numel()));
  });
}

int ref_multi_head_dilated_f64(const double* x, const double* wq, const double* wk, const double* wv,
                               const double* wo, int64_t n, int64_t dm, int64_t h, int64_t w, int64_t r,
                               const int64_t* offsets, double* out) {
  return multi_head(x, wq, wk, wv, wo, n, dm, h, w, r, offsets, out);
}
int ref_multi_head_dilated_f32(const float* x, const float* wq, const float* wk, const float* wv, const float* wo,
                               int64_t n, int64_t dm, int64_t h, int64_t w, int64_t r, const int64_t* offsets,
                               float* out) {
  return multi_head(x, wq, wk, wv, wo, n, dm, h, w, r, offsets, out);
}

// Backward of one dilated head on the reference's tape: the dilated branch
// of detail::attention_mix (encoder.hpp:204-219) on leaves q, k, v, with
// loss = sum(head o dO) so the head's incoming gradient is dO; ag::backward
// (autodiff.hpp:66-95) fills q/k/v grads.
int ref_dilated_backward_f64(const double* q, const double* k, const double* v, const double* dout, int64_t n,
                             int64_t d, int64_t dv, int64_t w, int64_t r, int64_t gamma, double* dq, double* dk,
                             double* dvo) {
  return guarded([&] {
    const int64_t off = gamma;
    AttentionConfig acfg = make_cfg(n, w, r, 1, d, &off, 0, 1, 1);
    acfg.validate();
    auto qv = ag::leaf(wrap(q, n, d)), kv = ag::leaf(wrap(k, n, d)), vv = ag::leaf(wrap(v, n, dv));
    const double sc = 1.0 / std::sqrt(static_cast<double>(d));
    ag::Var<double> head;
    bool first = true;
    for (Index s = 0; s < acfg.num_segments(); ++s) {
      const auto view = make_segment_view(acfg.seq_len, acfg.segment_len, acfg.interval, s, gamma);
      const auto m = static_cast<Index>(view.row_indices.size());
      if (m == 0) continue;
      auto qs = ag::slice_rows_strided(qv, view.row_indices.front(), acfg.interval, m);
      auto ks = ag::slice_rows_strided(kv, view.row_indices.front(), acfg.interval, m);
      auto vs = ag::slice_rows_strided(vv, view.row_indices.front(), acfg.interval, m);
      auto scores = ag::scale(ag::matmul(qs, ag::transpose(ks)), sc);
      auto placed = ag::scatter_rows(ag::matmul(ag::softmax_rows(scores), vs), view.row_indices, acfg.seq_len);
      head = first ? placed : ag::add(head, placed);
      first = false;
    }
    auto loss = ag::sum(ag::hadamard(head, ag::leaf(wrap(dout, n, dv))));
    ag::backward(loss);
    std::memcpy(dq, qv.grad().data(), sizeof(double) * static_cast<size_t>(n * d));
    std::memcpy(dk, kv.grad().data(), sizeof(double) * static_cast<size_t>(n * d));
    std::memcpy(dvo, vv.grad().data(), sizeof(double) * static_cast<size_t>(n * dv));
  });
}

// One pre-norm encoder block (encoder.hpp:241-248, the loop body of
// encoder_forward) on the reference's own ops: LN1 -> attention_mix (dilated,
// per-head wq/wk/wv, wo, bo) -> residual -> LN2 -> w1/b1 -> GELU(erf) -> w2/b2
// -> residual.  x [N x D]; wq/wk/wv [h x D x d]; mlp hidden = w1 cols.
int ref_encoder_block_f64(const double* x, int64_t n, int64_t dm, int64_t h, int64_t hidden, int64_t w, int64_t r,
                          const double* ln1_g, const double* ln1_b, const double* wq, const double* wk,
                          const double* wv, const double* wo, const double* bo, const double* ln2_g,
                          const double* ln2_b, const double* w1, const double* b1, const double* w2,
                          const double* b2, double* out) {
  return guarded([&] {
    EncoderConfig cfg;
    cfg.embed_dim = dm;
    cfg.num_heads = static_cast<int>(h);
    cfg.num_layers = 1;
    cfg.attention_mode = AttentionMode::dilated;
    cfg.segment_len = w;
    cfg.interval = r;
    // token count comes from the image geometry: a 1-channel image of
    // sqrt(N) x sqrt(N) patches of size 1
    const auto g = static_cast<Index>(std::llround(std::sqrt(static_cast<double>(n))));
    if (g * g != n) throw config_error("ref_encoder_block_f64: N must be a square");
    cfg.image_size = g;
    cfg.patch_size = 1;
    cfg.mlp_ratio = static_cast<double>(hidden) / static_cast<double>(dm);
    if (cfg.mlp_hidden() != hidden) throw config_error("ref_encoder_block_f64: hidden/D not representable");
    const int64_t d = dm / h;
    ParamSet<double> p;
    const std::string b = detail::block_prefix(0);
    auto vec = [](const double* src, int64_t len) { return Tensor<double>({len}, std::vector<double>(src, src + len)); };
    p.add(b + "ln1.g", vec(ln1_g, dm));
    p.add(b + "ln1.b", vec(ln1_b, dm));
    for (int64_t j = 0; j < h; ++j) {
      p.add(msg(b, "attn.wq", j), wrap(wq + j * dm * d, dm, d));
      p.add(msg(b, "attn.wk", j), wrap(wk + j * dm * d, dm, d));
      p.add(msg(b, "attn.wv", j), wrap(wv + j * dm * d, dm, d));
    }
    p.add(b + "attn.wo", wrap(wo, dm, dm));
    p.add(b + "attn.bo", vec(bo, dm));
    p.add(b + "ln2.g", vec(ln2_g, dm));
    p.add(b + "ln2.b", vec(ln2_b, dm));
    p.add(b + "mlp.w1", wrap(w1, dm, hidden));
    p.add(b + "mlp.b1", vec(b1, hidden));
    p.add(b + "mlp.w2", wrap(w2, hidden, dm));
    p.add(b + "mlp.b2", vec(b2, dm));
    cfg.validate();
    auto xv = ag::leaf(wrap(x, n, dm));
    auto normed = ag::layer_norm(xv, p.at(b + "ln1.g"), p.at(b + "ln1.b"));
    auto x1 = ag::add(xv, detail::attention_mix(normed, p, b, cfg));
    auto normed2 = ag::layer_norm(x1, p.at(b + "ln2.g"), p.at(b + "ln2.b"));
    auto hid = ag::gelu(ag::add_rowvec(ag::matmul(normed2, p.at(b + "mlp.w1")), p.at(b + "mlp.b1")));
    auto mixed = ag::add_rowvec(ag::matmul(hid, p.at(b + "mlp.w2")), p.at(b + "mlp.b2"));
    auto y = ag::add(x1, mixed);
    std::memcpy(out, y.value().data(), sizeof(double) * static_cast<size_t>(n * dm));
  });
}

// bench.hpp:173-176 bench_csv_header and :235-276 spearman_rank_correlation.
int ref_bench_csv_header(char* buf, int64_t cap) {
  return guarded([&] {
    const std::string h = bench_csv_header();
    std::snprintf(buf, static_cast<size_t>(cap), "%s", h.c_str());
  });
}
int ref_spearman(const double* a, const double* b, int64_t n, double* out) {
  return guarded([&] {
    *out = spearman_rank_correlation(std::vector<double>(a, a + n), std::vector<double>(b, b + n));
  });
}

}  // extern "C"
