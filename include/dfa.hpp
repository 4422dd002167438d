// include/dfa.hpp -- reference-shaped C++ API over the C-ABI (include/dfa.h).
//
// Mirrors attnkit's hot-path API (/root/reference/proj/include/attnkit/
// attention.hpp) so a caller of the reference switches by changing the
// namespace:
//
//   attnkit::AttentionConfig          -> dfa::AttentionConfig      (:24-66)
//   attnkit::make_segment_view        -> dfa::make_segment_view    (:84-98)
//   attnkit::dilated_attention(q,k,v,cfg,gamma,workers)
//                                     -> dfa::dilated_attention    (:280-301)
//   attnkit::multi_head_dilated(x,w,cfg,workers)
//                                     -> dfa::multi_head_dilated   (:340-360)
//   attnkit::flop_count / flop_csv_*  -> dfa::flop_count / ...     (:364-394)
//   attnkit::fault::recompose_perturb -> dfa::fault::ScopedPerturb (:237-241)
//
// and throws the same exception taxonomy (common.hpp:13-30):
// config_error, dimension_error, contract_error and std::out_of_range.
// Tensors are any row-major rank-2 type with rows(), cols(), data() and a
// constructor from a {rows, cols} shape -- attnkit::Tensor<float> qualifies.
// Computation runs on the GPU (fp32 validation kernel for float host tensors;
// dfa::forward for bf16 device batches).  Header-only; link libdfa.so.
#pragma once

#include <cstdint>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "dfa.h"

namespace dfa {

using Index = std::ptrdiff_t;

struct dimension_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct contract_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct config_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct unsupported_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(dfa_status_t st) {
  if (st == DFA_OK) return;
  const std::string m = dfa_last_error();
  switch (st) {
    case DFA_ERR_CONFIG:
      throw config_error(m);
    case DFA_ERR_DIMENSION:
      throw dimension_error(m);
    case DFA_ERR_OUT_OF_RANGE:
      throw std::out_of_range(m);
    case DFA_ERR_CONTRACT:
      throw contract_error(m);
    case DFA_ERR_CUDA:
      throw cuda_error(m);
    default:
      throw unsupported_error(m);
  }
}

enum class Kernel { naive, tiled };

struct AttentionConfig {
  Index seq_len = 0;
  Index segment_len = 0;
  Index interval = 1;
  int num_heads = 1;
  Index head_dim = 0;
  std::vector<Index> head_offsets;
  Kernel kernel = Kernel::naive;
  Index tile_size = 1;
  bool scale_scores = true;

  Index num_segments() const { return (seq_len + segment_len - 1) / segment_len; }
  Index model_dim() const { return static_cast<Index>(num_heads) * head_dim; }

  static std::vector<Index> spread_offsets(int heads, Index interval) {
    std::vector<Index> out(static_cast<std::size_t>(heads));
    for (int j = 0; j < heads; ++j) out[static_cast<std::size_t>(j)] = static_cast<Index>(j) % interval;
    return out;
  }

  // Plain-C view; `offsets` must outlive the returned struct.
  dfa_config_t to_c(std::vector<int64_t>& offsets, Index value_dim = 0) const {
    offsets.assign(head_offsets.begin(), head_offsets.end());
    dfa_config_t c{};
    c.seq_len = seq_len;
    c.segment_len = segment_len;
    c.interval = interval;
    c.num_heads = num_heads;
    c.head_dim = head_dim;
    c.value_dim = value_dim;
    c.head_offsets = offsets.empty() ? nullptr : offsets.data();
    c.kernel = kernel == Kernel::tiled ? DFA_KERNEL_TILED : DFA_KERNEL_NAIVE;
    c.tile_size = tile_size;
    c.scale_scores = scale_scores ? 1 : 0;
    return c;
  }

  void validate(bool require_full_coverage = false) const {
    if (head_offsets.size() != static_cast<std::size_t>(num_heads)) {
      std::ostringstream os;
      os << "attention: " << head_offsets.size() << " offsets for " << num_heads << " heads";
      throw config_error(os.str());
    }
    std::vector<int64_t> offs;
    const dfa_config_t c = to_c(offs);
    check(dfa_validate(&c, require_full_coverage ? 1 : 0));
  }

  // Adopt an attnkit::AttentionConfig (or any type with the same fields).
  template <class C>
  static AttentionConfig from(const C& o) {
    AttentionConfig c;
    c.seq_len = o.seq_len;
    c.segment_len = o.segment_len;
    c.interval = o.interval;
    c.num_heads = o.num_heads;
    c.head_dim = o.head_dim;
    c.head_offsets.assign(o.head_offsets.begin(), o.head_offsets.end());
    c.kernel = static_cast<int>(o.kernel) == 1 ? Kernel::tiled : Kernel::naive;
    c.tile_size = o.tile_size;
    c.scale_scores = o.scale_scores;
    return c;
  }
};

struct SegmentView {
  Index segment_index = 0;
  Index offset = 0;
  std::vector<Index> row_indices;
  bool operator==(const SegmentView&) const = default;
};

inline SegmentView make_segment_view(Index seq_len, Index segment_len, Index interval, Index segment_index,
                                     Index offset) {
  int64_t count = 0;
  check(dfa_segment_view(seq_len, segment_len, interval, segment_index, offset, nullptr, 0, &count));
  std::vector<int64_t> rows(static_cast<std::size_t>(count));
  check(dfa_segment_view(seq_len, segment_len, interval, segment_index, offset, rows.data(), count, &count));
  SegmentView v;
  v.segment_index = segment_index;
  v.offset = offset;
  v.row_indices.assign(rows.begin(), rows.end());
  return v;
}

struct FlopCount {
  std::uint64_t dense_mults = 0;
  std::uint64_t dilated_mults = 0;
  double ratio = 0.0;
};

inline FlopCount flop_count(const AttentionConfig& cfg) {
  cfg.validate();
  std::vector<int64_t> offs;
  const dfa_config_t c = cfg.to_c(offs);
  FlopCount fc;
  uint64_t dn = 0, dl = 0;
  check(dfa_flop_count(&c, &dn, &dl, &fc.ratio));
  fc.dense_mults = dn;
  fc.dilated_mults = dl;
  return fc;
}

inline std::string flop_csv_header() { return "N,w,r,h,d,dense_mults,dilated_mults,ratio"; }

inline std::string flop_csv_row(const AttentionConfig& cfg, const FlopCount& fc) {
  std::ostringstream os;
  os << cfg.seq_len << "," << cfg.segment_len << "," << cfg.interval << "," << cfg.num_heads << "," << cfg.head_dim
     << "," << fc.dense_mults << "," << fc.dilated_mults << "," << fc.ratio;
  return os.str();
}

// Device staging buffer for the host-tensor calls; grows on demand.
class Workspace {
 public:
  Workspace() = default;
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  ~Workspace() { dfa_workspace_destroy(ws_); }
  dfa_workspace_t* get(std::size_t bytes) {
    if (bytes > bytes_) {
      dfa_workspace_destroy(ws_);
      ws_ = nullptr;
      check(dfa_workspace_create(bytes, &ws_));
      bytes_ = bytes;
    }
    return ws_;
  }

 private:
  dfa_workspace_t* ws_ = nullptr;
  std::size_t bytes_ = 0;
};

inline Workspace& thread_workspace() {
  thread_local Workspace ws;
  return ws;
}

namespace detail {
template <class T>
void require_rank2(const T& t, const char* op) {
  if constexpr (requires { t.rank(); }) {
    if (t.rank() != 2) throw dimension_error(std::string(op) + ": expected rank-2 tensor");
  }
}
}  // namespace detail

// attention.hpp:280-301 on host tensors (GPU fp32 / f64 validation kernels).
// Same preconditions and error types as the reference: validate(); q/k widths
// and k/v rows agree (require_qkv :102-110); q and k have cfg.seq_len rows
// (:285-286); head_offset in [0, r) else std::out_of_range (:287-288).
// `workers` is accepted and ignored: the GPU grid replaces parallel_for.
template <class Tensor>
Tensor dilated_attention(const Tensor& q, const Tensor& k, const Tensor& v, const AttentionConfig& cfg,
                         Index head_offset, int workers = 1) {
  using Scalar = std::remove_cv_t<std::remove_pointer_t<decltype(q.data())>>;
  static_assert(std::is_same_v<Scalar, float> || std::is_same_v<Scalar, double>,
                "dfa::dilated_attention takes float or double tensors");
  (void)workers;
  cfg.validate();
  detail::require_rank2(q, "dilated_attention");
  detail::require_rank2(k, "dilated_attention");
  detail::require_rank2(v, "dilated_attention");
  if (q.cols() != k.cols()) throw dimension_error("dilated_attention: query/key width mismatch");
  if (k.rows() != v.rows()) throw dimension_error("dilated_attention: key/value row mismatch");
  if (q.rows() != cfg.seq_len || k.rows() != cfg.seq_len) {
    std::ostringstream os;
    os << "dilated_attention: expected " << cfg.seq_len << " rows, got " << q.rows();
    throw dimension_error(os.str());
  }
  if (head_offset < 0 || head_offset >= cfg.interval) {
    std::ostringstream os;
    os << "dilated_attention: head offset " << head_offset << " outside [0, " << cfg.interval << ")";
    throw std::out_of_range(os.str());
  }
  AttentionConfig one = cfg;
  one.num_heads = 1;
  one.head_offsets = {head_offset};
  one.head_dim = q.cols();
  std::vector<int64_t> offs;
  dfa_config_t c = one.to_c(offs, v.cols());
  // float tensors run the fp32 validation kernel, double tensors the f64
  // kernel (double arithmetic end to end, the reference's f64 mode)
  constexpr dfa_dtype_t dt = std::is_same_v<Scalar, double> ? DFA_F64 : DFA_F32;
  std::size_t bytes = 0;
  check(dfa_workspace_bytes(&c, dt, 1, 0, &bytes));
  Tensor out({q.rows(), v.cols()});
  check(dfa_forward_host(&c, dt, 1, q.data(), k.data(), v.data(), out.data(), nullptr, thread_workspace().get(bytes),
                         nullptr));
  return out;
}

// attention.hpp:340-360 multi_head_dilated(x, weights, cfg, workers) on host
// tensors: `Weights` has the reference's MultiHeadWeights members -- wq, wk,
// wv (h tensors of D x d) and wo (D x D) -- so attnkit::MultiHeadWeights<float>
// qualifies.  Same checks and error types: validate(true) (full coverage),
// weight shapes (MultiHeadWeights::validate), x = [N x D].  fp32 device path.
template <class Tensor, class Weights>
Tensor multi_head_dilated(const Tensor& x, const Weights& weights, const AttentionConfig& cfg, int workers = 1) {
  using Scalar = std::remove_cv_t<std::remove_pointer_t<decltype(x.data())>>;
  static_assert(std::is_same_v<Scalar, float>, "dfa::multi_head_dilated runs the fp32 device path");
  (void)workers;
  cfg.validate(/*require_full_coverage=*/true);
  const auto heads = static_cast<std::size_t>(cfg.num_heads);
  if (weights.wq.size() != heads || weights.wk.size() != heads || weights.wv.size() != heads) {
    std::ostringstream os;
    os << "multi_head_dilated: expected " << cfg.num_heads << " per-head projections";
    throw config_error(os.str());
  }
  const Index D = cfg.head_dim * cfg.num_heads, d = cfg.head_dim;
  for (std::size_t j = 0; j < heads; ++j)
    for (const auto* t : {&weights.wq[j], &weights.wk[j], &weights.wv[j]})
      if (t->rows() != D || t->cols() != d) {
        std::ostringstream os;
        os << "multi_head_dilated: head " << j << " projection is [" << t->rows() << "x" << t->cols()
           << "], expected [" << D << "x" << d << "]";
        throw dimension_error(os.str());
      }
  if (weights.wo.rows() != D || weights.wo.cols() != D) throw dimension_error("multi_head_dilated: bad output projection");
  detail::require_rank2(x, "multi_head_dilated");
  if (x.rows() != cfg.seq_len || x.cols() != D) {
    std::ostringstream os;
    os << "multi_head_dilated: input [" << x.rows() << "x" << x.cols() << "], expected [" << cfg.seq_len << "x" << D
       << "]";
    throw dimension_error(os.str());
  }
  // stack the per-head projections as [h, D, d] (the C-ABI layout)
  std::vector<float> wq(heads * D * d), wk(heads * D * d), wv(heads * D * d);
  for (std::size_t j = 0; j < heads; ++j)
    for (Index e = 0; e < D * d; ++e) {
      wq[j * D * d + e] = weights.wq[j].data()[e];
      wk[j * D * d + e] = weights.wk[j].data()[e];
      wv[j * D * d + e] = weights.wv[j].data()[e];
    }
  std::vector<int64_t> offs;
  dfa_config_t c = cfg.to_c(offs, 0);
  std::size_t bytes = 0;
  check(dfa_multi_head_host_workspace_bytes(&c, DFA_F32, 1, &bytes));
  Tensor out({cfg.seq_len, D});
  check(dfa_multi_head_dilated_host(&c, DFA_F32, 1, x.data(), wq.data(), wk.data(), wv.data(), weights.wo.data(),
                                    out.data(), thread_workspace().get(bytes)));
  return out;
}

// Batched multi-head device forward: q, k [B, N, h, d], v, o [B, N, h, d_v]
// device pointers; head j at cfg.head_offsets[j]; optional fp32 lse [B, h, N].
inline void forward(const AttentionConfig& cfg, dfa_dtype_t dtype, int64_t batch, const void* q, const void* k,
                    const void* v, void* o, float* lse = nullptr, void* stream = nullptr, Index value_dim = 0) {
  if (cfg.head_offsets.size() != static_cast<std::size_t>(cfg.num_heads)) cfg.validate();
  std::vector<int64_t> offs;
  const dfa_config_t c = cfg.to_c(offs, value_dim);
  check(dfa_forward(&c, dtype, batch, q, k, v, o, lse, stream));
}

namespace fault {
// attention.hpp:237-241: perturbs every forward's output while alive.
struct ScopedPerturb {
  ScopedPerturb() { dfa_set_fault_perturb(1); }
  ~ScopedPerturb() { dfa_set_fault_perturb(0); }
};
}  // namespace fault

}  // namespace dfa
