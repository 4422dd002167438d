// C-ABI layer (include/dfa.h): validation with the reference's rules and
// messages, geometry resolution, device-path dispatch, host-buffer entry
// points and the fault hook.  No CPU compute path exists: every forward is a
// device kernel (tcgen05 for bf16/d=64 geometries, SIMT otherwise).
#include <algorithm>
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <string>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif

#include "../../include/dfa.h"
#include "dfa_internal.h"

namespace {

thread_local std::string g_last_error;
thread_local int32_t g_launches = 0;
std::atomic<int32_t> g_fault{0};
std::atomic<int32_t> g_path_override{0};
std::atomic<int32_t> g_mb_mode{0};
std::atomic<int32_t> g_host_zero_copy{1};
// 1: a host-resident o is written in place too -- the kernel TMA-stores the
// kept rows over PCIe and host threads zero-fill the rest meanwhile
std::atomic<int32_t> g_host_kept_out{1};

dfa_status_t fail(dfa_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

// attention.hpp:44-65, same order of checks and the same message text.
dfa_status_t validate(const dfa_config_t* c, int32_t full) {
  if (!c) return fail(DFA_ERR_CONFIG, "attention: null config");
  const long long n = c->seq_len, w = c->segment_len, r = c->interval, h = c->num_heads, d = c->head_dim;
  if (n < 1) return fail(DFA_ERR_CONFIG, "attention: seq_len must be positive");
  if (w < 1 || w > n) return fail(DFA_ERR_CONFIG, "attention: need 1 <= w <= N, got w=%lld N=%lld", w, n);
  if (r < 1 || r > w) return fail(DFA_ERR_CONFIG, "attention: need 1 <= r <= w, got r=%lld w=%lld", r, w);
  if (h < 1) return fail(DFA_ERR_CONFIG, "attention: num_heads must be positive");
  if (d < 1) return fail(DFA_ERR_CONFIG, "attention: head_dim must be positive");
  if (!c->head_offsets) return fail(DFA_ERR_CONFIG, "attention: 0 offsets for %lld heads", h);
  for (long long j = 0; j < h; ++j) {
    const long long g = c->head_offsets[j];
    if (g < 0 || g >= r) return fail(DFA_ERR_CONFIG, "attention: offset %lld outside [0, %lld)", g, r);
  }
  if (c->kernel == DFA_KERNEL_TILED && c->tile_size < 1)
    return fail(DFA_ERR_CONFIG, "attention: tile_size must be >= 1");
  if (c->kernel != DFA_KERNEL_NAIVE && c->kernel != DFA_KERNEL_TILED)
    return fail(DFA_ERR_CONFIG, "attention: unknown kernel %d", (int)c->kernel);
  if (c->value_dim < 0) return fail(DFA_ERR_CONFIG, "attention: value_dim must be non-negative");
  if (full) {
    for (long long cls = 0; cls < r; ++cls) {
      bool hit = false;
      for (long long j = 0; j < h && !hit; ++j) hit = (c->head_offsets[j] % r) == cls;
      if (!hit)
        return fail(DFA_ERR_CONFIG,
                    "attention: offset class %lld of interval %lld is covered by no head; full coverage needs h >= r",
                    cls, r);
    }
  }
  return DFA_OK;
}

dfa_status_t resolve(const dfa_config_t* c, int64_t batch, dfa_impl::Geometry* g) {
  dfa_status_t st = validate(c, 0);
  if (st != DFA_OK) return st;
  if (batch < 0) return fail(DFA_ERR_DIMENSION, "dfa_forward: negative batch %lld", (long long)batch);
  if (c->num_heads > dfa_impl::kMaxHeads)
    return fail(DFA_ERR_UNSUPPORTED, "dfa_forward: %lld heads exceeds the device limit %d",
                (long long)c->num_heads, dfa_impl::kMaxHeads);
  g->B = batch;
  g->N = c->seq_len;
  g->w = c->segment_len;
  g->r = c->interval;
  g->h = c->num_heads;
  g->d = c->head_dim;
  g->dv = c->value_dim > 0 ? c->value_dim : c->head_dim;
  if (g->d > 256 || g->dv > 256)
    return fail(DFA_ERR_UNSUPPORTED, "dfa_forward: head_dim %lld / value_dim %lld exceed the device limit 256",
                (long long)g->d, (long long)g->dv);
  g->ldq = g->ldk = g->h * g->d;
  g->ldv = g->ldo = g->h * g->dv;
  g->n_seg = (g->N + g->w - 1) / g->w;
  g->m_max = (g->w + g->r - 1) / g->r;
  // attention.hpp:112-115: Scalar(1)/sqrt(Scalar(d)) in the working precision.
  g->scale = c->scale_scores ? 1.0f / sqrtf((float)g->d) : 1.0f;
  for (int j = 0; j < dfa_impl::kMaxHeads; ++j) g->offsets[j] = j < g->h ? (int32_t)c->head_offsets[j] : 0;
  return DFA_OK;
}

int pick_path(const dfa_impl::Geometry& g, dfa_dtype_t dtype, const void* q, const void* k, const void* v,
              const void* o) {
  const int ov = g_path_override.load();
  if (ov == DFA_PATH_SIMT) return DFA_PATH_SIMT;
  if (dfa_impl::sm100_supported(g, dtype, q, k, v, o)) return DFA_PATH_SM100_TCGEN05;
  if (ov == DFA_PATH_SM100_TCGEN05) return DFA_PATH_NONE;  // forced but not applicable
  return DFA_PATH_SIMT;
}

size_t elem_size(dfa_dtype_t t) { return t == DFA_F64 ? 8 : t == DFA_F32 ? 4 : 2; }

// Device address of pinned, mapped host memory (nullptr for pageable or device memory).
// Zero the rows of a host-resident [B][N][h][dv] o that no segment view keeps
// (n mod r != offset of head j; w % r == 0 on the tcgen05 path), split over
// host threads; streaming stores (no read-for-ownership of the lines).
void zero_unkept_rows_host(void* o, const dfa_impl::Geometry& g, size_t es) {
  const size_t piece = (size_t)g.dv * es, row = (size_t)g.h * piece;
  const int64_t rows = g.B * g.N;
  auto work = [&](int64_t r0, int64_t r1) {
    for (int64_t t = r0; t < r1; ++t) {
      const int64_t n = t % g.N;
      char* base = static_cast<char*>(o) + (size_t)t * row;
      for (int64_t j = 0; j < g.h; ++j) {
        if (n % g.r == g.offsets[j]) continue;
        char* dst = base + (size_t)j * piece;
#if defined(__x86_64__)
        if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && piece % 16 == 0) {
          const __m128i z = _mm_setzero_si128();
          for (size_t b = 0; b < piece; b += 16) _mm_stream_si128(reinterpret_cast<__m128i*>(dst + b), z);
          continue;
        }
#endif
        memset(dst, 0, piece);
      }
    }
#if defined(__x86_64__)
    _mm_sfence();
#endif
  };
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t nt = std::min<int64_t>(std::min<unsigned>(hw, 16u), std::max<int64_t>(1, rows / 4096));
  std::vector<std::thread> pool;
  try {  // helper i zeroes rows [rows i / nt, rows (i + 1) / nt)
    for (int64_t i = 1; i < nt; ++i) pool.emplace_back(work, rows * i / nt, rows * (i + 1) / nt);
  } catch (...) {  // no more threads: this one takes the helpers' share that was not started (nothing escapes the C-ABI)
    work(rows * (int64_t)(pool.size() + 1) / nt, rows);
  }
  work(0, rows / nt);
  for (auto& th : pool) th.join();
}

const void* mapped_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return (a.type == cudaMemoryTypeHost && a.devicePointer) ? a.devicePointer : nullptr;
}

}  // namespace

namespace dfa_impl {
dfa_status_t fail_msg(dfa_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}
}  // namespace dfa_impl

// Device staging for the host-buffer entry points, plus the copy streams and
// events of the chunked H2D -> kernel -> D2H pipeline (created on first use).
#ifndef DFA_HOST_CHUNKS
#define DFA_HOST_CHUNKS 16
#endif
constexpr int kHostChunks = DFA_HOST_CHUNKS;
struct dfa_workspace {
  void* dev = nullptr;
  size_t bytes = 0;
  bool pipe = false;
  cudaStream_t in_s = nullptr, out_s = nullptr;
  cudaEvent_t start = nullptr, in_done[kHostChunks] = {}, fwd_done[kHostChunks] = {};
};

extern "C" {

const char* dfa_last_error(void) { return g_last_error.c_str(); }
int32_t dfa_version(void) { return 100; }
int32_t dfa_last_launch_count(void) { return g_launches; }
void dfa_set_fault_perturb(int32_t armed) { g_fault.store(armed ? 1 : 0); }
int32_t dfa_get_fault_perturb(void) { return g_fault.load(); }
void dfa_set_path_override(int32_t path) { g_path_override.store(path); }
void dfa_set_multibranch_mode(int32_t mode) { g_mb_mode.store(mode); }
void dfa_set_multibranch_trace(uint64_t* trace) { dfa_impl::set_mb_trace(trace); }
void dfa_set_host_zero_copy(int32_t enabled) { g_host_zero_copy.store(enabled ? 1 : 0); }
void dfa_set_host_kept_out(int32_t enabled) { g_host_kept_out.store(enabled ? 1 : 0); }
void dfa_set_gemm_tile(int32_t bn) { dfa_impl::set_gemm_tile(bn); }

dfa_status_t dfa_host_transfer_bytes(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q,
                                     const void* k, const void* v, const void* o, int32_t with_lse, size_t* h2d,
                                     size_t* d2h) {
  dfa_impl::Geometry g;
  dfa_status_t st = resolve(cfg, batch, &g);
  if (st != DFA_OK) return st;
  if (!h2d || !d2h) return fail(DFA_ERR_DIMENSION, "dfa_host_transfer_bytes: null output");
  const size_t es = elem_size(dtype);
  *d2h = (size_t)(g.B * g.N * g.h * g.dv) * es + (with_lse ? (size_t)(g.B * g.h * g.N) * 4 : 0);
  const void* zq = g_host_zero_copy.load() ? mapped_host(q) : nullptr;
  const bool zero_copy = zq && mapped_host(k) && mapped_host(v) &&
                         pick_path(g, dtype, mapped_host(q), mapped_host(k), mapped_host(v), zq) ==
                             DFA_PATH_SM100_TCGEN05;
  if (!zero_copy) {
    *h2d = (size_t)(g.B * g.N * g.h) * (2 * g.d + g.dv) * es;
    return DFA_OK;
  }
  const void* zo = (o && g_host_kept_out.load()) ? mapped_host(o) : nullptr;
  const bool kept_out = zo && pick_path(g, dtype, mapped_host(q), mapped_host(k), mapped_host(v), zo) ==
                                  DFA_PATH_SM100_TCGEN05;
  // kept rows only: sum over heads and segments of the view sizes
  size_t rows = 0;
  for (int64_t j = 0; j < g.h; ++j)
    for (int64_t i = 0; i < g.n_seg; ++i) {
      int64_t m = 0;
      dfa_segment_view(g.N, g.w, g.r, i, g.offsets[j], nullptr, 0, &m);
      rows += (size_t)m;
    }
  *h2d = (size_t)g.B * rows * (size_t)(2 * g.d + g.dv) * es;
  if (kept_out) *d2h = (size_t)g.B * rows * (size_t)g.dv * es + (with_lse ? (size_t)(g.B * g.h * g.N) * 4 : 0);
  return DFA_OK;
}

dfa_status_t dfa_validate(const dfa_config_t* cfg, int32_t require_full_coverage) {
  return validate(cfg, require_full_coverage);
}

// attention.hpp:84-98
dfa_status_t dfa_segment_view(int64_t n, int64_t w, int64_t r, int64_t i, int64_t g, int64_t* rows, int64_t cap,
                              int64_t* count) {
  if (w < 1 || r < 1) return fail(DFA_ERR_CONFIG, "segment view: need w >= 1 and r >= 1");
  const int64_t n_seg = (n + w - 1) / w;
  if (i < 0 || i >= n_seg)
    return fail(DFA_ERR_OUT_OF_RANGE, "segment index %lld outside [0, %lld)", (long long)i, (long long)n_seg);
  if (g < 0 || g >= r)
    return fail(DFA_ERR_OUT_OF_RANGE, "segment offset %lld outside [0, %lld)", (long long)g, (long long)r);
  const int64_t begin = i * w;
  const int64_t end = begin + w < n ? begin + w : n;
  int64_t c = 0;
  for (int64_t row = begin + g; row < end; row += r) {
    if (rows && c < cap) rows[c] = row;
    ++c;
  }
  if (count) *count = c;
  return DFA_OK;
}

// attention.hpp:370-387
dfa_status_t dfa_flop_count(const dfa_config_t* cfg, uint64_t* dense, uint64_t* dilated, double* ratio) {
  dfa_status_t st = validate(cfg, 0);
  if (st != DFA_OK) return st;
  const uint64_t n = (uint64_t)cfg->seq_len, d = (uint64_t)cfg->head_dim, h = (uint64_t)cfg->num_heads;
  uint64_t dl = 0;
  const int64_t n_seg = (cfg->seq_len + cfg->segment_len - 1) / cfg->segment_len;
  for (int64_t j = 0; j < cfg->num_heads; ++j)
    for (int64_t i = 0; i < n_seg; ++i) {
      int64_t m = 0;
      dfa_segment_view(cfg->seq_len, cfg->segment_len, cfg->interval, i, cfg->head_offsets[j], nullptr, 0, &m);
      dl += 2u * (uint64_t)m * (uint64_t)m * d;
    }
  const uint64_t dn = h * 2u * n * n * d;
  if (dense) *dense = dn;
  if (dilated) *dilated = dl;
  if (ratio) *ratio = (double)dn / (double)dl;
  return DFA_OK;
}

dfa_status_t dfa_query_path(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, int32_t* path) {
  dfa_impl::Geometry g;
  dfa_status_t st = resolve(cfg, batch, &g);
  if (st != DFA_OK) return st;
  // Alignment is a property of the call's pointers; assume allocator alignment.
  static const char aligned[16] __attribute__((aligned(16))) = {0};
  *path = pick_path(g, dtype, aligned, aligned, aligned, aligned);
  return DFA_OK;
}

static dfa_status_t forward_impl(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q,
                                 const void* k, const void* v, void* o, float* lse, void* stream, uint64_t* trace,
                                 unsigned long long* watchdog = nullptr, bool apply_fault = true,
                                 const int64_t* ld = nullptr);

dfa_status_t dfa_forward(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q, const void* k,
                         const void* v, void* o, float* lse, void* stream) {
  return forward_impl(cfg, dtype, batch, q, k, v, o, lse, stream, nullptr);
}

dfa_status_t dfa_forward_strided(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q,
                                 int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* o,
                                 int64_t ldo, float* lse, void* stream) {
  const int64_t ld[4] = {ldq, ldk, ldv, ldo};
  return forward_impl(cfg, dtype, batch, q, k, v, o, lse, stream, nullptr, nullptr, true, ld);
}

dfa_status_t dfa_forward_traced(const dfa_config_t* cfg, int64_t batch, const void* q, const void* k, const void* v,
                                void* o, uint64_t* trace, void* stream) {
  if (!trace) return fail(DFA_ERR_DIMENSION, "dfa_forward_traced: null trace buffer");
  return forward_impl(cfg, DFA_BF16, batch, q, k, v, o, nullptr, stream, trace);
}

dfa_status_t dfa_forward_debug(const dfa_config_t* cfg, int64_t batch, const void* q, const void* k, const void* v,
                               void* o, uint64_t* trace, unsigned long long* watchdog, void* stream) {
  if (!trace) return fail(DFA_ERR_DIMENSION, "dfa_forward_debug: null trace buffer");
  return forward_impl(cfg, DFA_BF16, batch, q, k, v, o, nullptr, stream, trace, watchdog);
}

static dfa_status_t forward_impl(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q,
                                 const void* k, const void* v, void* o, float* lse, void* stream, uint64_t* trace,
                                 unsigned long long* watchdog, bool apply_fault, const int64_t* ld) {
  g_launches = 0;
  dfa_impl::Geometry g;
  dfa_status_t st = resolve(cfg, batch, &g);
  if (st != DFA_OK) return st;
  if (ld) {
    if (ld[0] < g.h * g.d || ld[1] < g.h * g.d || ld[2] < g.h * g.dv || ld[3] < g.h * g.dv)
      return fail(DFA_ERR_DIMENSION, "dfa_forward_strided: token strides (%lld, %lld, %lld, %lld) below h*d",
                  (long long)ld[0], (long long)ld[1], (long long)ld[2], (long long)ld[3]);
    g.ldq = ld[0];
    g.ldk = ld[1];
    g.ldv = ld[2];
    g.ldo = ld[3];
  }
  if (dtype != DFA_F32 && dtype != DFA_BF16 && dtype != DFA_F64)
    return fail(DFA_ERR_CONFIG, "dfa_forward: unknown dtype %d", (int)dtype);
  if (batch == 0) return DFA_OK;
  if (!q || !k || !v || !o) return fail(DFA_ERR_DIMENSION, "dfa_forward: null tensor pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int path = pick_path(g, dtype, q, k, v, o);
  cudaError_t err = cudaSuccess;
  int launches = 0;
  if (path == DFA_PATH_SM100_TCGEN05) {
    const char* why = "";
    launches = dfa_impl::launch_sm100(g, q, k, v, o, lse, s, &err, &why, trace, watchdog);
    if (launches == 0 && err != cudaSuccess)
      return fail(DFA_ERR_CUDA, "dfa_forward: sm100 path: %s (%s)", why, cudaGetErrorString(err));
  } else if (trace) {
    return fail(DFA_ERR_UNSUPPORTED, "dfa_forward_traced: only the tcgen05 path is instrumented");
  } else if (path == DFA_PATH_SIMT) {
    launches = dfa_impl::launch_simt(g, dtype, q, k, v, o, lse, s, &err);
  } else {
    return fail(DFA_ERR_UNSUPPORTED, "dfa_forward: forced tcgen05 path does not cover this call");
  }
  if (err != cudaSuccess) return fail(DFA_ERR_CUDA, "dfa_forward: launch failed: %s", cudaGetErrorString(err));
  if (apply_fault && g_fault.load()) {
    launches += dfa_impl::launch_perturb(dtype, o, s);
    err = cudaGetLastError();
    if (err != cudaSuccess) return fail(DFA_ERR_CUDA, "dfa_forward: fault hook: %s", cudaGetErrorString(err));
  }
  g_launches = launches;
  return DFA_OK;
}

dfa_status_t dfa_workspace_create(size_t bytes, dfa_workspace_t** ws) {
  if (!ws) return fail(DFA_ERR_DIMENSION, "dfa_workspace_create: null handle");
  auto* w = new dfa_workspace;
  if (bytes) {
    cudaError_t err = cudaMalloc(&w->dev, bytes);
    if (err != cudaSuccess) {
      delete w;
      return fail(DFA_ERR_CUDA, "dfa_workspace_create: %s", cudaGetErrorString(err));
    }
  }
  w->bytes = bytes;
  *ws = w;
  return DFA_OK;
}

dfa_status_t dfa_workspace_destroy(dfa_workspace_t* ws) {
  if (!ws) return DFA_OK;
  if (ws->pipe) {
    cudaStreamSynchronize(ws->in_s);
    cudaStreamSynchronize(ws->out_s);
    cudaEventDestroy(ws->start);
    for (int c = 0; c < kHostChunks; ++c) {
      cudaEventDestroy(ws->in_done[c]);
      cudaEventDestroy(ws->fwd_done[c]);
    }
    cudaStreamDestroy(ws->in_s);
    cudaStreamDestroy(ws->out_s);
  }
  if (ws->dev) cudaFree(ws->dev);
  delete ws;
  return DFA_OK;
}

dfa_status_t dfa_forward_host(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q,
                              const void* k, const void* v, void* o, float* lse, dfa_workspace_t* ws,
                              void* stream) {
  dfa_impl::Geometry g;
  dfa_status_t st = resolve(cfg, batch, &g);
  if (st != DFA_OK) return st;
  if (batch == 0) return DFA_OK;
  if (!ws) return fail(DFA_ERR_DIMENSION, "dfa_forward_host: null workspace");
  const size_t es = elem_size(dtype);
  const size_t bqk = (size_t)(g.B * g.N * g.h * g.d) * es;
  const size_t bv = (size_t)(g.B * g.N * g.h * g.dv) * es;
  const size_t bl = lse ? (size_t)(g.B * g.h * g.N) * 4 : 0;
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t need = up(bqk) * 2 + up(bv) * 2 + up(bl);
  if (ws->bytes < need)
    return fail(DFA_ERR_DIMENSION, "dfa_forward_host: workspace has %zu bytes, needs %zu", ws->bytes, need);
  char* base = static_cast<char*>(ws->dev);
  char* dq = base;
  char* dk = base + up(bqk);
  char* dv = base + 2 * up(bqk);
  char* dout = base + 2 * up(bqk) + up(bv);
  float* dl = lse ? reinterpret_cast<float*>(base + 2 * up(bqk) + 2 * up(bv)) : nullptr;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t err = cudaSuccess;
  if (!ws->pipe) {
    bool ok = cudaStreamCreateWithFlags(&ws->in_s, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&ws->out_s, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&ws->start, cudaEventDisableTiming) == cudaSuccess;
    for (int c = 0; ok && c < kHostChunks; ++c)
      ok = cudaEventCreateWithFlags(&ws->in_done[c], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&ws->fwd_done[c], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) return fail(DFA_ERR_CUDA, "dfa_forward_host: stream/event creation failed");
    ws->pipe = true;
  }
  // Zero-copy inputs: when q, k, v are pinned host memory mapped into the
  // device address space and the call takes the tcgen05 path, the kernel's
  // TMA boxes read the kept rows straight over PCIe -- half (r = 2) or less
  // of the tensors' bytes ever cross the bus, and no staging copy exists.
  const void* zq = g_host_zero_copy.load() ? mapped_host(q) : nullptr;
  const void* zk = zq ? mapped_host(k) : nullptr;
  const void* zv = zk ? mapped_host(v) : nullptr;
  const bool zero_copy = zv && pick_path(g, dtype, zq, zk, zv, dout) == DFA_PATH_SM100_TCGEN05;
  // Kept rows out in place: o itself is mapped pinned memory -- one launch
  // writes the kept rows straight into it (the only output bytes that cross
  // PCIe) while host threads zero-fill the rows no view keeps.
  const void* zo = zero_copy && g_host_kept_out.load() ? mapped_host(o) : nullptr;
  if (zo && pick_path(g, dtype, zq, zk, zv, zo) == DFA_PATH_SM100_TCGEN05) {
    const char* why = "";
    const int n = dfa_impl::launch_sm100(g, zq, zk, zv, const_cast<void*>(zo), dl, s, &err, &why, nullptr, nullptr,
                                         false, /*kept_only=*/true);
    if (n == 0 || err != cudaSuccess)
      return fail(DFA_ERR_CUDA, "dfa_forward_host: sm100 path: %s (%s)", why, cudaGetErrorString(err));
    int launches = n;
    if (lse && (err = cudaMemcpyAsync(lse, dl, bl, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return fail(DFA_ERR_CUDA, "dfa_forward_host: lse D2H: %s", cudaGetErrorString(err));
#ifndef DFA_PROBE_NO_HOST_ZERO
    zero_unkept_rows_host(o, g, es);  // host threads, concurrent with the kernel
#endif
    if ((err = cudaStreamSynchronize(s)) != cudaSuccess)
      return fail(DFA_ERR_CUDA, "dfa_forward_host: %s", cudaGetErrorString(err));
    if (g_fault.load()) {  // after the zero fill: element 0 may lie in a zero-filled row
      launches += dfa_impl::launch_perturb(dtype, const_cast<void*>(zo), s);
      if ((err = cudaStreamSynchronize(s)) != cudaSuccess)
        return fail(DFA_ERR_CUDA, "dfa_forward_host: fault hook: %s", cudaGetErrorString(err));
    }
    g_launches = launches;
    return DFA_OK;
  }
  // Pipeline over image chunks: H2D of chunk c+1 (copy engine 1) overlaps
  // the kernel of chunk c and the D2H of chunk c-1 (copy engine 2), so the
  // call costs ~max(H2D, D2H) instead of their sum.
  const int64_t n_chunks = std::min<int64_t>(kHostChunks, g.B);
  const int64_t per = (g.B + n_chunks - 1) / n_chunks;
  const size_t img_qk = bqk / (size_t)g.B, img_v = bv / (size_t)g.B, img_l = bl / (size_t)g.B;
  int launches = 0;
  if ((err = cudaEventRecord(ws->start, s)) != cudaSuccess ||
      (err = cudaStreamWaitEvent(ws->in_s, ws->start, 0)) != cudaSuccess)
    return fail(DFA_ERR_CUDA, "dfa_forward_host: %s", cudaGetErrorString(err));
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int64_t b0 = c * per, nb = std::min<int64_t>(per, g.B - b0);
    if (nb <= 0) break;
    const size_t oqk = (size_t)b0 * img_qk, ov = (size_t)b0 * img_v, ol = (size_t)b0 * img_l;
    if (zero_copy) {
      st = dfa_forward(cfg, dtype, nb, static_cast<const char*>(zq) + oqk, static_cast<const char*>(zk) + oqk,
                       static_cast<const char*>(zv) + ov, dout + ov, dl ? dl + ol / 4 : nullptr, stream);
      if (st != DFA_OK) return st;
      launches += g_launches;
    } else {
    if ((err = cudaMemcpyAsync(dq + oqk, static_cast<const char*>(q) + oqk, nb * img_qk, cudaMemcpyHostToDevice,
                               ws->in_s)) != cudaSuccess ||
        (err = cudaMemcpyAsync(dk + oqk, static_cast<const char*>(k) + oqk, nb * img_qk, cudaMemcpyHostToDevice,
                               ws->in_s)) != cudaSuccess ||
        (err = cudaMemcpyAsync(dv + ov, static_cast<const char*>(v) + ov, nb * img_v, cudaMemcpyHostToDevice,
                               ws->in_s)) != cudaSuccess ||
        (err = cudaEventRecord(ws->in_done[c], ws->in_s)) != cudaSuccess ||
        (err = cudaStreamWaitEvent(s, ws->in_done[c], 0)) != cudaSuccess)
      return fail(DFA_ERR_CUDA, "dfa_forward_host: H2D: %s", cudaGetErrorString(err));
    st = dfa_forward(cfg, dtype, nb, dq + oqk, dk + oqk, dv + ov, dout + ov, dl ? dl + ol / 4 : nullptr, stream);
    if (st != DFA_OK) return st;
    launches += g_launches;
    }
    if ((err = cudaEventRecord(ws->fwd_done[c], s)) != cudaSuccess ||
        (err = cudaStreamWaitEvent(ws->out_s, ws->fwd_done[c], 0)) != cudaSuccess ||
        (err = cudaMemcpyAsync(static_cast<char*>(o) + ov, dout + ov, nb * img_v, cudaMemcpyDeviceToHost,
                               ws->out_s)) != cudaSuccess ||
        (lse && (err = cudaMemcpyAsync(reinterpret_cast<char*>(lse) + ol, reinterpret_cast<char*>(dl) + ol,
                                       nb * img_l, cudaMemcpyDeviceToHost, ws->out_s)) != cudaSuccess))
      return fail(DFA_ERR_CUDA, "dfa_forward_host: D2H: %s", cudaGetErrorString(err));
  }
  if ((err = cudaStreamSynchronize(ws->out_s)) != cudaSuccess || (err = cudaStreamSynchronize(s)) != cudaSuccess)
    return fail(DFA_ERR_CUDA, "dfa_forward_host: %s", cudaGetErrorString(err));
  g_launches = launches;
  return DFA_OK;
}

static size_t up256(size_t x) { return (x + 255) & ~(size_t)255; }

dfa_status_t dfa_multibranch_workspace_bytes(const dfa_config_t* base, int32_t nb, dfa_dtype_t dtype, int64_t batch,
                                             size_t* bytes) {
  dfa_impl::Geometry g;
  dfa_status_t st = resolve(base, batch, &g);
  if (st != DFA_OK) return st;
  if (nb < 1 || nb > dfa_impl::kMaxBranches)
    return fail(DFA_ERR_CONFIG, "multibranch: need 1..%d branches, got %d", dfa_impl::kMaxBranches, (int)nb);
  const size_t es = elem_size(dtype);
  *bytes = (size_t)nb * (up256((size_t)(g.B * g.N * g.h * g.dv) * es) + up256((size_t)(g.B * g.h * g.N) * 4));
  return DFA_OK;
}

dfa_status_t dfa_forward_multibranch(const dfa_config_t* base, int32_t nb, const dfa_branch_t* branches,
                                     dfa_dtype_t dtype, int64_t batch, const void* q, const void* k, const void* v,
                                     void* o, float* lse, void* workspace, size_t ws_bytes, void* stream) {
  size_t need = 0;
  dfa_status_t st = dfa_multibranch_workspace_bytes(base, nb, dtype, batch, &need);
  if (st != DFA_OK) return st;
  if (!branches) return fail(DFA_ERR_CONFIG, "multibranch: null branch list");
  if (dtype != DFA_F32 && dtype != DFA_BF16) return fail(DFA_ERR_UNSUPPORTED, "multibranch: dtype %d (f32 / bf16)", (int)dtype);
  if (ws_bytes < need || !workspace)
    return fail(DFA_ERR_DIMENSION, "multibranch: workspace has %zu bytes, needs %zu", ws_bytes, need);
  g_launches = 0;
  // validate every branch before launching anything
  dfa_config_t cfgs[dfa_impl::kMaxBranches];
  dfa_impl::Geometry gb[dfa_impl::kMaxBranches];
  bool fused = dtype == DFA_BF16 && g_path_override.load() != DFA_PATH_SIMT;
  for (int b = 0; b < nb; ++b) {
    cfgs[b] = *base;
    cfgs[b].segment_len = branches[b].segment_len;
    cfgs[b].interval = branches[b].interval;
    cfgs[b].head_offsets = branches[b].head_offsets;
    st = resolve(&cfgs[b], batch, &gb[b]);
    if (st != DFA_OK) return st;
    fused = fused && dfa_impl::sm100_supported(gb[b], dtype, q, k, v, o);
  }
  if (batch == 0) return DFA_OK;
  if (!q || !k || !v || !o) return fail(DFA_ERR_DIMENSION, "multibranch: null tensor pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const dfa_impl::Geometry& g = gb[0];
  const size_t es = elem_size(dtype);
  const size_t ob = up256((size_t)(g.B * g.N * g.h * g.dv) * es), lb = up256((size_t)(g.B * g.h * g.N) * 4);
  cudaError_t err = cudaSuccess;
  int launches = 0;
  if (fused && nb > 1 && g_mb_mode.load() == DFA_MB_AUTO) {
    // Every branch and the LSE combine in one persistent tcgen05 kernel
    // (dfa_mb_sm100.cu); a set outside its envelope takes the per-branch path.
    const char* why = "";
    const int n = dfa_impl::launch_mb_sm100(gb, nb, q, k, v, o, lse, s, &err, &why, nullptr);
    if (n < 0) return fail(DFA_ERR_CUDA, "multibranch: %s (%s)", why, cudaGetErrorString(err));
    launches = n;
    if (n > 0) fused = false;  // done
  }
  if (launches > 0) {
    // fused single-kernel path taken
  } else if (fused) {
    // Fused epilogue combine: branch 0 writes o (zero rows included) and the
    // running lse; every later branch LSE-merges its kept rows into them in
    // its epilogue.  Stream order separates the branches.
    float* run_lse = lse ? lse : static_cast<float*>(workspace);
    for (int b = 0; b < nb; ++b) {
      const char* why = "";
      const int n = dfa_impl::launch_sm100(gb[b], q, k, v, o, run_lse, s, &err, &why, nullptr, nullptr, b > 0);
      if (n == 0 || err != cudaSuccess)
        return fail(DFA_ERR_CUDA, "multibranch: branch %d: %s (%s)", b, why, cudaGetErrorString(err));
      launches += n;
    }
  } else {
    // General path (fp32 validation mode, SIMT geometries): every branch
    // writes o_b and lse_b to the workspace, then one combine kernel.
    const void* outs[dfa_impl::kMaxBranches];
    const float* lses[dfa_impl::kMaxBranches];
    for (int b = 0; b < nb; ++b) {
      char* base_ptr = static_cast<char*>(workspace) + (size_t)b * (ob + lb);
      st = forward_impl(&cfgs[b], dtype, batch, q, k, v, base_ptr, reinterpret_cast<float*>(base_ptr + ob), stream,
                        nullptr, nullptr, false);
      if (st != DFA_OK) return st;
      launches += g_launches;
      outs[b] = base_ptr;
      lses[b] = reinterpret_cast<const float*>(base_ptr + ob);
    }
    launches += dfa_impl::launch_combine(dtype, g.B, g.N, g.h, g.dv, nb, outs, lses, o, lse, s, &err);
    if (err != cudaSuccess) return fail(DFA_ERR_CUDA, "multibranch combine: %s", cudaGetErrorString(err));
  }
  if (g_fault.load()) {
    launches += dfa_impl::launch_perturb(dtype, o, s);
    err = cudaGetLastError();
    if (err != cudaSuccess) return fail(DFA_ERR_CUDA, "multibranch: fault hook: %s", cudaGetErrorString(err));
  }
  g_launches = launches;
  return DFA_OK;
}

dfa_status_t dfa_multibranch_plan(const dfa_config_t* base, int32_t nb, const dfa_branch_t* branches, int64_t batch,
                                  int32_t grid, void* descs, size_t capacity, int32_t* n_desc, int32_t* lcm_interval,
                                  int32_t* rows_per_group_log2, int32_t* desc_bytes) {
  if (nb < 2 || nb > dfa_impl::kMaxBranches)
    return fail(DFA_ERR_CONFIG, "multibranch plan: need 2..%d branches, got %d", dfa_impl::kMaxBranches, (int)nb);
  if (!branches || !n_desc || !lcm_interval || !rows_per_group_log2 || !desc_bytes)
    return fail(DFA_ERR_DIMENSION, "multibranch plan: null argument");
  dfa_config_t cfgs[dfa_impl::kMaxBranches];
  dfa_impl::Geometry gb[dfa_impl::kMaxBranches];
  for (int b = 0; b < nb; ++b) {
    cfgs[b] = *base;
    cfgs[b].segment_len = branches[b].segment_len;
    cfgs[b].interval = branches[b].interval;
    cfgs[b].head_offsets = branches[b].head_offsets;
    dfa_status_t st = resolve(&cfgs[b], batch, &gb[b]);
    if (st != DFA_OK) return st;
  }
  const char* why = "";
  if (!dfa_impl::mb_plan_host(gb, nb, grid > 0 ? grid : 148, descs, capacity, n_desc, lcm_interval,
                              rows_per_group_log2, desc_bytes, &why))
    return fail(DFA_ERR_UNSUPPORTED, "multibranch plan: %s", why);
  return DFA_OK;
}

dfa_status_t dfa_backward_workspace_bytes(const dfa_config_t* cfg, int64_t batch, size_t* bytes) {
  dfa_impl::Geometry g;
  dfa_status_t st = resolve(cfg, batch, &g);
  if (st != DFA_OK) return st;
  if (!bytes) return fail(DFA_ERR_DIMENSION, "dfa_backward_workspace_bytes: null output");
  *bytes = up256((size_t)(g.B * g.h * g.N) * 4);
  return DFA_OK;
}

// Backward of dfa_forward (the reference's tape for the dilated branch of
// detail::attention_mix, encoder.hpp:204-219).  lse is dfa_forward's output.
dfa_status_t dfa_backward(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q, const void* k,
                          const void* v, const void* o, const float* lse, const void* dout, void* dq, void* dk,
                          void* dv, void* workspace, size_t ws_bytes, void* stream) {
  g_launches = 0;
  dfa_impl::Geometry g;
  dfa_status_t st = resolve(cfg, batch, &g);
  if (st != DFA_OK) return st;
  if (dtype != DFA_F32 && dtype != DFA_BF16) return fail(DFA_ERR_UNSUPPORTED, "dfa_backward: dtype %d (f32 / bf16)", (int)dtype);
  if (batch == 0) return DFA_OK;
  if (!q || !k || !v || !o || !lse || !dout || !dq || !dk || !dv)
    return fail(DFA_ERR_DIMENSION, "dfa_backward: null tensor pointer");
  const size_t need = up256((size_t)(g.B * g.h * g.N) * 4);
  if (!workspace || ws_bytes < need)
    return fail(DFA_ERR_DIMENSION, "dfa_backward: workspace has %zu bytes, needs %zu", ws_bytes, need);
  cudaError_t err = cudaSuccess;
  const char* why = "";
  const bool allow = g_path_override.load() != DFA_PATH_SIMT;
  const int n = dfa_impl::launch_backward(g, dtype, q, k, v, o, dout, lse, static_cast<float*>(workspace), dq, dk, dv,
                                          reinterpret_cast<cudaStream_t>(stream), &err, allow, &why);
  if (err != cudaSuccess || n == 0)
    return fail(DFA_ERR_CUDA, "dfa_backward: launch failed: %s (%s)", cudaGetErrorString(err), why);
  g_launches = n;
  return DFA_OK;
}

// tensor.hpp:175-195 matmul + the layers' epilogue (include/dfa.h).
dfa_status_t dfa_gemm(dfa_dtype_t dtype, int64_t batch, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                      int64_t sa, const void* B, int64_t ldb, int64_t sb, void* D, int64_t ldd, int64_t sd,
                      const void* C, int64_t ldc, float beta, const void* bias, int32_t gelu, void* stream) {
  g_launches = 0;
  if (dtype != DFA_F32 && dtype != DFA_BF16) return fail(DFA_ERR_UNSUPPORTED, "dfa_gemm: dtype %d (f32 / bf16)", (int)dtype);
  if (batch < 0 || M < 0 || N < 0 || K < 0)
    return fail(DFA_ERR_DIMENSION, "dfa_gemm: negative extent (batch %lld, M %lld, N %lld, K %lld)", (long long)batch,
                (long long)M, (long long)N, (long long)K);
  if (lda < K || ldb < N || ldd < N || (C && ldc < N))
    return fail(DFA_ERR_DIMENSION, "dfa_gemm: row strides below the row widths");
  if (batch == 0 || M == 0 || N == 0) return DFA_OK;
  if (!A || !B || !D) return fail(DFA_ERR_DIMENSION, "dfa_gemm: null operand");
  const char* why = "";
  if (!dfa_impl::gemm_rowmajor(dtype, M, N, K, A, lda, sa, B, ldb, sb, D, ldd, sd, C, ldc, beta, bias, (int)batch,
                               reinterpret_cast<cudaStream_t>(stream), &why, gelu != 0))
    return fail(DFA_ERR_CUDA, "dfa_gemm: %s", why);
  g_launches = 1;
  return DFA_OK;
}

// ------------------------------------------------------------ §8(f) 1-2

static dfa_status_t layer_geometry(const dfa_config_t* cfg, int64_t batch, dfa_impl::Geometry* g, const char* who) {
  dfa_status_t st = validate(cfg, 1);  // attention.hpp:343 / EncoderConfig::validate: full coverage
  if (st != DFA_OK) return st;
  st = resolve(cfg, batch, g);
  if (st != DFA_OK) return st;
  if (cfg->value_dim != 0 && cfg->value_dim != cfg->head_dim)
    return fail(DFA_ERR_DIMENSION, "%s: value_dim must equal head_dim", who);
  if (g->h * g->d > 1024) return fail(DFA_ERR_UNSUPPORTED, "%s: model dim %lld > 1024", who, (long long)(g->h * g->d));
  return DFA_OK;
}

dfa_status_t dfa_multi_head_workspace_bytes(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch,
                                            size_t* bytes) {
  dfa_impl::Geometry g;
  dfa_status_t st = layer_geometry(cfg, batch, &g, "multi_head_dilated");
  if (st != DFA_OK) return st;
  if (dtype != DFA_F32 && dtype != DFA_BF16)
    return fail(DFA_ERR_UNSUPPORTED, "multi_head_dilated: dtype %d (f32 / bf16)", (int)dtype);
  const size_t es = elem_size(dtype), D = (size_t)(g.h * g.d);
  *bytes = 4 * up256((size_t)(g.B * g.N) * D * es) + up256(3 * D * D * es);
  return DFA_OK;
}

// x [M, D] -> qkv [M, 3, h, d] with ONE GEMM against the packed [D, 3, h, d]
// weights, then the core reads q / k / v as column blocks (token stride 3hd).
static dfa_status_t fused_qkv_attention(const dfa_config_t* cfg, dfa_dtype_t dtype, const dfa_impl::Geometry& g,
                                        const void* x, const void* wq, const void* wk, const void* wv, char* qkv,
                                        char* wpack, void* att, cudaStream_t s, int* launches,
                                        const char* who) {
  const int64_t M = g.B * g.N, D = g.h * g.d;
  const char* why = "";
  *launches += dfa_impl::launch_pack_qkv(dtype, wq, wk, wv, wpack, g.h, D, g.d, s);
  if (!dfa_impl::gemm_rowmajor(dtype, M, 3 * D, D, x, D, 0, wpack, 3 * D, 0, qkv, 3 * D, 0, nullptr, 0, 0.0f, nullptr,
                               1, s, &why))
    return fail(DFA_ERR_CUDA, "%s: QKV projection: %s", who, why);
  ++*launches;
  const size_t es = elem_size(dtype);
  const int64_t ld[4] = {3 * D, 3 * D, 3 * D, D};
  dfa_status_t st = forward_impl(cfg, dtype, g.B, qkv, qkv + D * es, qkv + 2 * D * es, att, nullptr,
                                 reinterpret_cast<void*>(s), nullptr, nullptr, false, ld);
  if (st != DFA_OK) return st;
  *launches += g_launches;
  return DFA_OK;
}

// Offset-class split of a multi-head layer (bf16, r > 1, r | N, r | w): head j
// only ever reads rows n = gamma_j (mod r) of its q / k / v, and its attention
// output is zero on every other row.  Grouping heads by gamma, each class g runs
//   qkv_g = x[rows = g mod r] W_qkv[class g columns]   (M / r rows)
//   att_g = core(qkv_g) on the class's t'-streams       (N / r, w / r, r = 1)
//   out[rows = g mod r] = att_g Wo[class g rows] (+ bias, + C)
// -- the same result as the dense layer with 1/r of the projection FLOPs and
// bytes and no zero rows materialised.  qkv holds the classes back to back;
// the class-major Wo copy sits behind them in the same region (the dense
// layout needs 3 M D elements there, this one 3 M D / r + D D).
static bool class_split_ok(const dfa_impl::Geometry& g, dfa_dtype_t dtype) {
  if (dtype != DFA_BF16 || g.r < 2 || g.N % g.r != 0 || g.w % g.r != 0 || g_path_override.load() == DFA_PATH_SIMT)
    return false;
  // the class-major Wo copy must fit behind the classes' qkv in the dense
  // layout's 3 M D region (not the case for tiny M against a wide model)
  const size_t es = elem_size(dtype), M = (size_t)(g.B * g.N), D = (size_t)(g.h * g.d);
  return up256(3 * (M / (size_t)g.r) * D * es) + D * D * es <= 3 * up256(M * D * es);
}

static dfa_status_t class_split_layer(const dfa_config_t* cfg, dfa_dtype_t dtype, const dfa_impl::Geometry& g,
                                      const void* x, const void* wq, const void* wk, const void* wv, const void* wo,
                                      const void* bias, const void* resid, void* out, char* qkv, char* att,
                                      char* wpack, cudaStream_t s, int* launches, const char* who) {
  const int64_t M = g.B * g.N, D = g.h * g.d, r = g.r, Mr = M / r;
  const size_t es = elem_size(dtype);
  char* wopack = qkv + up256((size_t)(3 * Mr * D) * es);
  *launches += dfa_impl::launch_pack_class(dtype, wq, wk, wv, wo, wpack, wopack, g.h, D, g.d, g.offsets, s);
  const char* why = "";
  bool equal = g.h % r == 0;  // every class holds h / r heads (e.g. spread offsets j mod r)
  for (int64_t gc = 0; equal && gc < r; ++gc) {
    int64_t cnt = 0;
    for (int64_t j = 0; j < g.h; ++j) cnt += g.offsets[j] == gc ? 1 : 0;
    equal = cnt == g.h / r;
  }
  if (equal) {
    // Equal classes: the r classes' buffers lie back to back, so each stage is
    // ONE call -- a strided-batched GEMM over the classes (A rows offset by the
    // class, weight columns / rows by the class's block) and one core launch
    // with batch r B (class-major images): fuller waves than r separate calls.
    const int64_t hd = (g.h / r) * g.d;
    if (!dfa_impl::gemm_rowmajor(dtype, Mr, 3 * hd, D, x, r * D, D, wpack, 3 * D, 3 * hd, qkv, 3 * hd, Mr * 3 * hd,
                                 nullptr, 0, 0.0f, nullptr, (int)r, s, &why))
      return fail(DFA_ERR_CUDA, "%s: QKV projection: %s", who, why);
    ++*launches;
    std::vector<int64_t> zero_offs((size_t)(g.h / r), 0);
    dfa_config_t cc = *cfg;
    cc.seq_len = g.N / r;
    cc.segment_len = g.w / r;
    cc.interval = 1;
    cc.num_heads = g.h / r;
    cc.head_offsets = zero_offs.data();
    const int64_t ld[4] = {3 * hd, 3 * hd, 3 * hd, hd};
    dfa_status_t st = forward_impl(&cc, dtype, g.B * r, qkv, qkv + hd * es, qkv + 2 * hd * es, att, nullptr,
                                   reinterpret_cast<void*>(s), nullptr, nullptr, false, ld);
    if (st != DFA_OK) return st;
    *launches += g_launches;
    if (!dfa_impl::gemm_rowmajor(dtype, Mr, D, hd, att, hd, Mr * hd, wopack, D, hd * D, out, r * D, D, resid, r * D,
                                 resid ? 1.0f : 0.0f, bias, (int)r, s, &why))
      return fail(DFA_ERR_CUDA, "%s: output projection: %s", who, why);
    ++*launches;
    return DFA_OK;
  }
  int64_t start = 0;  // first class-major head position of the class
  for (int64_t gc = 0; gc < r; ++gc) {
    int64_t cnt = 0;
    for (int64_t j = 0; j < g.h; ++j) cnt += g.offsets[j] == gc ? 1 : 0;
    if (cnt == 0) continue;  // full coverage (validated) makes every class non-empty
    const int64_t hd = cnt * g.d;
    char* q_g = qkv + (size_t)(3 * Mr * start * g.d) * es;
    char* a_g = att + (size_t)(Mr * start * g.d) * es;
    if (!dfa_impl::gemm_rowmajor(dtype, Mr, 3 * hd, D, static_cast<const char*>(x) + gc * D * es, r * D, 0,
                                 wpack + (size_t)(3 * start * g.d) * es, 3 * D, 0, q_g, 3 * hd, 0, nullptr, 0, 0.0f,
                                 nullptr, 1, s, &why))
      return fail(DFA_ERR_CUDA, "%s: QKV projection (class %lld): %s", who, (long long)gc, why);
    ++*launches;
    std::vector<int64_t> zero_offs((size_t)cnt, 0);
    dfa_config_t cc = *cfg;
    cc.seq_len = g.N / r;
    cc.segment_len = g.w / r;
    cc.interval = 1;
    cc.num_heads = cnt;
    cc.head_offsets = zero_offs.data();
    const int64_t ld[4] = {3 * hd, 3 * hd, 3 * hd, hd};
    dfa_status_t st = forward_impl(&cc, dtype, g.B, q_g, q_g + hd * es, q_g + 2 * hd * es, a_g, nullptr,
                                   reinterpret_cast<void*>(s), nullptr, nullptr, false, ld);
    if (st != DFA_OK) return st;
    *launches += g_launches;
    const void* c_g = resid ? static_cast<const char*>(resid) + gc * D * es : nullptr;
    if (!dfa_impl::gemm_rowmajor(dtype, Mr, D, hd, a_g, hd, 0, wopack + (size_t)(start * g.d * D) * es, D, 0,
                                 static_cast<char*>(out) + gc * D * es, r * D, 0, c_g, r * D, c_g ? 1.0f : 0.0f,
                                 bias, 1, s, &why))
      return fail(DFA_ERR_CUDA, "%s: output projection (class %lld): %s", who, (long long)gc, why);
    ++*launches;
    start += cnt;
  }
  return DFA_OK;
}

dfa_status_t dfa_multi_head_dilated(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* x,
                                    const void* wq, const void* wk, const void* wv, const void* wo, void* out,
                                    void* workspace, size_t ws_bytes, void* stream) {
  g_launches = 0;
  dfa_impl::Geometry g;
  dfa_status_t st = layer_geometry(cfg, batch, &g, "multi_head_dilated");
  if (st != DFA_OK) return st;
  size_t need = 0;
  st = dfa_multi_head_workspace_bytes(cfg, dtype, batch, &need);
  if (st != DFA_OK) return st;
  if (!workspace || ws_bytes < need)
    return fail(DFA_ERR_DIMENSION, "multi_head_dilated: workspace has %zu bytes, needs %zu", ws_bytes, need);
  if (batch == 0) return DFA_OK;
  if (!x || !wq || !wk || !wv || !wo || !out) return fail(DFA_ERR_DIMENSION, "multi_head_dilated: null pointer");
  const int64_t M = g.B * g.N, D = g.h * g.d;
  const size_t es = elem_size(dtype), act = up256((size_t)(M * D) * es);
  char* base = static_cast<char*>(workspace);
  char* qkv = base;                   // [M, 3, h, d]
  void* att = base + 3 * act;         // [M, h, d]
  char* wpack = base + 4 * act;       // [D, 3, h, d]
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int launches = 0;
  if (class_split_ok(g, dtype)) {
    st = class_split_layer(cfg, dtype, g, x, wq, wk, wv, wo, nullptr, nullptr, out, qkv, static_cast<char*>(att),
                           wpack, s, &launches, "multi_head_dilated");
    if (st != DFA_OK) return st;
  } else {
    st = fused_qkv_attention(cfg, dtype, g, x, wq, wk, wv, qkv, wpack, att, s, &launches, "multi_head_dilated");
    if (st != DFA_OK) return st;
    const char* why = "";
    if (!dfa_impl::gemm_rowmajor(dtype, M, D, D, att, D, 0, wo, D, 0, out, D, 0, nullptr, 0, 0.0f, nullptr, 1, s,
                                 &why))
      return fail(DFA_ERR_CUDA, "multi_head_dilated: output projection: %s", why);
    ++launches;
  }
  if (g_fault.load()) launches += dfa_impl::launch_perturb(dtype, out, s);
  g_launches = launches;
  return DFA_OK;
}

// attention.hpp:340-360 on HOST buffers (synchronous; the reference-shaped
// C++ adapter dfa::multi_head_dilated calls this).
dfa_status_t dfa_multi_head_host_workspace_bytes(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch,
                                                 size_t* bytes) {
  size_t dev = 0;
  dfa_status_t st = dfa_multi_head_workspace_bytes(cfg, dtype, batch, &dev);
  if (st != DFA_OK) return st;
  const size_t es = elem_size(dtype), D = (size_t)(cfg->num_heads * cfg->head_dim);
  *bytes = dev + 2 * up256((size_t)(batch * cfg->seq_len) * D * es) + 4 * up256(D * D * es);
  return DFA_OK;
}

dfa_status_t dfa_multi_head_dilated_host(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* x,
                                         const void* wq, const void* wk, const void* wv, const void* wo, void* out,
                                         dfa_workspace_t* ws) {
  size_t need = 0, dev_need = 0;
  dfa_status_t st = dfa_multi_head_host_workspace_bytes(cfg, dtype, batch, &need);
  if (st != DFA_OK) return st;
  st = dfa_multi_head_workspace_bytes(cfg, dtype, batch, &dev_need);
  if (st != DFA_OK) return st;
  if (!ws || ws->bytes < need)
    return fail(DFA_ERR_DIMENSION, "multi_head_dilated: workspace has %zu bytes, needs %zu", ws ? ws->bytes : 0,
                need);
  if (batch == 0) return DFA_OK;
  if (!x || !wq || !wk || !wv || !wo || !out) return fail(DFA_ERR_DIMENSION, "multi_head_dilated: null pointer");
  const size_t es = elem_size(dtype), D = (size_t)(cfg->num_heads * cfg->head_dim);
  const size_t act = (size_t)(batch * cfg->seq_len) * D * es, wb = D * D * es;
  char* base = static_cast<char*>(ws->dev);
  char* dx = base + dev_need;
  char* dout = dx + up256(act);
  char* dw[4];
  for (int i = 0; i < 4; ++i) dw[i] = dout + up256(act) + i * up256(wb);
  const void* hw[4] = {wq, wk, wv, wo};
  cudaError_t err = cudaMemcpy(dx, x, act, cudaMemcpyHostToDevice);
  for (int i = 0; i < 4 && err == cudaSuccess; ++i) err = cudaMemcpy(dw[i], hw[i], wb, cudaMemcpyHostToDevice);
  if (err != cudaSuccess) return fail(DFA_ERR_CUDA, "multi_head_dilated: H2D: %s", cudaGetErrorString(err));
  st = dfa_multi_head_dilated(cfg, dtype, batch, dx, dw[0], dw[1], dw[2], dw[3], dout, base, dev_need, nullptr);
  if (st != DFA_OK) return st;
  if ((err = cudaMemcpy(out, dout, act, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return fail(DFA_ERR_CUDA, "multi_head_dilated: D2H: %s", cudaGetErrorString(err));
  return DFA_OK;
}

dfa_status_t dfa_encoder_block_workspace_bytes(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch,
                                               int64_t hidden, size_t* bytes) {
  dfa_impl::Geometry g;
  dfa_status_t st = layer_geometry(cfg, batch, &g, "encoder_block");
  if (st != DFA_OK) return st;
  if (dtype != DFA_F32 && dtype != DFA_BF16)
    return fail(DFA_ERR_UNSUPPORTED, "encoder_block: dtype %d (f32 / bf16)", (int)dtype);
  if (hidden < 1) return fail(DFA_ERR_CONFIG, "encoder: mlp_ratio must yield a positive width");
  const size_t es = elem_size(dtype), D = (size_t)(g.h * g.d);
  const size_t act = up256((size_t)(g.B * g.N) * D * es);
  *bytes = 6 * act + up256((size_t)(g.B * g.N * hidden) * es) + up256(3 * D * D * es);
  return DFA_OK;
}

dfa_status_t dfa_encoder_block_forward(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* x,
                                       const dfa_block_weights_t* wt, void* out, void* workspace, size_t ws_bytes,
                                       void* stream) {
  g_launches = 0;
  if (!wt) return fail(DFA_ERR_DIMENSION, "encoder_block: null weights");
  dfa_impl::Geometry g;
  dfa_status_t st = layer_geometry(cfg, batch, &g, "encoder_block");
  if (st != DFA_OK) return st;
  size_t need = 0;
  st = dfa_encoder_block_workspace_bytes(cfg, dtype, batch, wt->hidden, &need);
  if (st != DFA_OK) return st;
  if (!workspace || ws_bytes < need)
    return fail(DFA_ERR_DIMENSION, "encoder_block: workspace has %zu bytes, needs %zu", ws_bytes, need);
  if (batch == 0) return DFA_OK;
  const void* ptrs[] = {wt->ln1_g, wt->ln1_b, wt->wq, wt->wk, wt->wv, wt->wo, wt->bo,
                        wt->ln2_g, wt->ln2_b, wt->w1, wt->b1, wt->w2, wt->b2};
  for (const void* p : ptrs)
    if (!p) return fail(DFA_ERR_DIMENSION, "encoder_block: null weight pointer");
  if (!x || !out) return fail(DFA_ERR_DIMENSION, "encoder_block: null tensor pointer");
  const int64_t M = g.B * g.N, D = g.h * g.d, H = wt->hidden;
  const size_t es = elem_size(dtype), act = up256((size_t)(M * D) * es);
  char* base = static_cast<char*>(workspace);
  void* ln = base;
  char* qkv = base + act;        // [M, 3, h, d]
  void* att = base + 4 * act;
  void* x1 = base + 5 * act;
  char* hid = base + 6 * act;
  char* wpack = hid + up256((size_t)(M * H) * es);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const char* why = "";
  int launches = 0;
  auto gemm = [&](int64_t m, int64_t n, int64_t k, const void* a, const void* b, void* d, const void* c,
                  const void* bias, bool gelu = false) {
    ++launches;
    return dfa_impl::gemm_rowmajor(dtype, m, n, k, a, k, 0, b, n, 0, d, n, 0, c, n, c ? 1.0f : 0.0f, bias, 1, s, &why,
                                   gelu);
  };
  launches += dfa_impl::launch_layer_norm(dtype, x, wt->ln1_g, wt->ln1_b, ln, M, (int)D, s);
  if (class_split_ok(g, dtype)) {  // x1 = x + attention_mix(LN1 x) Wo + bo, per offset class
    st = class_split_layer(cfg, dtype, g, ln, wt->wq, wt->wk, wt->wv, wt->wo, wt->bo, x, x1, qkv,
                           static_cast<char*>(att), wpack, s, &launches, "encoder_block");
    if (st != DFA_OK) return st;
  } else {
    st = fused_qkv_attention(cfg, dtype, g, ln, wt->wq, wt->wk, wt->wv, qkv, wpack, att, s, &launches,
                             "encoder_block");
    if (st != DFA_OK) return st;
    if (!gemm(M, D, D, att, wt->wo, x1, x, wt->bo)) return fail(DFA_ERR_CUDA, "encoder_block: wo: %s", why);
  }
  launches += dfa_impl::launch_layer_norm(dtype, x1, wt->ln2_g, wt->ln2_b, ln, M, (int)D, s);
  // GELU in the reference's erf form (tensor.hpp:262-265) inside the w1
  // GEMM's epilogue -- no separate pass over the hidden activations.
  if (!gemm(M, H, D, ln, wt->w1, hid, nullptr, wt->b1, true)) return fail(DFA_ERR_CUDA, "encoder_block: w1+gelu: %s", why);
  if (!gemm(M, D, H, hid, wt->w2, out, x1, wt->b2)) return fail(DFA_ERR_CUDA, "encoder_block: w2: %s", why);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return fail(DFA_ERR_CUDA, "encoder_block: %s", cudaGetErrorString(err));
  g_launches = launches;
  return DFA_OK;
}

dfa_status_t dfa_workspace_bytes(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, int32_t with_lse,
                                 size_t* bytes) {
  dfa_impl::Geometry g;
  dfa_status_t st = resolve(cfg, batch, &g);
  if (st != DFA_OK) return st;
  const size_t es = elem_size(dtype);
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  *bytes = up((size_t)(g.B * g.N * g.h * g.d) * es) * 2 + up((size_t)(g.B * g.N * g.h * g.dv) * es) * 2 +
           (with_lse ? up((size_t)(g.B * g.h * g.N) * 4) : 0);
  return DFA_OK;
}

// attention.hpp:280-301 on host buffers: single head at `head_offset`.
dfa_status_t dfa_dilated_attention_host(const dfa_config_t* cfg, dfa_dtype_t dtype, const void* q, const void* k,
                                        const void* v, int64_t head_offset, int32_t workers, void* out,
                                        dfa_workspace_t* ws) {
  (void)workers;
  dfa_status_t st = validate(cfg, 0);
  if (st != DFA_OK) return st;
  if (head_offset < 0 || head_offset >= cfg->interval)
    return fail(DFA_ERR_OUT_OF_RANGE, "dilated_attention: head offset %lld outside [0, %lld)",
                (long long)head_offset, (long long)cfg->interval);
  dfa_config_t one = *cfg;
  one.num_heads = 1;
  one.head_offsets = &head_offset;
  return dfa_forward_host(&one, dtype, 1, q, k, v, out, nullptr, ws, nullptr);
}

}  // extern "C"
