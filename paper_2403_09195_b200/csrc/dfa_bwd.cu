// Backward of the Dilated Flash Attention core:
// given q, k, v, the forward output o, its per-row log-sum-exp lse and the
// incoming gradient dO, produce dq, dk, dv -- what the reference's tape
// computes for the dilated branch of detail::attention_mix
// (encoder.hpp:204-219; ops autodiff.hpp:99-179, 269-289).
//
// Flash-style recomputation, no N x N or m x m buffers:
//   P_ij  = exp(s_ij * sc - lse_i)            (s = q_i . k_j, sc after the dot)
//   Delta_i = dO_i . O_i                      (== rowsum(dP o P), softmax bwd)
//   dS_ij = P_ij (dO_i . v_j - Delta_i)
//   dv_j  = sum_i P_ij dO_i,  dk_j = sc sum_i dS_ij q_i,  dq_i = sc sum_j dS_ij k_j
// Three kernels, all deterministic (no atomics; every output row is written
// by exactly one thread group):
//   delta_kernel  Delta for every row (one warp per row)
//   dkdv_kernel   CTA = (image, head, segment, 128/PARTS key rows of the view)
//   dq_kernel     CTA = (image, head, segment, 128/PARTS query rows of the view)
// A row of width DMAX is split over PARTS adjacent lanes (32 columns each) so
// the per-row state stays in registers; dot products reduce with shuffles.
// Rows no view selects get exact zeros (their gradient is 0).  fp32
// arithmetic, f32 or bf16 I/O, any geometry the forward SIMT kernel takes.
#include <cuda_bf16.h>
#include <math.h>

#include <algorithm>

#include "dfa_internal.h"

namespace dfa_impl {
namespace {

struct BwdParams {
  int64_t N, w, r, h, d, dv, n_chunks;
  float scale;
  int32_t offsets[kMaxHeads];
};

template <typename T>
__device__ __forceinline__ float ld(const T* p);
template <>
__device__ __forceinline__ float ld<float>(const float* p) {
  return *p;
}
template <>
__device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ T cvt(float x);
template <>
__device__ __forceinline__ float cvt<float>(float x) {
  return x;
}
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

template <int PARTS>
__device__ __forceinline__ float part_sum(float x) {
#pragma unroll
  for (int o = PARTS / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Segment geometry shared by the kernels (make_segment_view closed form,
// attention.hpp:84-98): view rows are seg_begin + g + t*r, t < m.
struct SegView {
  int64_t begin, rows, m;
};
__device__ __forceinline__ SegView seg_view(const BwdParams& p, int64_t seg, int64_t g) {
  SegView s;
  s.begin = seg * p.w;
  const int64_t end = min(s.begin + p.w, p.N);
  s.rows = end - s.begin;
  s.m = g >= s.rows ? 0 : (s.rows - g + p.r - 1) / p.r;
  return s;
}

// Delta_i = dO_i . O_i for every row of [B, N, h, dv]; delta is [B, h, N].
// One thread per row: 16-byte vector loads when the row allows them (the
// row-of-a-warp form issued 2-byte loads and int64 divisions per row).
template <typename T>
__global__ void __launch_bounds__(256) delta_kernel(const T* __restrict__ o, const T* __restrict__ dout,
                                                    float* __restrict__ delta, int64_t rows, int64_t N, int64_t h,
                                                    int64_t dv) {
  constexpr int V = 16 / sizeof(T);
  const bool vec = dv % V == 0 && ((reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(dout)) & 15u) == 0;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < rows;
       row += (int64_t)gridDim.x * blockDim.x) {
    const T* a = o + row * dv;
    const T* b = dout + row * dv;
    float acc = 0.0f;
    if (vec && dv == 64) {  // the common head width: all 16 loads in flight at once
      uint4 x[64 / V], y[64 / V];
#pragma unroll
      for (int i = 0; i < 64 / V; ++i) {
        x[i] = reinterpret_cast<const uint4*>(a)[i];
        y[i] = reinterpret_cast<const uint4*>(b)[i];
      }
#pragma unroll
      for (int i = 0; i < 64 / V; ++i) {
        const T* xa = reinterpret_cast<const T*>(&x[i]);
        const T* ya = reinterpret_cast<const T*>(&y[i]);
#pragma unroll
        for (int e = 0; e < V; ++e) acc = fmaf(ld(xa + e), ld(ya + e), acc);
      }
    } else if (vec) {
      for (int64_t c = 0; c < dv; c += V) {
        const uint4 x = *reinterpret_cast<const uint4*>(a + c);
        const uint4 y = *reinterpret_cast<const uint4*>(b + c);
        const T* xa = reinterpret_cast<const T*>(&x);
        const T* ya = reinterpret_cast<const T*>(&y);
#pragma unroll
        for (int e = 0; e < V; ++e) acc = fmaf(ld(xa + e), ld(ya + e), acc);
      }
    } else {
      for (int64_t c = 0; c < dv; ++c) acc = fmaf(ld(a + c), ld(b + c), acc);
    }
    const int64_t j = row % h, rest = row / h;
    const int64_t n = rest % N, bb = rest / N;
    delta[(bb * h + j) * N + n] = acc;
  }
}

// Delta on the tcgen05 path (bf16, dv = 64, w % r == 0): only the rows a
// view keeps (n % r == gamma_j) -- every other row of O is exactly zero and
// its Delta is never read -- so half (r = 2) to 1/8 of the O / dO bytes of
// delta_kernel.  Eight lanes share a 128-byte row (fully coalesced 16-byte
// loads: a thread-per-row form at a 1.5 KB row stride ran at ~2 TB/s), a
// warp covers 4 rows per load and 16 rows per iteration with all 8 loads in
// flight; the dot product reduces over the 8 lanes with shuffles.
__global__ void __launch_bounds__(256) delta_kept_kernel(const uint4* __restrict__ o, const uint4* __restrict__ dout,
                                                         float* __restrict__ delta, int64_t B, int64_t N, int64_t r,
                                                         int64_t h, const __grid_constant__ BwdParams p) {
  // 32-bit index decode (the launcher guarantees B * h * N < 2^31): int64
  // division is a long emulated sequence and made this pass issue-bound
  const uint32_t T = (uint32_t)(N / r), total = (uint32_t)(B * h * T), hh = (uint32_t)h;
  const int lane = threadIdx.x & 31, sub = lane >> 3, ch = lane & 7;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 16; base < total; base += warps * 16) {
    uint4 x[4], y[4];
    int64_t out[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      // kept row, order (b, t', j): the h heads' 128-byte chunks of the same
      // token rows are read together (DRAM page locality)
      const uint32_t idx = base + 4 * u + sub;
      out[u] = -1;
      x[u] = y[u] = make_uint4(0, 0, 0, 0);
      if (idx < total) {
        const uint32_t bt = idx / hh, j = idx - bt * hh;
        const uint32_t b = bt / T, t = bt - b * T;
        const uint32_t n = t * (uint32_t)r + (uint32_t)p.offsets[j];
        const int64_t at = (((int64_t)b * N + n) * h + j) * 8 + ch;
        x[u] = o[at];
        y[u] = dout[at];
        out[u] = ((int64_t)b * h + j) * N + n;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t xa[4] = {x[u].x, x[u].y, x[u].z, x[u].w}, ya[4] = {y[u].x, y[u].y, y[u].z, y[u].w};
      float acc = 0.0f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc = fmaf(__uint_as_float(xa[e] << 16), __uint_as_float(ya[e] << 16), acc);
        acc = fmaf(__uint_as_float(xa[e] & 0xffff0000u), __uint_as_float(ya[e] & 0xffff0000u), acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      if (ch == 0 && out[u] >= 0) delta[out[u]] = acc;
    }
  }
}

template <typename T, int DMAX, int PARTS, int QT>
__global__ void __launch_bounds__(128) dkdv_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                   const T* __restrict__ v, const T* __restrict__ dout,
                                                   const float* __restrict__ lse, const float* __restrict__ delta,
                                                   T* __restrict__ dk, T* __restrict__ dv,
                                                   const __grid_constant__ BwdParams p) {
  constexpr int E = DMAX / PARTS;
  constexpr int ROWS = 128 / PARTS;
  __shared__ float qs[QT][DMAX];
  __shared__ float gs[QT][DMAX];
  __shared__ float ls[QT], ds[QT];

  const int tid = threadIdx.x;
  const int rr = tid / PARTS, pp = tid % PARTS;
  const int64_t seg = blockIdx.x / p.n_chunks, chunk = blockIdx.x % p.n_chunks;
  const int64_t j = blockIdx.y, b = blockIdx.z;
  const int64_t g = p.offsets[j];
  const SegView sv = seg_view(p, seg, g);
  const int64_t hd = p.h * p.d, hdv = p.h * p.dv;
  const T* qb = q + b * p.N * hd + j * p.d;
  const T* kb = k + b * p.N * hd + j * p.d;
  const T* vb = v + b * p.N * hdv + j * p.dv;
  const T* gb = dout + b * p.N * hdv + j * p.dv;
  const float* lb = lse + (b * p.h + j) * p.N;
  const float* db = delta + (b * p.h + j) * p.N;
  T* dkb = dk + b * p.N * hd + j * p.d;
  T* dvb = dv + b * p.N * hdv + j * p.dv;

  if (chunk == 0) {  // unselected rows of the segment: zero gradient
    for (int64_t l = tid; l < sv.rows; l += blockDim.x) {
      if (l >= g && (l - g) % p.r == 0) continue;
      const int64_t row = sv.begin + l;
      for (int64_t c = 0; c < p.d; ++c) dkb[row * hd + c] = cvt<T>(0.0f);
      for (int64_t c = 0; c < p.dv; ++c) dvb[row * hdv + c] = cvt<T>(0.0f);
    }
  }
  if (chunk * ROWS >= sv.m) return;
  const int64_t t = chunk * ROWS + rr;
  const bool active = t < sv.m;
  const int64_t krow = sv.begin + g + t * p.r;
  float kr[E], vr[E], ak[E], av[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int c = pp * E + e;
    kr[e] = (active && c < p.d) ? ld(kb + krow * hd + c) : 0.0f;
    vr[e] = (active && c < p.dv) ? ld(vb + krow * hdv + c) : 0.0f;
    ak[e] = av[e] = 0.0f;
  }
  for (int64_t i0 = 0; i0 < sv.m; i0 += QT) {
    __syncthreads();
    for (int e = tid; e < QT * DMAX; e += blockDim.x) {
      const int ii = e / DMAX, c = e % DMAX;
      const int64_t ti = i0 + ii;
      const int64_t qrow = sv.begin + g + ti * p.r;
      qs[ii][c] = (ti < sv.m && c < p.d) ? ld(qb + qrow * hd + c) : 0.0f;
      gs[ii][c] = (ti < sv.m && c < p.dv) ? ld(gb + qrow * hdv + c) : 0.0f;
    }
    if (tid < QT) {
      const int64_t ti = i0 + tid;
      const int64_t qrow = sv.begin + g + ti * p.r;
      ls[tid] = ti < sv.m ? lb[qrow] : INFINITY;  // P = 0 for padding rows
      ds[tid] = ti < sv.m ? db[qrow] : 0.0f;
    }
    __syncthreads();
#pragma unroll 1
    for (int ii = 0; ii < QT; ++ii) {
      float s = 0.0f, dp = 0.0f;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        s = fmaf(qs[ii][pp * E + e], kr[e], s);
        dp = fmaf(gs[ii][pp * E + e], vr[e], dp);
      }
      s = part_sum<PARTS>(s);
      dp = part_sum<PARTS>(dp);
      const float pij = __expf(s * p.scale - ls[ii]);
      const float dsc = pij * (dp - ds[ii]) * p.scale;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        av[e] = fmaf(pij, gs[ii][pp * E + e], av[e]);
        ak[e] = fmaf(dsc, qs[ii][pp * E + e], ak[e]);
      }
    }
  }
  if (active) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int c = pp * E + e;
      if (c < p.d) dkb[krow * hd + c] = cvt<T>(ak[e]);
      if (c < p.dv) dvb[krow * hdv + c] = cvt<T>(av[e]);
    }
  }
}

template <typename T, int DMAX, int PARTS, int KT>
__global__ void __launch_bounds__(128) dq_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                 const T* __restrict__ v, const T* __restrict__ dout,
                                                 const float* __restrict__ lse, const float* __restrict__ delta,
                                                 T* __restrict__ dq, const __grid_constant__ BwdParams p) {
  constexpr int E = DMAX / PARTS;
  constexpr int ROWS = 128 / PARTS;
  __shared__ float ks[KT][DMAX];
  __shared__ float vs[KT][DMAX];

  const int tid = threadIdx.x;
  const int rr = tid / PARTS, pp = tid % PARTS;
  const int64_t seg = blockIdx.x / p.n_chunks, chunk = blockIdx.x % p.n_chunks;
  const int64_t j = blockIdx.y, b = blockIdx.z;
  const int64_t g = p.offsets[j];
  const SegView sv = seg_view(p, seg, g);
  const int64_t hd = p.h * p.d, hdv = p.h * p.dv;
  const T* qb = q + b * p.N * hd + j * p.d;
  const T* kb = k + b * p.N * hd + j * p.d;
  const T* vb = v + b * p.N * hdv + j * p.dv;
  const T* gb = dout + b * p.N * hdv + j * p.dv;
  T* dqb = dq + b * p.N * hd + j * p.d;

  if (chunk == 0) {
    for (int64_t l = tid; l < sv.rows; l += blockDim.x) {
      if (l >= g && (l - g) % p.r == 0) continue;
      const int64_t row = sv.begin + l;
      for (int64_t c = 0; c < p.d; ++c) dqb[row * hd + c] = cvt<T>(0.0f);
    }
  }
  if (chunk * ROWS >= sv.m) return;
  const int64_t t = chunk * ROWS + rr;
  const bool active = t < sv.m;
  const int64_t qrow = sv.begin + g + t * p.r;
  float qr[E], gr[E], aq[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int c = pp * E + e;
    qr[e] = (active && c < p.d) ? ld(qb + qrow * hd + c) : 0.0f;
    gr[e] = (active && c < p.dv) ? ld(gb + qrow * hdv + c) : 0.0f;
    aq[e] = 0.0f;
  }
  const float li = active ? lse[(b * p.h + j) * p.N + qrow] : INFINITY;
  const float di = active ? delta[(b * p.h + j) * p.N + qrow] : 0.0f;
  for (int64_t k0 = 0; k0 < sv.m; k0 += KT) {
    __syncthreads();
    for (int e = tid; e < KT * DMAX; e += blockDim.x) {
      const int jj = e / DMAX, c = e % DMAX;
      const int64_t tk = k0 + jj;
      const int64_t krow = sv.begin + g + tk * p.r;
      ks[jj][c] = (tk < sv.m && c < p.d) ? ld(kb + krow * hd + c) : 0.0f;
      vs[jj][c] = (tk < sv.m && c < p.dv) ? ld(vb + krow * hdv + c) : 0.0f;
    }
    __syncthreads();
    const int kt = (int)(sv.m - k0 < KT ? sv.m - k0 : KT);
#pragma unroll 1
    for (int jj = 0; jj < kt; ++jj) {
      float s = 0.0f, dp = 0.0f;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        s = fmaf(qr[e], ks[jj][pp * E + e], s);
        dp = fmaf(gr[e], vs[jj][pp * E + e], dp);
      }
      s = part_sum<PARTS>(s);
      dp = part_sum<PARTS>(dp);
      const float pij = __expf(s * p.scale - li);
      const float dsc = pij * (dp - di) * p.scale;
#pragma unroll
      for (int e = 0; e < E; ++e) aq[e] = fmaf(dsc, ks[jj][pp * E + e], aq[e]);
    }
  }
  if (active) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int c = pp * E + e;
      if (c < p.d) dqb[qrow * hd + c] = cvt<T>(aq[e]);
    }
  }
}

template <typename T, int DMAX, int PARTS, int TILE>
int launch_bwd_t(const Geometry& g, const void* q, const void* k, const void* v, const void* o, const void* dout,
                 const float* lse, float* delta, void* dq, void* dk, void* dv, cudaStream_t stream, cudaError_t* err) {
  BwdParams p;
  p.N = g.N;
  p.w = g.w;
  p.r = g.r;
  p.h = g.h;
  p.d = g.d;
  p.dv = g.dv;
  constexpr int ROWS = 128 / PARTS;
  p.n_chunks = (g.m_max + ROWS - 1) / ROWS;
  if (p.n_chunks < 1) p.n_chunks = 1;
  p.scale = g.scale;
  for (int i = 0; i < kMaxHeads; ++i) p.offsets[i] = i < g.h ? g.offsets[i] : 0;
  const int64_t rows = g.B * g.N * g.h;
  delta_kernel<T><<<(unsigned)std::min<int64_t>((rows + 255) / 256, 148 * 32), 256, 0, stream>>>(
      (const T*)o, (const T*)dout, delta, rows, g.N, g.h, g.dv);
  dim3 grid((unsigned)(g.n_seg * p.n_chunks), (unsigned)g.h, (unsigned)g.B);
  dkdv_kernel<T, DMAX, PARTS, TILE><<<grid, 128, 0, stream>>>((const T*)q, (const T*)k, (const T*)v,
                                                               (const T*)dout, lse, delta, (T*)dk, (T*)dv, p);
  dq_kernel<T, DMAX, PARTS, TILE><<<grid, 128, 0, stream>>>((const T*)q, (const T*)k, (const T*)v, (const T*)dout,
                                                             lse, delta, (T*)dq, p);
  *err = cudaGetLastError();
  return 3;
}

template <typename T>
int launch_bwd_dtype(const Geometry& g, const void* q, const void* k, const void* v, const void* o, const void* dout,
                     const float* lse, float* delta, void* dq, void* dk, void* dv, cudaStream_t stream,
                     cudaError_t* err) {
  const int64_t dm = g.d > g.dv ? g.d : g.dv;
  if (dm <= 16) return launch_bwd_t<T, 16, 1, 32>(g, q, k, v, o, dout, lse, delta, dq, dk, dv, stream, err);
  if (dm <= 32) return launch_bwd_t<T, 32, 1, 32>(g, q, k, v, o, dout, lse, delta, dq, dk, dv, stream, err);
  if (dm <= 64) return launch_bwd_t<T, 64, 2, 32>(g, q, k, v, o, dout, lse, delta, dq, dk, dv, stream, err);
  if (dm <= 128) return launch_bwd_t<T, 128, 4, 16>(g, q, k, v, o, dout, lse, delta, dq, dk, dv, stream, err);
  return launch_bwd_t<T, 256, 8, 8>(g, q, k, v, o, dout, lse, delta, dq, dk, dv, stream, err);
}

}  // namespace

int launch_backward(const Geometry& g, int dtype, const void* q, const void* k, const void* v, const void* o,
                    const void* dout, const float* lse, float* delta, void* dq, void* dk, void* dv,
                    cudaStream_t stream, cudaError_t* err, bool allow_sm100, const char** why) {
  const void* ptrs[] = {q, k, v, dout, dq, dk, dv};
  if (allow_sm100 && bwd_sm100_supported(g, dtype, ptrs, 7)) {
    if ((reinterpret_cast<uintptr_t>(o) & 15u) == 0 && g.B * g.h * g.N < ((int64_t)1 << 31)) {
      BwdParams bp{};
      for (int j = 0; j < kMaxHeads; ++j) bp.offsets[j] = g.offsets[j];
      const int64_t kept = g.B * g.h * (g.N / g.r);
      delta_kept_kernel<<<(unsigned)std::min<int64_t>((kept + 127) / 128, 148 * 16), 256, 0, stream>>>(
          (const uint4*)o, (const uint4*)dout, delta, g.B, g.N, g.r, g.h, bp);
    } else {
      const int64_t rows = g.B * g.N * g.h;
      delta_kernel<__nv_bfloat16><<<(unsigned)std::min<int64_t>((rows + 255) / 256, 148 * 32), 256, 0, stream>>>(
          (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, delta, rows, g.N, g.h, g.dv);
    }
    const int n = launch_bwd_sm100(g, q, k, v, dout, lse, delta, dq, dk, dv, stream, err, why);
    return n ? n + 1 : 0;
  }
  if (dtype == 0) return launch_bwd_dtype<float>(g, q, k, v, o, dout, lse, delta, dq, dk, dv, stream, err);
  return launch_bwd_dtype<__nv_bfloat16>(g, q, k, v, o, dout, lse, delta, dq, dk, dv, stream, err);
}

}  // namespace dfa_impl
