// Callers either side of the hot path:
//   * multi_head_dilated (attention.hpp:340-360): per-head Q/K/V projections
//     -> dilated core per head -> concat -> output projection;
//   * one pre-norm encoder block (encoder.hpp:241-248): LN1 -> attention_mix
//     (+ bo) -> residual -> LN2 -> W1 + b1 -> GELU(erf) -> W2 + b2 -> residual.
//
// B200 layout: activations stay in the core's [B, N, h, d] = [B*N, D] layout
// end to end, so the projections write exactly what the TMA boxes of the
// attention kernel read and the concat of the heads IS the attention output
// -- no gather, scatter or transpose pass exists.  The GEMMs are this
// library's own tcgen05 kernel (dfa_gemm.cu: bias, residual and the erf GELU
// in its epilogue); this file holds LayerNorm, a standalone erf-GELU and the
// weight-packing kernels.
#include <cuda_bf16.h>
#include <math.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "dfa_internal.h"
#include "sm100_ptx.cuh"

namespace dfa_impl {
namespace {

template <typename T>
__device__ __forceinline__ float ldf(const T* p);
template <>
__device__ __forceinline__ float ldf<float>(const float* p) {
  return *p;
}
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ T stf(float x);
template <>
__device__ __forceinline__ float stf<float>(float x) {
  return x;
}
template <>
__device__ __forceinline__ __nv_bfloat16 stf<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// 16-byte vectors of 8 bf16 / 4 f32 values.
template <typename T>
struct Vec {
  static constexpr int kN = 16 / sizeof(T);
  uint4 raw;
  __device__ __forceinline__ float get(int e) const { return ldf(reinterpret_cast<const T*>(&raw) + e); }
  __device__ __forceinline__ void set(int e, float x) { reinterpret_cast<T*>(&raw)[e] = stf<T>(x); }
};

// tensor.hpp:281-300 / autodiff.hpp:191-243 layer_norm: population variance,
// eps 1e-5, y = (x - mean) / sqrt(var + eps) * g + b.  One warp per row; lane
// l holds 16-byte vectors l, l + 32, ... of the row in registers (D <= 1024 for
// bf16), two-pass mean / variance in fp32 with warp shuffles, 16-byte stores.
// Requires D % (16 / sizeof(T)) == 0 and 16-byte aligned rows (checked by the
// launcher, which falls back to the scalar form otherwise).
template <typename T, int kMaxVec>
__global__ void __launch_bounds__(256) layer_norm_vec_kernel(const T* __restrict__ x, const T* __restrict__ g,
                                                             const T* __restrict__ b, T* __restrict__ y,
                                                             int64_t rows, int cols) {
  constexpr int V = Vec<T>::kN;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int nv = cols / V;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
  Vec<T> v[kMaxVec];
  float sum = 0.0f;
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i) {
    const int vi = lane + 32 * i;
    v[i].raw = vi < nv ? xr[vi] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int e = 0; e < V; ++e) sum += v[i].get(e);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / (float)cols;
  float var = 0.0f;
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i)
    if (lane + 32 * i < nv)
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const float d = v[i].get(e) - mean;
        var = fmaf(d, d, var);
      }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
  const float inv = 1.0f / sqrtf(var / (float)cols + 1e-5f);
  uint4* yr = reinterpret_cast<uint4*>(y + row * cols);
  const uint4* gv = reinterpret_cast<const uint4*>(g);
  const uint4* bv = reinterpret_cast<const uint4*>(b);
#pragma unroll
  for (int i = 0; i < kMaxVec; ++i) {
    const int vi = lane + 32 * i;
    if (vi >= nv) continue;
    Vec<T> gg, bb, out;
    gg.raw = gv[vi];
    bb.raw = bv[vi];
#pragma unroll
    for (int e = 0; e < V; ++e) out.set(e, (v[i].get(e) - mean) * inv * gg.get(e) + bb.get(e));
    yr[vi] = out.raw;
  }
}

// bf16 production form of layer_norm_vec_kernel: the same two-pass fp32
// statistics with rows kept as packed float pairs (FADD2 / FFMA2 / FMUL2) and
// bf16 unpacked by shifts (~6 instructions per element instead of the
// generic form's ~33 on per-element bf16 insert / extract).  Each warp owns
// kRows consecutive rows and issues all their 16-byte loads before any math,
// so kRows x D x 2 bytes per warp are in flight (one row per warp left the
// pass latency-bound at ~2.8 TB/s).  kVec = 16-byte vectors per lane.
template <int kVec, int kRows>
__global__ void __launch_bounds__(256) layer_norm_bf16_kernel(const __nv_bfloat16* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ g,
                                                              const __nv_bfloat16* __restrict__ b,
                                                              __nv_bfloat16* __restrict__ y, int64_t rows, int cols) {
  const int lane = threadIdx.x & 31;
  const int64_t row0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kRows;
  if (row0 >= rows) return;
  const int nv = cols / 8;
  const float rc = 1.0f / (float)cols;
  uint4 raw[kRows][kVec];
#pragma unroll
  for (int rr = 0; rr < kRows; ++rr) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + (row0 + rr) * cols);
#pragma unroll
    for (int i = 0; i < kVec; ++i) {
      const int vi = lane + 32 * i;
      raw[rr][i] = (vi < nv && row0 + rr < rows) ? xr[vi] : make_uint4(0, 0, 0, 0);
    }
  }
  uint4 graw[kVec], braw[kVec];
#pragma unroll
  for (int i = 0; i < kVec; ++i) {
    const int vi = lane + 32 * i;
    graw[i] = vi < nv ? reinterpret_cast<const uint4*>(g)[vi] : make_uint4(0, 0, 0, 0);
    braw[i] = vi < nv ? reinterpret_cast<const uint4*>(b)[vi] : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int rr = 0; rr < kRows; ++rr) {
    if (row0 + rr >= rows) break;
    float2 v[kVec][4];
    float2 s2 = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < kVec; ++i) {
      const uint32_t w[4] = {raw[rr][i].x, raw[rr][i].y, raw[rr][i].z, raw[rr][i].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[i][e] = ptx::bf16x2_to_float2(w[e]);
        s2 = ptx::fadd2(s2, v[i][e]);
      }
    }
    float sum = s2.x + s2.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float mean = sum * rc;
    const float2 nm = make_float2(-mean, -mean);
    float2 q2 = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < kVec; ++i) {
      if (lane + 32 * i >= nv) continue;  // padded lanes hold zeros, not x - mean
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[i][e] = ptx::fadd2(v[i][e], nm);
        q2 = ptx::ffma2(v[i][e], v[i][e], q2);
      }
    }
    float var = q2.x + q2.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
    const float inv = 1.0f / sqrtf(var * rc + 1e-5f);
    const float2 inv2 = make_float2(inv, inv);
    uint4* yr = reinterpret_cast<uint4*>(y + (row0 + rr) * cols);
#pragma unroll
    for (int i = 0; i < kVec; ++i) {
      const int vi = lane + 32 * i;
      if (vi >= nv) continue;
      const uint32_t gw[4] = {graw[i].x, graw[i].y, graw[i].z, graw[i].w};
      const uint32_t bw[4] = {braw[i].x, braw[i].y, braw[i].z, braw[i].w};
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 t =
            ptx::ffma2(ptx::fmul2(v[i][e], inv2), ptx::bf16x2_to_float2(gw[e]), ptx::bf16x2_to_float2(bw[e]));
        o[e] = ptx::pack_bf16x2(t.x, t.y);
      }
      yr[vi] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// Scalar fallback (any D <= 1024, any alignment).
template <typename T>
__global__ void __launch_bounds__(256) layer_norm_kernel(const T* __restrict__ x, const T* __restrict__ g,
                                                         const T* __restrict__ b, T* __restrict__ y, int64_t rows,
                                                         int cols) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const T* xr = x + row * cols;
  float v[32];
  float sum = 0.0f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int c = lane + 32 * i;
    v[i] = c < cols ? ldf(xr + c) : 0.0f;
    sum += v[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / (float)cols;
  float var = 0.0f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int c = lane + 32 * i;
    const float d = c < cols ? v[i] - mean : 0.0f;
    var = fmaf(d, d, var);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
  const float inv = 1.0f / sqrtf(var / (float)cols + 1e-5f);
  T* yr = y + row * cols;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int c = lane + 32 * i;
    if (c < cols) yr[c] = stf<T>((v[i] - mean) * inv * ldf(g + c) + ldf(b + c));
  }
}

// erf(x) to ~1e-7 absolute (Abramowitz & Stegun 7.1.26 refined: a rational
// polynomial in t = 1/(1 + p|x|) times exp(-x^2) on MUFU), ~3x cheaper than
// the correctly-rounded erff; the GELU below stays within 1e-7 * |x| of the
// erf form the reference uses (tensor.hpp:262-265).
__device__ __forceinline__ float erf_fast(float x) {
  const float ax = fabsf(x);
  const float t = __frcp_rn(fmaf(0.3275911f, ax, 1.0f));
  float y = fmaf(1.061405429f, t, -1.453152027f);
  y = fmaf(y, t, 1.421413741f);
  y = fmaf(y, t, -0.284496736f);
  y = fmaf(y, t, 0.254829592f);
  y *= t;
  const float r = fmaf(-y, __expf(-ax * ax), 1.0f);
  return copysignf(r, x);
}

// tensor.hpp:262-265 gelu_scalar: x * 0.5 * (1 + erf(x / sqrt(2))), in place,
// 16-byte vectors (n % V == 0 and 16-byte alignment; scalar tail otherwise).
template <typename T>
__global__ void __launch_bounds__(256) gelu_kernel(const T* __restrict__ xin, T* __restrict__ x, int64_t n, bool vec) {
  constexpr int V = Vec<T>::kN;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const uint4* xi = reinterpret_cast<const uint4*>(xin);
    uint4* xv = reinterpret_cast<uint4*>(x);
    const int64_t nv = n / V;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
      Vec<T> a;
      a.raw = xi[i];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const float t = a.get(e);
        a.set(e, t * 0.5f * (1.0f + erf_fast(t * 0.70710678118654752f)));
      }
      xv[i] = a.raw;
    }
    done = nv * V;
  }
  for (int64_t i = done + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = ldf(xin + i);
    x[i] = stf<T>(v * 0.5f * (1.0f + erff(v * 0.70710678118654752f)));
  }
}

// bf16 production GELU: x * Phi(x) with Phi(x) = (1 + tanh(x (a + b x^2))) / 2,
// a, b refitted to the erf form (max |error| 2.7e-4 over all x, plus
// tanh.approx's 2^-11 relative) -- below bf16's resolution of the result, on
// one MUFU.TANH and ~4 packed ops per element instead of erf's two MUFU ops
// and ~30 scalar ones.  The fp32 validation mode keeps erf_fast.
__global__ void __launch_bounds__(256) gelu_bf16_kernel(const uint4* __restrict__ xin, uint4* __restrict__ x,
                                                        int64_t nv) {
  const float2 a2 = make_float2(0.80015708f, 0.80015708f), b2 = make_float2(0.03470089f, 0.03470089f);
  const float2 h2 = make_float2(0.5f, 0.5f);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
    const uint4 r = xin[i];
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 v = ptx::bf16x2_to_float2(w[e]);
      const float2 u = ptx::fmul2(v, ptx::ffma2(ptx::fmul2(v, v), b2, a2));
      const float2 hv = ptx::fmul2(v, h2);
      const float2 t = ptx::ffma2(hv, make_float2(ptx::tanh_approx(u.x), ptx::tanh_approx(u.y)), hv);
      o[e] = ptx::pack_bf16x2(t.x, t.y);
    }
    x[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// wq/wk/wv [h, D, d] -> [D, 3, h, d]: column block (which, j) of the fused
// QKV projection is head j's D x d matrix of q / k / v.
template <typename T>
__global__ void __launch_bounds__(256) pack_qkv_kernel(const T* __restrict__ wq, const T* __restrict__ wk,
                                                       const T* __restrict__ wv, T* __restrict__ out, int64_t h,
                                                       int64_t D, int64_t d) {
  // 32-bit index decode (weights are far below 2^31 elements; int64 division
  // made this tiny pass take ~13 us)
  const uint32_t ud = (uint32_t)d, uh = (uint32_t)h, uD = (uint32_t)D;
  const uint32_t n = 3u * uD * uh * ud;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t i1 = i / ud, e = i - i1 * ud;
    const uint32_t i2 = i1 / uh, j = i1 - i2 * uh;
    const uint32_t c = i2 / 3u, which = i2 - c * 3u;
    const T* src = which == 0 ? wq : (which == 1 ? wk : wv);
    out[i] = src[((size_t)j * uD + c) * ud + e];
  }
}

// Offset-class packing (multi-head layers with r > 1, see class_split in
// dfa_api.cpp): heads grouped by gamma_j, class-major.  pos[j] = head j's
// position in that order, cls[j] its class, start[g] / cnt[g] the classes'
// first position / size.
struct ClassPack {
  int32_t pos[kMaxHeads], cls[kMaxHeads], start[kMaxHeads], cnt[kMaxHeads];
};

// wq/wk/wv [h, D, d] -> [D, 3 D] with class g's columns [3 d start_g, 3 d (start_g + cnt_g))
// laid out [3][cnt_g][d]: one GEMM per class writes that class's q | k | v.
template <typename T>
__global__ void __launch_bounds__(256) pack_qkv_class_kernel(const T* __restrict__ wq, const T* __restrict__ wk,
                                                             const T* __restrict__ wv, T* __restrict__ out,
                                                             uint32_t h, uint32_t D, uint32_t d,
                                                             const __grid_constant__ ClassPack cp) {
  const uint32_t n = 3u * D * h * d;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    // source order (c, which, j, e) -- i = ((c * 3 + which) * h + j) * d + e
    const uint32_t i1 = i / d, e = i - i1 * d;
    const uint32_t i2 = i1 / h, j = i1 - i2 * h;
    const uint32_t c = i2 / 3u, which = i2 - c * 3u;
    const T* src = which == 0 ? wq : (which == 1 ? wk : wv);
    const uint32_t g = (uint32_t)cp.cls[j], jr = (uint32_t)(cp.pos[j] - cp.start[g]);
    const uint32_t col = 3u * d * (uint32_t)cp.start[g] + (which * (uint32_t)cp.cnt[g] + jr) * d + e;
    out[(size_t)c * 3u * D + col] = src[((size_t)j * D + c) * d + e];
  }
}

// wo [h d, D] -> rows in class-major head order (row pos_j d + e <- j d + e).
template <typename T>
__global__ void __launch_bounds__(256) pack_wo_class_kernel(const T* __restrict__ wo, T* __restrict__ out,
                                                            uint32_t h, uint32_t D, uint32_t d,
                                                            const __grid_constant__ ClassPack cp) {
  const uint32_t n = h * d * D;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t r = i / D, c = i - r * D;
    const uint32_t j = r / d, e = r - j * d;
    out[((size_t)cp.pos[j] * d + e) * D + c] = wo[i];
  }
}

// Both class packings in one launch, 16-byte vectors (d % V == 0, D % V ==
// 0, aligned pointers): the per-call weight packing of the class-split layer
// was two scalar kernels of ~5 us each (integer divides per element).
template <typename T>
__global__ void __launch_bounds__(256) pack_class_vec_kernel(const T* __restrict__ wq, const T* __restrict__ wk,
                                                             const T* __restrict__ wv, const T* __restrict__ wo,
                                                             T* __restrict__ qkv_out, T* __restrict__ wo_out,
                                                             uint32_t h, uint32_t D, uint32_t d,
                                                             const __grid_constant__ ClassPack cp) {
  constexpr uint32_t V = 16 / sizeof(T);
  const uint32_t dv = d / V, Dv = D / V;
  const uint32_t n1 = 3u * D * h * dv, n2 = h * d * Dv;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n1 + n2; i += gridDim.x * blockDim.x) {
    if (i < n1) {
      // (c, which, j, e / V) -> the packed [D, class-major q|k|v] column block
      const uint32_t i1 = i / dv, e = (i - i1 * dv) * V;
      const uint32_t i2 = i1 / h, j = i1 - i2 * h;
      const uint32_t c = i2 / 3u, which = i2 - c * 3u;
      const T* src = which == 0 ? wq : (which == 1 ? wk : wv);
      const uint32_t g = (uint32_t)cp.cls[j], jr = (uint32_t)(cp.pos[j] - cp.start[g]);
      const uint32_t col = 3u * d * (uint32_t)cp.start[g] + (which * (uint32_t)cp.cnt[g] + jr) * d + e;
      *reinterpret_cast<uint4*>(qkv_out + (size_t)c * 3u * D + col) =
          *reinterpret_cast<const uint4*>(src + ((size_t)j * D + c) * d + e);
    } else {
      const uint32_t k = i - n1, r = k / Dv, cv = (k - r * Dv) * V;
      const uint32_t j = r / d, e = r - j * d;
      *reinterpret_cast<uint4*>(wo_out + ((size_t)cp.pos[j] * d + e) * D + cv) =
          *reinterpret_cast<const uint4*>(wo + (size_t)r * D + cv);
    }
  }
}

}  // namespace

int launch_layer_norm(int dtype, const void* x, const void* g, const void* b, void* y, int64_t rows, int cols,
                      cudaStream_t stream) {
  const unsigned grid = (unsigned)((rows * 32 + 255) / 256);
  const unsigned grid_vec = (unsigned)((rows + 7) / 8);  // one row per warp (looping rows per warp measured slower)
  const bool al = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(b) |
                    reinterpret_cast<uintptr_t>(y)) & 15u) == 0;
  if (dtype == 0) {
    if (al && cols % 4 == 0 && cols <= 4 * 32 * 8)
      layer_norm_vec_kernel<float, 8><<<grid_vec, 256, 0, stream>>>((const float*)x, (const float*)g, (const float*)b,
                                                               (float*)y, rows, cols);
    else
      layer_norm_kernel<float><<<grid, 256, 0, stream>>>((const float*)x, (const float*)g, (const float*)b,
                                                         (float*)y, rows, cols);
  } else {
    using B = __nv_bfloat16;
    const unsigned grid_r = (unsigned)((rows + 31) / 32);  // 8 warps x 4 rows per block
    if (al && cols % 8 == 0 && cols <= 8 * 32 * 2)
      layer_norm_bf16_kernel<2, 4><<<grid_r, 256, 0, stream>>>((const B*)x, (const B*)g, (const B*)b, (B*)y, rows,
                                                              cols);
    else if (al && cols % 8 == 0 && cols <= 8 * 32 * 4)
      layer_norm_bf16_kernel<4, 2><<<(unsigned)((rows + 15) / 16), 256, 0, stream>>>((const B*)x, (const B*)g,
                                                                                      (const B*)b, (B*)y, rows, cols);
    else
      layer_norm_kernel<B><<<grid, 256, 0, stream>>>((const B*)x, (const B*)g, (const B*)b, (B*)y, rows, cols);
  }
  return 1;
}

int launch_pack_qkv(int dtype, const void* wq, const void* wk, const void* wv, void* out, int64_t h, int64_t D,
                    int64_t d, cudaStream_t stream) {
  const unsigned grid = (unsigned)std::min<int64_t>((3 * D * h * d + 255) / 256, 148 * 8);
  if (dtype == 0)
    pack_qkv_kernel<float><<<grid, 256, 0, stream>>>((const float*)wq, (const float*)wk, (const float*)wv,
                                                     (float*)out, h, D, d);
  else
    pack_qkv_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>((const __nv_bfloat16*)wq, (const __nv_bfloat16*)wk,
                                                             (const __nv_bfloat16*)wv, (__nv_bfloat16*)out, h, D, d);
  return 1;
}

int launch_pack_class(int dtype, const void* wq, const void* wk, const void* wv, const void* wo, void* qkv_out,
                      void* wo_out, int64_t h, int64_t D, int64_t d, const int32_t* offsets, cudaStream_t stream) {
  ClassPack cp{};
  int32_t r_max = 0;
  for (int j = 0; j < h; ++j) r_max = std::max(r_max, offsets[j] + 1);
  int32_t at = 0;
  for (int32_t g = 0; g < r_max; ++g) {
    cp.start[g] = at;
    for (int j = 0; j < h; ++j)
      if (offsets[j] == g) {
        cp.pos[j] = at++;
        cp.cls[j] = g;
      }
    cp.cnt[g] = at - cp.start[g];
  }
  const unsigned grid = (unsigned)std::min<int64_t>((3 * D * D + 255) / 256, 148 * 8);
  const int64_t V = dtype == 0 ? 4 : 8;
  const bool vec = d % V == 0 && D % V == 0 &&
                   ((reinterpret_cast<uintptr_t>(wq) | reinterpret_cast<uintptr_t>(wk) | reinterpret_cast<uintptr_t>(wv) |
                     reinterpret_cast<uintptr_t>(wo) | reinterpret_cast<uintptr_t>(qkv_out) |
                     reinterpret_cast<uintptr_t>(wo_out)) & 15u) == 0;
  if (vec) {
    const unsigned gv = (unsigned)std::min<int64_t>((4 * D * h * d / V + 255) / 256, 148 * 8);
    if (dtype == 0)
      pack_class_vec_kernel<float><<<gv, 256, 0, stream>>>((const float*)wq, (const float*)wk, (const float*)wv,
                                                          (const float*)wo, (float*)qkv_out, (float*)wo_out,
                                                          (uint32_t)h, (uint32_t)D, (uint32_t)d, cp);
    else
      pack_class_vec_kernel<__nv_bfloat16><<<gv, 256, 0, stream>>>(
          (const __nv_bfloat16*)wq, (const __nv_bfloat16*)wk, (const __nv_bfloat16*)wv, (const __nv_bfloat16*)wo,
          (__nv_bfloat16*)qkv_out, (__nv_bfloat16*)wo_out, (uint32_t)h, (uint32_t)D, (uint32_t)d, cp);
    return 1;
  }
  if (dtype == 0) {
    pack_qkv_class_kernel<float><<<grid, 256, 0, stream>>>((const float*)wq, (const float*)wk, (const float*)wv,
                                                           (float*)qkv_out, (uint32_t)h, (uint32_t)D, (uint32_t)d, cp);
    pack_wo_class_kernel<float><<<grid, 256, 0, stream>>>((const float*)wo, (float*)wo_out, (uint32_t)h, (uint32_t)D,
                                                          (uint32_t)d, cp);
  } else {
    using B = __nv_bfloat16;
    pack_qkv_class_kernel<B><<<grid, 256, 0, stream>>>((const B*)wq, (const B*)wk, (const B*)wv, (B*)qkv_out,
                                                       (uint32_t)h, (uint32_t)D, (uint32_t)d, cp);
    pack_wo_class_kernel<B><<<grid, 256, 0, stream>>>((const B*)wo, (B*)wo_out, (uint32_t)h, (uint32_t)D,
                                                      (uint32_t)d, cp);
  }
  return 2;
}

int launch_gelu(int dtype, const void* xin, void* x, int64_t n, cudaStream_t stream) {
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(xin)) & 15u) == 0;
  const int64_t per = dtype == 0 ? 4 : 8;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n / per + 255) / 256, 148 * 64));
  if (dtype == 0)
    gelu_kernel<float><<<grid, 256, 0, stream>>>((const float*)xin, (float*)x, n, vec);
  else if (vec && n % 8 == 0)
    gelu_bf16_kernel<<<grid, 256, 0, stream>>>((const uint4*)xin, (uint4*)x, n / 8);
  else
    gelu_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>((const __nv_bfloat16*)xin, (__nv_bfloat16*)x, n, vec);
  return 1;
}

}  // namespace dfa_impl
