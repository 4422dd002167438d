// LSE-weighted combine of several dilated-attention branches (north_star
// extension; the reference has a single (w, r) per config -- SPEC.md:204).
//
// Branch b produced O_b [B, N, h, d_v] (normalised, dtype) and lse_b [B, h, N]
// (natural log, -inf where the branch selects no row).  For every (image,
// row, head):  O = sum_b e^{lse_b} O_b / sum_b e^{lse_b}, computed with the
// max-subtracted weights; rows covered by no branch stay exactly 0 and get
// lse = -inf.  One thread per (b, n, j) row, 16-byte vector loads/stores;
// purely HBM-bound (K reads of O_b + lse, one write of O).
#include <cuda_bf16.h>
#include <math.h>

#include "dfa_internal.h"

namespace dfa_impl {
namespace {

struct CombineParams {
  int64_t rows;  // B * N * h
  int64_t N, h, dv;
  int32_t nb;
  const void* o[kMaxBranches];
  const float* lse[kMaxBranches];
};

template <typename T>
__device__ __forceinline__ float tof(T x);
template <>
__device__ __forceinline__ float tof<float>(float x) {
  return x;
}
template <>
__device__ __forceinline__ float tof<__nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}

template <typename T>
__global__ void __launch_bounds__(256) combine_kernel(const __grid_constant__ CombineParams p, T* __restrict__ out,
                                                      float* __restrict__ lse_out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // row index over [B, N, h]
  if (r >= p.rows) return;
  const int64_t j = r % p.h;
  const int64_t n = (r / p.h) % p.N;
  const int64_t b = r / (p.h * p.N);
  const int64_t li = (b * p.h + j) * p.N + n;  // lse index [B, h, N]
  float lv[kMaxBranches];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < kMaxBranches; ++k) {
    lv[k] = k < p.nb ? p.lse[k][li] : -INFINITY;
    m = fmaxf(m, lv[k]);
  }
  T* orow = out + r * p.dv;
  if (m == -INFINITY) {
    for (int64_t c = 0; c < p.dv; ++c) orow[c] = T(0.0f);
    if (lse_out) lse_out[li] = -INFINITY;
    return;
  }
  float wsum = 0.0f;
#pragma unroll
  for (int k = 0; k < kMaxBranches; ++k) {
    lv[k] = (k < p.nb && lv[k] != -INFINITY) ? __expf(lv[k] - m) : 0.0f;
    wsum += lv[k];
  }
  const float inv = 1.0f / wsum;
  for (int64_t c0 = 0; c0 < p.dv; c0 += 8) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < kMaxBranches; ++k) {
      if (k >= p.nb || lv[k] == 0.0f) continue;
      const T* src = reinterpret_cast<const T*>(p.o[k]) + r * p.dv + c0;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (c0 + e < p.dv) acc[e] = fmaf(lv[k], tof(src[e]), acc[e]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (c0 + e < p.dv) orow[c0 + e] = T(acc[e] * inv);
  }
  if (lse_out) lse_out[li] = m + logf(wsum);
}

}  // namespace

int launch_combine(int dtype, int64_t B, int64_t N, int64_t h, int64_t dv, int nb, const void* const* o,
                   const float* const* lse, void* out, float* lse_out, cudaStream_t stream, cudaError_t* err) {
  CombineParams p;
  p.rows = B * N * h;
  p.N = N;
  p.h = h;
  p.dv = dv;
  p.nb = nb;
  for (int k = 0; k < kMaxBranches; ++k) {
    p.o[k] = k < nb ? o[k] : nullptr;
    p.lse[k] = k < nb ? lse[k] : nullptr;
  }
  const unsigned grid = (unsigned)((p.rows + 255) / 256);
  if (dtype == 0)
    combine_kernel<float><<<grid, 256, 0, stream>>>(p, (float*)out, lse_out);
  else
    combine_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(p, (__nv_bfloat16*)out, lse_out);
  *err = cudaGetLastError();
  return 1;
}

}  // namespace dfa_impl
