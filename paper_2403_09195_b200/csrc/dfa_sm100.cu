// Dilated Flash Attention forward for sm_100a: TMA + tcgen05 + TMEM.
//
// Reference path: attnkit::dilated_attention (attention.hpp:280-301):
// per segment i and head offset gamma, gather rows i*w+gamma+t*r
// (make_segment_view :84-98, sparsify_segment :210-222), softmax attention
// among them (naive_attention :119-127 / tiled_attention :147-207), scatter
// back into a zero-initialised [N, d] (recompose :246-274).
//
// B200 restatement.  With N % r == 0 the [B, N, h, d] bf16 tensor IS the
// contiguous 4-D tensor [B*N/r][r][h][d]; row n of image b sits at
// (t' = (b*N+n)/r, gamma' = n % r).  For head j the view rows of ALL segments
// are the t'-stream at gamma' = gamma_j, and segment i is the contiguous block
// t' in [i*m, i*m+m) (m = w/r when r | w; the tail segment is shorter).  So the
// segment + strided gather of the reference is a plain TMA box
// (d=64, h=1, gamma'=1, t'=128) at coordinates (0, j, gamma_j, t'0): no index
// arrays, no gather kernel.  Attention is block-diagonal in t'-space.
//
// One CTA = one 128-row query tile of one (b, j) t'-stream.  Key tiles of 128
// t'-rows cover the union of the segments the query tile touches; keys outside
// a query's own segment are masked (only needed when m is not a multiple of
// 128 or at the tail).  Per key tile:
//   S = Q K^T       tcgen05.mma M=128 N=128 K=64, fp32 accumulator in TMEM
//   softmax         4 warps, thread = query row = TMEM lane; tcgen05.ld of the
//                   row, exp2 with the 1/sqrt(d)*log2(e) fold, running max with
//                   a lazy (threshold 2^8) rescale of O, P packed to bf16 and
//                   written back into TMEM over the consumed S columns
//   O += P V        tcgen05.mma with A = P from TMEM, B = V (MN-major) in smem
// Epilogue: O / l, bf16, stored at rows t'*r + gamma_j; the same threads write
// the rows of the other r-1 offset classes as exact zeros, so the output
// needs no memset and every byte of o is written exactly once.
//
// Warp roles (160 threads): warps 0-3 softmax + epilogue (TMEM lanes 0-127),
// warp 4 = producer: one elected lane issues all TMA loads and MMAs.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>

#include <mutex>

#include "dfa_internal.h"
#include "sm100_ptx.cuh"

namespace dfa_impl {
namespace {

constexpr int kD = 64;                // head_dim handled by this kernel
constexpr int kBM = 128;              // query rows per CTA (MMA M)
constexpr int kBN = 128;              // keys per tile (MMA N of Q K^T, K of P V)
constexpr int kTileBytes = 128 * 128; // 128 rows x 128 B (64 bf16), SW128
constexpr int kStages = 2;            // K/V ring depth
constexpr int kThreads = 160;
constexpr uint32_t kTmemCols = 256;   // S/P at [0,128), O at [128,192)
constexpr uint32_t kColS = 0, kColO = 128;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: p <= 2^8 before a rescale

struct __align__(1024) SmemLayout {
  uint8_t q[kTileBytes];
  uint8_t k[kStages][kTileBytes];
  uint8_t v[kStages][kTileBytes];
  uint64_t bar_q;
  uint64_t bar_full[kStages];
  uint64_t bar_empty[kStages];
  uint64_t bar_s;
  uint64_t bar_p;
  uint64_t bar_o;
  uint32_t tmem_base;
};

struct Sm100Params {
  int64_t N, T;        // T = N / r (t'-stream length per (b, j))
  int64_t m;           // t'-rows per full segment (w / r)
  int32_t r, h, n_qt;  // n_qt = ceil(T / 128)
  float c;             // scale * log2(e)
  float scale;
  int32_t offsets[kMaxHeads];
};

__device__ __forceinline__ uint32_t tmem_addr(uint32_t base, uint32_t lane, uint32_t col) {
  return base + (lane << 16) + col;
}

__global__ void __launch_bounds__(kThreads, 1)
    dfa_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, __nv_bfloat16* __restrict__ o,
                     float* __restrict__ lse, const __grid_constant__ Sm100Params p) {
  extern __shared__ uint8_t smem_raw[];
  SmemLayout& sm = *reinterpret_cast<SmemLayout*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();

  // Work item: query tile qt of stream (b, j).
  const int64_t idx = blockIdx.x;
  const int32_t qt = (int32_t)(idx % p.n_qt);
  const int64_t bj = idx / p.n_qt;
  const int32_t j = (int32_t)(bj % p.h);
  const int64_t b = bj / p.h;
  const int32_t gamma = p.offsets[j];
  const int64_t t0 = (int64_t)qt * kBM;                 // first query t' (stream-local)
  const int64_t t_last = min(t0 + kBM, p.T) - 1;        // last valid query t'
  const int64_t kv_lo = (t0 / p.m) * p.m;               // first key t' (segment start)
  const int64_t kv_hi = min((t_last / p.m + 1) * p.m, p.T);
  const int32_t n_kv = (int32_t)((kv_hi - kv_lo + kBN - 1) / kBN);
  const int64_t row0 = b * p.T;                          // stream origin in global t'

  if (warp == 4) {
    if (lane == 0) {
      ptx::mbar_init(&sm.bar_q, 1);
      for (int s = 0; s < kStages; ++s) {
        ptx::mbar_init(&sm.bar_full[s], 1);
        ptx::mbar_init(&sm.bar_empty[s], 1);
      }
      ptx::mbar_init(&sm.bar_s, 1);
      ptx::mbar_init(&sm.bar_p, kBM);
      ptx::mbar_init(&sm.bar_o, 1);
      ptx::fence_barrier_init();
      ptx::tma_prefetch_desc(&tm_q);
      ptx::tma_prefetch_desc(&tm_k);
      ptx::tma_prefetch_desc(&tm_v);
    }
  } else if (warp == 0) {
    ptx::tmem_alloc<kTmemCols>(&sm.tmem_base);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp == 4) {
    // ------------------------------------------------------------ producer
    if (ptx::elect_one()) {
      const uint64_t pol_q = ptx::policy_evict_first();
      const uint64_t pol_kv = ptx::policy_evict_last();
      ptx::mbar_arrive_expect_tx(&sm.bar_q, kTileBytes);
      ptx::tma_load_4d(sm.q, &tm_q, &sm.bar_q, 0, j, gamma, (int32_t)(row0 + t0), pol_q);
      for (int kt = 0; kt < n_kv && kt < kStages; ++kt) {
        const int32_t kr = (int32_t)(row0 + kv_lo + (int64_t)kt * kBN);
        ptx::mbar_arrive_expect_tx(&sm.bar_full[kt], 2 * kTileBytes);
        ptx::tma_load_4d(sm.k[kt], &tm_k, &sm.bar_full[kt], 0, j, gamma, kr, pol_kv);
        ptx::tma_load_4d(sm.v[kt], &tm_v, &sm.bar_full[kt], 0, j, gamma, kr, pol_kv);
      }
      constexpr uint32_t idesc_qk = ptx::idesc_bf16(kBM, kBN, 0, 0);  // K-major A and B
      constexpr uint32_t idesc_pv = ptx::idesc_bf16(kBM, kD, 0, 1);   // A (TMEM) K-major, V MN-major
      const uint32_t q_addr = ptx::smem_u32(sm.q);
      auto issue_qk = [&](int kt) {
        const int s = kt % kStages;
        ptx::mbar_wait(&sm.bar_full[s], (kt / kStages) & 1);
        ptx::tc_fence_after();
        const uint32_t k_addr = ptx::smem_u32(sm.k[s]);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          ptx::mma_ss(tbase + kColS, ptx::sdesc_sw128(q_addr + kk * 32), ptx::sdesc_sw128(k_addr + kk * 32),
                      idesc_qk, kk > 0);
        }
        ptx::tc_commit(&sm.bar_s);
      };
      ptx::mbar_wait(&sm.bar_q, 0);
      issue_qk(0);
      for (int kt = 0; kt < n_kv; ++kt) {
        const int s = kt % kStages;
        ptx::mbar_wait(&sm.bar_p, kt & 1);  // softmax wrote P_kt (and rescaled O)
        ptx::tc_fence_after();
        const uint32_t v_addr = ptx::smem_u32(sm.v[s]);
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          ptx::mma_ts(tbase + kColO, tbase + kColS + kk * 8, ptx::sdesc_sw128(v_addr + kk * 2048), idesc_pv,
                      (kt > 0 || kk > 0) ? 1u : 0u);
        }
        ptx::tc_commit(&sm.bar_empty[s]);
        if (kt + 1 < n_kv) issue_qk(kt + 1);  // in-order after PV_kt: safe to overwrite P_kt
        if (kt + kStages < n_kv) {
          ptx::mbar_wait(&sm.bar_empty[s], (kt / kStages) & 1);
          const int32_t kr = (int32_t)(row0 + kv_lo + (int64_t)(kt + kStages) * kBN);
          ptx::mbar_arrive_expect_tx(&sm.bar_full[s], 2 * kTileBytes);
          ptx::tma_load_4d(sm.k[s], &tm_k, &sm.bar_full[s], 0, j, gamma, kr, pol_kv);
          ptx::tma_load_4d(sm.v[s], &tm_v, &sm.bar_full[s], 0, j, gamma, kr, pol_kv);
        }
      }
      ptx::tc_commit(&sm.bar_o);
    }
  } else {
    // ----------------------------------------------- softmax + epilogue
    const uint32_t row = warp * 32 + lane;  // query row in tile == TMEM lane
    const int64_t tq = t0 + row;            // stream-local t'
    const bool valid_q = tq < p.T;
    const int64_t hd = (int64_t)p.h * kD;
    __nv_bfloat16* const ob = o + (b * p.N) * hd + (int64_t)j * kD;

    // Zero rows of the other offset classes while the first tiles load.
    if (valid_q) {
      for (int32_t gz = 0; gz < p.r; ++gz) {
        if (gz == gamma) continue;
        uint8_t* dst = reinterpret_cast<uint8_t*>(ob + (tq * p.r + gz) * hd);
#pragma unroll
        for (int c = 0; c < 8; ++c) ptx::st_global_v4(dst + 16 * c, 0u, 0u, 0u, 0u);
        if (lse) lse[(b * p.h + j) * p.N + tq * p.r + gz] = -INFINITY;
      }
    }

    // The query's own segment, as a key range in t'.
    const int64_t seg_lo = valid_q ? (tq / p.m) * p.m : 0;
    const int64_t seg_hi = valid_q ? min(seg_lo + p.m, p.T) : 0;
    const uint32_t lane_base = (warp * 32) << 16;
    float mref = -INFINITY;  // running reference max (raw score units)
    float l = 0.0f;
    for (int kt = 0; kt < n_kv; ++kt) {
      ptx::mbar_wait(&sm.bar_s, kt & 1);
      ptx::tc_fence_after();
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tbase + lane_base + kColS + 32 * c, sr[c]);
      ptx::tmem_ld_wait();
      const int64_t k0 = kv_lo + (int64_t)kt * kBN;
      const int32_t lo = (int32_t)(seg_lo - k0 < 0 ? 0 : (seg_lo - k0 > kBN ? kBN : seg_lo - k0));
      const int32_t hi = (int32_t)(seg_hi - k0 < 0 ? 0 : (seg_hi - k0 > kBN ? kBN : seg_hi - k0));
      float tmax = -INFINITY;
      if (lo == 0 && hi == kBN) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e) tmax = fmaxf(tmax, __uint_as_float(sr[c][e]));
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int col = 32 * c + e;
            const float s = (col >= lo && col < hi) ? __uint_as_float(sr[c][e]) : -INFINITY;
            sr[c][e] = __float_as_uint(s);
            tmax = fmaxf(tmax, s);
          }
      }
      // Lazy rescale: move the reference max only when the new max exceeds it
      // by more than 2^8 in probability (FA4-style); otherwise p <= 256.
      // (tcgen05.ld/st are warp-collective: the O round trip is warp-uniform,
      // lanes that keep their reference max use corr = 1.)
      const bool move = tmax > mref && (mref == -INFINITY || (tmax - mref) * p.c > kRescaleThreshold);
      const bool fix_o = move && mref != -INFINITY;
      if (__any_sync(0xffffffffu, fix_o)) {
        const float corr = fix_o ? ptx::ex2((mref - tmax) * p.c) : 1.0f;
        l *= corr;
        uint32_t orow[2][32];
        ptx::tmem_ld32(tbase + lane_base + kColO, orow[0]);
        ptx::tmem_ld32(tbase + lane_base + kColO + 32, orow[1]);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e) orow[c][e] = __float_as_uint(__uint_as_float(orow[c][e]) * corr);
        ptx::tmem_st32(tbase + lane_base + kColO, orow[0]);
        ptx::tmem_st32(tbase + lane_base + kColO + 32, orow[1]);
      }
      if (move) mref = tmax;
      const float neg = (mref == -INFINITY) ? 0.0f : -mref * p.c;
      float lsum = 0.0f;
      uint32_t pk[2][32];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float p0 = ptx::ex2(fmaf(__uint_as_float(sr[c][e]), p.c, neg));
          const float p1 = ptx::ex2(fmaf(__uint_as_float(sr[c][e + 1]), p.c, neg));
          lsum += p0 + p1;
          pk[c >> 1][(c & 1) * 16 + e / 2] = ptx::pack_bf16x2(p0, p1);
        }
      l += lsum;
      ptx::tmem_st32(tbase + lane_base + kColS, pk[0]);
      ptx::tmem_st32(tbase + lane_base + kColS + 32, pk[1]);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&sm.bar_p);
    }

    // ---------------------------------------------------------- epilogue
    ptx::mbar_wait(&sm.bar_o, 0);
    ptx::tc_fence_after();
    uint32_t orow[2][32];
    ptx::tmem_ld32(tbase + lane_base + kColO, orow[0]);
    ptx::tmem_ld32(tbase + lane_base + kColO + 32, orow[1]);
    ptx::tmem_ld_wait();
    if (valid_q) {
      const float inv = 1.0f / l;
      uint8_t* dst = reinterpret_cast<uint8_t*>(ob + (tq * p.r + gamma) * hd);
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          const float* f = reinterpret_cast<const float*>(&orow[c][e]);
          ptx::st_global_v4(dst + (c * 32 + e) * 2, ptx::pack_bf16x2(f[0] * inv, f[1] * inv),
                            ptx::pack_bf16x2(f[2] * inv, f[3] * inv), ptx::pack_bf16x2(f[4] * inv, f[5] * inv),
                            ptx::pack_bf16x2(f[6] * inv, f[7] * inv));
        }
      if (lse) lse[(b * p.h + j) * p.N + tq * p.r + gamma] = mref * p.scale + logf(l);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tbase);
  }
}

// ---------------------------------------------------------------- host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) == cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// [B*N/r][r][h][64] bf16 view; box (64, 1, 1, 128), 128-byte swizzle.
bool make_map(CUtensorMap* map, const void* base, int64_t rows_div_r, int64_t r, int64_t h) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)kD, (cuuint64_t)h, (cuuint64_t)r, (cuuint64_t)rows_div_r};
  cuuint64_t strides[3] = {(cuuint64_t)kD * 2, (cuuint64_t)h * kD * 2, (cuuint64_t)r * h * kD * 2};
  cuuint32_t box[4] = {kD, 1, 1, 128};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult res = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS;
}

}  // namespace

bool sm100_supported(const Geometry& g, int dtype, const void* q, const void* k, const void* v, const void* o) {
  if (dtype != 1) return false;                   // bf16 only
  if (g.d != kD || g.dv != kD) return false;       // head_dim 64
  if (g.N % g.r != 0) return false;                // t'-stream view needs r | N
  if (g.w % g.r != 0) return false;                // segments are contiguous t'-blocks
  if (g.h > kMaxHeads) return false;
  auto al = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; };
  if (!al(q) || !al(k) || !al(v) || !al(o)) return false;
  const int64_t T = g.N / g.r;
  if (g.B * T > (int64_t)INT32_MAX - 256) return false;  // TMA coordinates are int32
  return true;
}

int launch_sm100(const Geometry& g, const void* q, const void* k, const void* v, void* o, float* lse,
                 cudaStream_t stream, cudaError_t* err, const char** why) {
  const int64_t T = g.N / g.r;
  CUtensorMap mq, mk, mv;
  if (!make_map(&mq, q, g.B * T, g.r, g.h) || !make_map(&mk, k, g.B * T, g.r, g.h) ||
      !make_map(&mv, v, g.B * T, g.r, g.h)) {
    *why = "cuTensorMapEncodeTiled failed";
    *err = cudaErrorInvalidValue;
    return 0;
  }
  Sm100Params p;
  p.N = g.N;
  p.T = T;
  p.m = g.w / g.r;
  p.r = (int32_t)g.r;
  p.h = (int32_t)g.h;
  p.n_qt = (int32_t)((T + kBM - 1) / kBM);
  p.scale = g.scale;
  p.c = g.scale * kLog2e;
  for (int i = 0; i < kMaxHeads; ++i) p.offsets[i] = i < g.h ? g.offsets[i] : 0;
  const size_t smem = sizeof(SmemLayout) + 1024;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(dfa_sm100_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (attr_err != cudaSuccess) {
    *err = attr_err;
    *why = "cudaFuncSetAttribute failed";
    return 0;
  }
  const int64_t n_cta = g.B * g.h * p.n_qt;
  dfa_sm100_kernel<<<(unsigned)n_cta, kThreads, smem, stream>>>(mq, mk, mv, (__nv_bfloat16*)o, lse, p);
  *err = cudaGetLastError();
  return 1;
}

}  // namespace dfa_impl
