// Row-major GEMMs of the layers either side of the hot path (SURVEY §8(f)
// rows 1-2: the Q/K/V and output projections of multi_head_dilated,
// attention.hpp:340-360, and the MLP of the encoder block, encoder.hpp:241-248):
//
//   D[b] = epi(A[b] B[b] + bias + beta C[b])     b < batch
//   A [M, K] (lda, batch stride sa), B [K, N] (ldb, sb), C / D [M, N] (ldc / ldd, sd)
//   epi = identity or GELU in the reference's erf form, x Phi(x)
//         (tensor.hpp:262-265: 0.5 x (1 + erf(x / sqrt 2)))
//
// bf16 (the production mode): a persistent, warp-specialised tcgen05 kernel.
//   * warp 0     TMA producer: A tile [128 x 64] (K-major, SW128) and B tile
//                [64 x BN] as BN/64 boxes of [64 x 64] (N-major, SW128) per
//                stage; 3-4 stage ring.
//   * warp 1     MMA issuer (one elected lane): D_tmem += A B, M = 128, N = BN,
//                K = 16 per instruction; B is an MN-major operand whose 64-wide
//                N atoms sit 8 KB apart (LBO).  Two TMEM accumulators (2 x BN
//                columns) so the epilogue of tile i overlaps the main loop of
//                tile i + 1.
//   * warp 2     TMEM allocator.
//   * warps 4-11 epilogue, two groups of 128 threads (thread = accumulator row =
//                TMEM lane) splitting the 64-column chunks: tcgen05.ld -> + bias
//                -> + beta C (C's chunk TMA-loaded into the group's staging
//                tile) -> GELU -> bf16 -> SW128 staging -> TMA store.
// Row-strided operands (the offset-class split of the layers: rows n = g mod r
// of x, every r-th row of the output) are just TMA strides: A's and D's row
// stride is r D and the class is the batch coordinate -- no gather or scatter
// pass exists.  Edges (M, N, K not multiples of the tile) are TMA zero-fill on
// load and clipping on store.
//
// f32 (the validation mode) and operands TMA cannot describe (16-byte
// alignment) run a SIMT tile kernel with the same epilogue, fp32 FFMA
// accumulation, no TF32.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <atomic>
#include <mutex>

#include "dfa_internal.h"
#include "sm100_ptx.cuh"

namespace dfa_impl {
namespace {

// Profiling probes (variant builds only, results wrong): 1 = the epilogue
// only hands the accumulator back; 2 = no A loads (the MMAs run on stale tiles).
#ifndef DFA_GEMM_PROBE
#define DFA_GEMM_PROBE 0
#endif
constexpr int kGM = 128;        // tile rows (MMA M, TMEM lanes)
constexpr int kGK = 64;         // K per stage: one 128-byte swizzle atom of bf16
constexpr int kGThreads = 384;  // warps 0-3 control, 4-11 epilogue
constexpr int kGTile = kGM * 128;  // bytes of a [128 x 64] bf16 tile
constexpr int kPanelBytes = 144 * 1024;  // resident B panel (K x BN bf16) capacity

// Two main-loop forms:
//  * resident (kRes): each CTA owns ONE column block (batch entry b, tile
//    column nt) whose whole B panel [K x BN] sits in shared memory, and a
//    contiguous run of its m-tiles; only A streams through the ring.  CTAs
//    i .. i + NT - 1 hold the NT column blocks of the same batch entry and
//    the same run of rows, so they read each A tile from DRAM once and from
//    L2 NT - 1 times, while the weights are read once per CTA (K <= 384 at
//    BN = 192: the projections, w1).
//  * streaming: A and B tiles both stream (long K: w2); tiles strided over
//    the grid with n fastest so A's rows are reused from L2.
template <int BN, bool kRes, int kStgT>
struct GemmSmem {
  // budget: A ring + B (panel or ring) + staging tiles within 224 KB
  static constexpr int kNC = BN / 64;
  // k-tiles a resident panel holds: K <= 384 up to BN = 192, K <= 256 at 256
  static constexpr int kPanelStages = kPanelBytes / (kNC * kGK * 128) < 6 ? kPanelBytes / (kNC * kGK * 128) : 6;
  // staging tiles per epilogue group: 2 lets consecutive chunks' stores
  // overlap (heavy epilogues: GELU, residual); 1 leaves room for a deeper A
  // ring (the light ones are load-latency bound)
  static constexpr int kStg = kStgT;
  static constexpr int kStages = kRes ? (224 * 1024 - kPanelStages * kNC * kGK * 128 - 2 * kStg * kGTile) / kGTile
                                      : (224 * 1024 - 2 * kStg * kGTile) / (kGTile + kNC * kGK * 128);
  static constexpr int kBStages = kRes ? kPanelStages : kStages;
  uint8_t a[kStages][kGTile];
  uint8_t b[kBStages][kNC][kGK * 128];     // panel (k-tiles) or ring stages
  uint8_t stage[2][kStg][kGTile];          // staging tiles per epilogue group
  uint64_t full[kStages], empty[kStages];
  uint64_t acc_full[2], acc_empty[2];
  uint64_t cload[2];
  uint64_t b_full;                          // resident panel loaded
  uint32_t tmem_base;
};

struct GemmParams {
  int32_t M, N, K, batch;
  int32_t a_batched, b_batched;  // 0: the operand is shared by every batch entry (batch stride 0)
  int32_t mt, nt, n_tiles, ktiles;
  int32_t n_keys, rows_per_key, ctas_per_key;  // resident: column blocks, m-tiles per block, CTAs per block
  int32_t has_c, gelu;
  float beta;
  const __nv_bfloat16* bias;
};

__device__ __forceinline__ float gelu_erf(float x) {
  // tensor.hpp:262-265: 0.5 x (1 + erf(x / sqrt(2)))
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}

// GELU of the bf16 epilogue on a pair: x Phi(x) with Phi(x) = (1 + tanh(y)) / 2,
// y = x (a + b x^2), a and b minimax-fitted to the erf form
// (tensor.hpp:262-265): max |GELU error| 2.7e-4 over all x, plus
// tanh.approx's 2^-11 relative -- far below the bf16 result's rounding step
// (2^-9 relative) -- on one MUFU op and 5 packed FMA-pipe ops per pair
// instead of erff's ~20 instructions per element.  (fp32, the validation
// mode, keeps erff.)
__device__ __forceinline__ float2 gelu2(float2 v) {
  const float2 x2 = ptx::fmul2(v, v);
  const float2 t = ptx::ffma2(x2, make_float2(0.03470089f, 0.03470089f), make_float2(0.80015708f, 0.80015708f));
  const float2 y = ptx::fmul2(v, t);
  const float2 hx = ptx::fmul2(v, make_float2(0.5f, 0.5f));
  return ptx::ffma2(hx, make_float2(ptx::tanh_approx(y.x), ptx::tanh_approx(y.y)), hx);
}

// Epilogue kinds (compile-time so the per-element path is straight-line
// code): bit 0 bias, bit 1 residual C, bit 2 GELU; kEpiAny reads the
// runtime flags.
constexpr int kEpiBias = 1, kEpiC = 2, kEpiGelu = 4, kEpiAny = -1;

// Tile t -> (batch b, first row m0, column block nt).  Resident: t counts
// this CTA's own m-tiles of its column block (key = blockIdx.x % n_keys).
template <bool kRes>
__device__ __forceinline__ void decode_tile(const GemmParams& p, int32_t t, int32_t* b, int32_t* m0, int32_t* nt) {
  if (kRes) {
    const int32_t key = blockIdx.x % p.n_keys;
    if (p.b_batched) {  // a B panel per batch entry: key = (b, nt)
      *b = key / p.nt;
      *nt = key % p.nt;
      *m0 = t * kGM;
    } else {  // shared weights: key = nt, the rows run over (b, m)
      *nt = key;
      *b = t / p.mt;
      *m0 = (t % p.mt) * kGM;
    }
  } else {  // (b, m, n): consecutive tiles share A's rows (L2)
    *nt = t % p.nt;
    const int32_t rest = t / p.nt;
    *m0 = (rest % p.mt) * kGM;
    *b = rest / p.mt;
  }
}

// This CTA's tiles: a contiguous run of its column block's m-tiles
// (resident) or a grid-strided set.
template <bool kRes>
__device__ __forceinline__ void tile_range(const GemmParams& p, int32_t* t0, int32_t* t1, int32_t* dt) {
  if (kRes) {
    const int32_t j = blockIdx.x / p.n_keys;
    *t0 = (int32_t)(((int64_t)j * p.rows_per_key) / p.ctas_per_key);
    *t1 = (int32_t)(((int64_t)(j + 1) * p.rows_per_key) / p.ctas_per_key);
    *dt = 1;
  } else {
    *t0 = blockIdx.x;
    *t1 = p.n_tiles;
    *dt = gridDim.x;
  }
}

template <int BN, bool kRes, int kStgT, int kEpi>
__global__ void __launch_bounds__(kGThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                      const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_d,
                      const __grid_constant__ GemmParams p) {
  using Smem = GemmSmem<BN, kRes, kStgT>;
  constexpr int S = Smem::kStages;
  const bool has_bias = kEpi == kEpiAny ? p.bias != nullptr : (kEpi & kEpiBias) != 0;
  const bool has_c = kEpi == kEpiAny ? p.has_c != 0 : (kEpi & kEpiC) != 0;
  const bool has_gelu = kEpi == kEpiAny ? p.gelu != 0 : (kEpi & kEpiGelu) != 0;
  constexpr int NC = BN / 64;
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  int32_t t0, t1, dt;
  tile_range<kRes>(p, &t0, &t1, &dt);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&sm.full[s], 1);
      ptx::mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&sm.acc_full[b], 1);
      ptx::mbar_init(&sm.acc_empty[b], 2 * kGM);
      ptx::mbar_init(&sm.cload[b], 1);
    }
    ptx::mbar_init(&sm.b_full, 1);
    ptx::fence_barrier_init();
    ptx::tma_prefetch_desc(&tm_a);
    ptx::tma_prefetch_desc(&tm_b);
    ptx::tma_prefetch_desc(&tm_c);
    ptx::tma_prefetch_desc(&tm_d);
  } else if (warp == 2) {
    ptx::tmem_alloc<512>(&sm.tmem_base);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = sm.tmem_base;
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();

  if (warp == 0) {
    // ================================================================ producer
    if (ptx::elect_one()) {
      const uint64_t pol_a = ptx::policy_evict_normal();  // activations: re-read by the other column blocks
      const uint64_t pol_b = ptx::policy_evict_last();   // weights: reused by every CTA
      uint32_t it = 0, pan = 0;
      for (int32_t t = t0; t < t1; t += dt) {
        int32_t b, m0, nt;
        decode_tile<kRes>(p, t, &b, &m0, &nt);
        const int32_t n0 = nt * BN;
        if (kRes && pan == 0) {  // the CTA's column block: its whole B panel, once
          ptx::mbar_arrive_expect_tx(&sm.b_full, (uint32_t)(p.ktiles * NC * kGK * 128));
          for (int32_t kt = 0; kt < p.ktiles; ++kt)
#pragma unroll
            for (int c = 0; c < NC; ++c)
              ptx::tma_load_3d(sm.b[kt][c], &tm_b, &sm.b_full, n0 + 64 * c, kt * kGK, b * p.b_batched, pol_b);
          pan = 1;
        }
        for (int32_t kt = 0; kt < p.ktiles; ++kt, ++it) {
          const uint32_t s = it % S;
          ptx::mbar_wait(&sm.empty[s], ((it / S) & 1) ^ 1);
          if (DFA_GEMM_PROBE == 2 && kRes) {
            ptx::mbar_arrive(&sm.full[s]);
            continue;
          }
          ptx::mbar_arrive_expect_tx(&sm.full[s], kRes ? kGTile : kGTile + NC * kGK * 128);
          ptx::tma_load_3d(sm.a[s], &tm_a, &sm.full[s], kt * kGK, m0, b * p.a_batched, pol_a);
          if (!kRes) {
#pragma unroll
            for (int c = 0; c < NC; ++c)
              ptx::tma_load_3d(sm.b[s][c], &tm_b, &sm.full[s], n0 + 64 * c, kt * kGK, b * p.b_batched, pol_b);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================================================ MMA issuer
    if (ptx::elect_one()) {
      constexpr uint32_t idesc = ptx::idesc_bf16(kGM, BN, 0, 1);  // A K-major, B MN-major
      uint32_t it = 0, tc = 0;
      if (kRes && t0 < t1) ptx::mbar_wait(&sm.b_full, 0);  // the CTA's B panel
      for (int32_t t = t0; t < t1; t += dt, ++tc) {
        const uint32_t buf = tc & 1;
        ptx::mbar_wait(&sm.acc_empty[buf], ((tc >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t dcol = tbase + buf * BN;
        for (int32_t kt = 0; kt < p.ktiles; ++kt, ++it) {
          const uint32_t s = it % S;
          ptx::mbar_wait(&sm.full[s], (it / S) & 1);
          ptx::tc_fence_after();
          const uint64_t ad = ptx::sdesc_sw128(ptx::smem_u32(sm.a[s]));
          // MN-major B: 64-column atoms 8 KB apart (LBO), 8-row groups 1 KB apart (SBO)
          const uint64_t bd = ptx::sdesc_sw128(ptx::smem_u32(sm.b[kRes ? kt : s][0]), 1024, kGK * 128);
#pragma unroll
          for (int kk = 0; kk < kGK / 16; ++kk)
            ptx::mma_ss(dcol, ad + (uint64_t)(2 * kk), bd + (uint64_t)(kk * (2048 >> 4)), idesc,
                        (kt > 0 || kk > 0) ? 1u : 0u);
          ptx::tc_commit(&sm.empty[s]);
        }
        ptx::tc_commit(&sm.acc_full[buf]);
      }
    }
  } else if (warp >= 4) {
    // ============================================================== epilogue
    const uint32_t grp = (warp - 4) / 4;
    const uint32_t row = (warp % 4) * 32 + lane;
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const bool leader = (warp % 4) == 0 && lane == 0;
    const uint32_t bar_id = 1 + grp;
    constexpr int kStg = Smem::kStg;
    const uint64_t pol_c = ptx::policy_evict_first();
    uint32_t tc = 0, cl_par = 0, sc = 0;  // sc: chunks this group stored (staging rotation)
    for (int32_t t = t0; t < t1; t += dt, ++tc) {
      int32_t b, m0, nt;
      decode_tile<kRes>(p, t, &b, &m0, &nt);
      const int32_t n0 = nt * BN;
      const uint32_t buf = tc & 1;
      // the residual chunk of this group's first column block lands in the
      // staging tile while the main loop still runs
      if (has_c && leader && (int)grp < NC && n0 + 64 * (int)grp < p.N && DFA_GEMM_PROBE != 1) {
        ptx::tma_store_wait_read<kStg - 1>();
        ptx::mbar_arrive_expect_tx(&sm.cload[grp], kGTile);
        ptx::tma_load_3d(sm.stage[grp][sc % kStg], &tm_c, &sm.cload[grp], n0 + 64 * grp, m0, b, pol_c);
      }
      ptx::mbar_wait(&sm.acc_full[buf], (tc >> 1) & 1);
      ptx::tc_fence_after();
      for (int c = grp; c < NC && DFA_GEMM_PROBE != 1; c += 2) {
        const int32_t col0 = n0 + 64 * c;
        if (col0 >= p.N) break;
        uint8_t* stg = sm.stage[grp][sc % kStg];
        const uint32_t stage_addr = ptx::smem_u32(stg);
        if (has_c) {
          if (c != (int)grp && leader) {  // later chunks: load once this buffer's last store drained
            ptx::tma_store_wait_read<kStg - 1>();
            ptx::mbar_arrive_expect_tx(&sm.cload[grp], kGTile);
            ptx::tma_load_3d(stg, &tm_c, &sm.cload[grp], col0, m0, b, pol_c);
          }
          ptx::mbar_wait(&sm.cload[grp], cl_par);
          cl_par ^= 1;
        } else {
          if (leader) ptx::tma_store_wait_read<kStg - 1>();  // this buffer's previous store has been read
          ptx::named_bar_sync(bar_id, kGM);
        }
        uint32_t acc[2][32];
        ptx::tmem_ld32(tbase + lane_base + buf * BN + 64 * c, acc[0]);
        ptx::tmem_ld32(tbase + lane_base + buf * BN + 64 * c + 32, acc[1]);
        ptx::tmem_ld_wait();
        const bool full_bias = has_bias && col0 + 64 <= p.N;
        const uint4* bp = reinterpret_cast<const uint4*>(p.bias + col0);  // 8 bias values per 16-byte load
        const float2 beta2 = make_float2(p.beta, p.beta);
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          const uint32_t addr = stage_addr + row * 128 + ((c8 ^ (row & 7)) * 16);
          float2 v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            v[e] = make_float2(__uint_as_float(acc[c8 >> 2][(c8 & 3) * 8 + 2 * e]),
                               __uint_as_float(acc[c8 >> 2][(c8 & 3) * 8 + 2 * e + 1]));
          if (full_bias) {
            const uint4 w = bp[c8];
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = ptx::fadd2(v[e], ptx::unpack_bf16x2(ww[e]));
          } else if (has_bias) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int col = col0 + 8 * c8 + e;
              const float bv = col < p.N ? __bfloat162float(p.bias[col]) : 0.0f;
              if (e & 1)
                v[e >> 1].y += bv;
              else
                v[e >> 1].x += bv;
            }
          }
          if (has_c) {
            uint32_t prev[4];
            ptx::ld_shared_v4(addr, prev);
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = ptx::ffma2(beta2, ptx::unpack_bf16x2(prev[e]), v[e]);
          }
          if (has_gelu) {
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = gelu2(v[e]);
          }
          ptx::st_shared_v4(addr, ptx::pack_bf16x2(v[0].x, v[0].y), ptx::pack_bf16x2(v[1].x, v[1].y),
                            ptx::pack_bf16x2(v[2].x, v[2].y), ptx::pack_bf16x2(v[3].x, v[3].y));
        }
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(bar_id, kGM);
        if (leader) {
          ptx::tma_store_3d(&tm_d, stg, col0, m0, b);
          ptx::tma_store_commit();
        }
        ++sc;
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&sm.acc_empty[buf]);
    }
    if (leader) ptx::tma_store_wait_all<0>();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tbase);
  }
}

// ------------------------------------------------------- SIMT (f32 / fallback)
template <typename T>
__device__ __forceinline__ float ld_f(const T* p);
template <>
__device__ __forceinline__ float ld_f<float>(const float* p) {
  return *p;
}
template <>
__device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ T to_t(float x);
template <>
__device__ __forceinline__ float to_t<float>(float x) {
  return x;
}
template <>
__device__ __forceinline__ __nv_bfloat16 to_t<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

struct SimtGemmParams {
  int64_t M, N, K, lda, sa, ldb, sb, ldd, sd, ldc;
  float beta;
  int32_t gelu;
};

// 64 x 64 output tile per CTA, 256 threads x (4 x 4) outputs, K tiles of 16,
// fp32 FFMA (no TF32): the validation mode's GEMM.
template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const T* __restrict__ A, const T* __restrict__ B,
                                                        const T* __restrict__ C, const T* __restrict__ bias,
                                                        T* __restrict__ D, const __grid_constant__ SimtGemmParams p) {
  __shared__ float as[16][64 + 1];
  __shared__ float bs[16][64];
  const int64_t b = blockIdx.z;
  const int64_t m0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const T* Ab = A + b * p.sa;
  const T* Bb = B + b * p.sb;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < p.K; k0 += 16) {
    for (int e = threadIdx.x; e < 64 * 16; e += 256) {
      const int mm = e / 16, kk = e % 16;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      as[kk][mm] = (gm < p.M && gk < p.K) ? ld_f(Ab + gm * p.lda + gk) : 0.0f;
      const int kb = e / 64, nn = e % 64;
      const int64_t gn = n0 + nn, gkb = k0 + kb;
      bs[kb][nn] = (gn < p.N && gkb < p.K) ? ld_f(Bb + gkb * p.ldb + gn) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = as[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gm = m0 + ty * 4 + i, gn = n0 + tx * 4 + j;
      if (gm >= p.M || gn >= p.N) continue;
      float v = acc[i][j];
      if (bias) v += ld_f(bias + gn);
      if (C) v = fmaf(p.beta, ld_f(C + b * p.sd + gm * p.ldc + gn), v);
      if (p.gelu) v = gelu_erf(v);
      D[b * p.sd + gm * p.ldd + gn] = to_t<T>(v);
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
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

// Row-major bf16 matrix [batch][rows][cols] with row stride ld and batch
// stride sb (elements); box (64 cols, box_rows rows, 1), 128-byte swizzle.
#ifndef DFA_GEMM_PROMO_A
#define DFA_GEMM_PROMO_A CU_TENSOR_MAP_L2_PROMOTION_L2_128B
#endif
bool map3(CUtensorMap* map, const void* base, int64_t cols, int64_t rows, int64_t batch, int64_t ld, int64_t sb,
          uint32_t box_rows, CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)(batch > 1 ? sb : rows * ld) * 2};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tma_ok(const void* p, int64_t ld, int64_t sb, int batch) {
  if (reinterpret_cast<uintptr_t>(p) & 15u) return false;
  if ((ld * 2) % 16 != 0) return false;
  if (batch > 1 && (sb * 2) % 16 != 0) return false;
  return true;
}

template <int BN, bool kRes, int kStg, int kEpi = kEpiAny>
int launch_bn(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int64_t sa, const void* B, int64_t ldb,
              int64_t sb, void* D, int64_t ldd, int64_t sd, const void* C, int64_t ldc, float beta, const void* bias,
              int batch, cudaStream_t stream, const char** why, bool gelu) {
  CUtensorMap ma, mb, mc, md;
  const int a_bat = (batch > 1 && sa != 0) ? batch : 1, b_bat = (batch > 1 && sb != 0) ? batch : 1;
  if (!map3(&ma, A, K, M, a_bat, lda, sa, kGM, (CUtensorMapL2promotion)DFA_GEMM_PROMO_A) || !map3(&mb, B, N, K, b_bat, ldb, sb, kGK) ||
      !map3(&md, D, N, M, batch, ldd, sd, kGM) || !map3(&mc, C ? C : D, N, M, batch, C ? ldc : ldd, sd, kGM)) {
    *why = "cuTensorMapEncodeTiled failed (GEMM operands)";
    return 0;
  }
  GemmParams p;
  p.M = (int32_t)M;
  p.N = (int32_t)N;
  p.K = (int32_t)K;
  p.batch = batch;
  p.a_batched = a_bat > 1 ? 1 : 0;
  p.b_batched = b_bat > 1 ? 1 : 0;
  p.mt = (int32_t)((M + kGM - 1) / kGM);
  p.nt = (int32_t)((N + BN - 1) / BN);
  p.n_tiles = p.mt * p.nt * batch;
  p.ktiles = (int32_t)((K + kGK - 1) / kGK);
  p.n_keys = (int32_t)((p.b_batched ? batch : 1) * p.nt);
  p.rows_per_key = (int32_t)(p.b_batched ? p.mt : (int64_t)p.mt * batch);
  p.ctas_per_key = std::max(1, device_sms() / p.n_keys);
  p.has_c = C ? 1 : 0;
  p.gelu = gelu ? 1 : 0;
  p.beta = beta;
  p.bias = static_cast<const __nv_bfloat16*>(bias);
  using Smem = GemmSmem<BN, kRes, kStg>;
  const size_t smem = sizeof(Smem) + 1024;
  static_assert(sizeof(Smem) + 1024 <= 232448, "GEMM shared memory exceeds 227 KB");
  static_assert(Smem::kStages >= 2, "GEMM A ring needs >= 2 stages");
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(gemm_sm100_kernel<BN, kRes, kStg, kEpi>), smem);
  if (e != cudaSuccess) {
    *why = "cudaFuncSetAttribute failed (GEMM)";
    return 0;
  }
  const int grid = kRes ? p.n_keys * p.ctas_per_key : (int)std::min<int64_t>(p.n_tiles, device_sms());
  e = launch_pdl(gemm_sm100_kernel<BN, kRes, kStg, kEpi>, grid, kGThreads, smem, stream, ma, mb, mc, md, p);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    *why = cudaGetErrorString(e);
    return 0;
  }
  return 1;
}

std::atomic<int> g_force_bn{0};  // measurement knob (dfa_set_gemm_tile); 0 = auto

#ifndef DFA_GEMM_STG
#define DFA_GEMM_STG 0
#endif
// Plain projections with K >= 256 and N % 192 == 0 (the class-split QKV
// GEMM) stream 192-wide tiles; otherwise the resident panel at BN = 128
// whenever it fits (K <= 384: a resident 192-wide panel leaves only 3 A
// stages and the main loop is load-latency bound); light epilogues take a
// 6-deep A ring with one staging tile per group, GELU / residual epilogues
// 4 stages and two.  GELU epilogues with N % 256 == 0 stream 256-wide tiles;
// longer K streams A and B tiles (BN = 192, 4 stages).
int launch_dispatch(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int64_t sa, const void* B,
                    int64_t ldb, int64_t sb, void* D, int64_t ldd, int64_t sd, const void* C, int64_t ldc, float beta,
                    const void* bias, int batch, cudaStream_t stream, const char** why, bool gelu, int force_bn) {
  const int64_t ktiles = (K + kGK - 1) / kGK;
  const bool heavy = gelu || C != nullptr;
  const int stg = DFA_GEMM_STG ? DFA_GEMM_STG : (heavy ? 2 : 1);
#define DFA_GEMM_ARGS M, N, K, A, lda, sa, B, ldb, sb, D, ldd, sd, C, ldc, beta, bias, batch, stream, why, gelu
  const int bn_res = force_bn ? force_bn : 128;
  const int64_t keys = (batch > 1 && sb != 0 ? batch : 1) * ((N + bn_res - 1) / bn_res);
  const int epi = (bias ? kEpiBias : 0) | (C ? kEpiC : 0) | (gelu ? kEpiGelu : 0);
  // plain projections with K >= 256 whose N splits into 192-wide blocks (the
  // class-split QKV GEMM: N = 3 h d / r): streaming 192-wide tiles measured
  // 3-7% faster than the resident 128-wide panel (fewer A re-reads; the
  // resident 192-wide panel leaves only 3 A stages and lost)
  if (!force_bn && !DFA_GEMM_STG && epi == 0 && ktiles >= 4 && N % 192 == 0)
    return launch_bn<192, false, 2>(DFA_GEMM_ARGS);
  if (ktiles <= 6 && keys <= device_sms() && (bn_res == 128 || bn_res == 64)) {
    if (bn_res == 64) return stg == 1 ? launch_bn<64, true, 1>(DFA_GEMM_ARGS) : launch_bn<64, true, 2>(DFA_GEMM_ARGS);
    if (!DFA_GEMM_STG && !force_bn) {  // the layers' epilogues, straight-line
      if (epi == 0) return launch_bn<128, true, 1, 0>(DFA_GEMM_ARGS);
      if (epi == (kEpiBias | kEpiC)) return launch_bn<128, true, 2, kEpiBias | kEpiC>(DFA_GEMM_ARGS);
      // GELU epilogues: 256-wide tiles (two chunks per group per tile keep
      // the TMA store of one chunk under the math of the next): measured
      // 0.40 vs 0.45 ms on w1 at config 2
      if (epi == (kEpiBias | kEpiGelu) && N % 256 == 0)
        return launch_bn<256, false, 1, kEpiBias | kEpiGelu>(DFA_GEMM_ARGS);
    }
    return stg == 1 ? launch_bn<128, true, 1>(DFA_GEMM_ARGS) : launch_bn<128, true, 2>(DFA_GEMM_ARGS);
  }
  if (!force_bn && epi == (kEpiBias | kEpiC)) return launch_bn<192, false, 2, kEpiBias | kEpiC>(DFA_GEMM_ARGS);
  switch (force_bn ? force_bn : 192) {
    case 64: return launch_bn<64, false, 2>(DFA_GEMM_ARGS);
    case 128: return launch_bn<128, false, 2>(DFA_GEMM_ARGS);
    case 256: return launch_bn<256, false, 1>(DFA_GEMM_ARGS);
    default: return launch_bn<192, false, 2>(DFA_GEMM_ARGS);
  }
#undef DFA_GEMM_ARGS
}

}  // namespace

int gemm_rowmajor(int dtype, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int64_t sa, const void* B,
                  int64_t ldb, int64_t sb, void* D, int64_t ldd, int64_t sd, const void* C, int64_t ldc, float beta,
                  const void* bias, int batch, cudaStream_t stream, const char** why, bool gelu) {
  if (M <= 0 || N <= 0 || batch <= 0) return 1;
  ensure_context();
  const bool tc = dtype == 1 && K > 0 && M < INT32_MAX / 2 && N < INT32_MAX / 2 && tma_ok(A, lda, sa, batch) &&
                  tma_ok(B, ldb, sb, batch) && tma_ok(D, ldd, sd, batch) && (!C || tma_ok(C, ldc, sd, batch)) &&
                  (!bias || (reinterpret_cast<uintptr_t>(bias) & 15u) == 0);
  if (tc) return launch_dispatch(M, N, K, A, lda, sa, B, ldb, sb, D, ldd, sd, C, ldc, beta, bias, batch, stream, why,
                                 gelu, g_force_bn.load());
  SimtGemmParams p{M, N, K, lda, sa, ldb, sb, ldd, sd, ldc, beta, gelu ? 1 : 0};
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64), (unsigned)batch);
  if (dtype == 0)
    gemm_simt_kernel<float><<<grid, 256, 0, stream>>>((const float*)A, (const float*)B, (const float*)C,
                                                       (const float*)bias, (float*)D, p);
  else
    gemm_simt_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(
        (const __nv_bfloat16*)A, (const __nv_bfloat16*)B, (const __nv_bfloat16*)C, (const __nv_bfloat16*)bias,
        (__nv_bfloat16*)D, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *why = cudaGetErrorString(e);
    return 0;
  }
  return 1;
}

void set_gemm_tile(int bn) { g_force_bn.store(bn); }

}  // namespace dfa_impl
