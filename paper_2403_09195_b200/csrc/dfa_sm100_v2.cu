// Forward kernel "v2": four query slots of 128 rows per unit (512 t'-rows),
// 64-key S tiles, one S buffer per slot.  Same math, layout, boundary and
// output semantics as dfa_sm100_kernel (dfa_sm100.cu -- read its header
// first); what changes is the concurrency.  v1's ncu sweep shows neither the
// MUFU (XU ~60%) nor the issue slots saturated on compute-bound shapes: the
// two softmax slots spend their time waiting on the serial
// Q K^T -> softmax -> P V chain.  Four slots (one warp of each per SMSP) give
// every SMSP four independent softmax streams to interleave.
//
// TMEM (512 columns): S_s at 64 s (P_s, bf16, over its first 32 columns),
// O_s at 256 + 64 s.
//
// Step order (identical in every role).  Slots whose key ranges start at the
// same key tile form a group and share that tile's K / V loads.  Round rho
// visits the slots in order; slot s is active while rho < len_s and uses key
// tile kt0_s + rho.  Round-robin over the groups keeps all four slots busy
// even when they sit in different segments (m = 256: slots {0,1} and {2,3}).
// Within a group the lengths are non-decreasing, so the active members of a
// round are a suffix of the group: the first active one loads the tile, the
// last one releases it.
//
// Warp roles (768 threads, one CTA per SM, persistent over units):
//   warp 0      TMA producer: Q_0..Q_3 (one stage per slot), K tiles (ring)
//   warp 1      Q K^T issuer: S_s = Q_s K^T (M=128, N=64); S_s is reused once
//               the slot's previous P V completed (s_free[s])
//   warp 2      TMEM allocator, then P V issuer: O_s += P_s V (A = P_s in TMEM)
//   warp 3      TMA producer: V tiles (ring)
//   warps 4-19  softmax of slots 0-3 (thread = query row = TMEM lane)
//   warps 20-23 epilogue: O / l -> bf16 -> TMA store + zero boxes (+ lse)
// Merge mode (multi-branch) stays on v1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <mutex>

#include "dfa_internal.h"
#include "sm100_ptx.cuh"

namespace dfa_impl {
namespace {

constexpr int kD = 64;
constexpr int kBM = 128;             // rows per slot
constexpr int kSlots = 4;
constexpr int kUnit = kSlots * kBM;  // t'-rows per unit
constexpr int kBN = 64;              // keys per step
constexpr int kQTile = kBM * 128;    // 16 KB
constexpr int kKVTile = kBN * 128;   // 8 KB
#ifndef DFA_V2_STAGES
#define DFA_V2_STAGES 6
#endif
constexpr int kKStages = DFA_V2_STAGES, kVStages = DFA_V2_STAGES;
constexpr int kThreads = 768;
constexpr float kLog2e = 1.4426950408889634f;
#ifndef DFA_RESCALE_THR
#define DFA_RESCALE_THR 8.0f
#endif
#ifndef DFA_V2_POLY_MASK
#define DFA_V2_POLY_MASK 0x8888u
#endif
constexpr float kThr = DFA_RESCALE_THR;
constexpr uint32_t kPolyMask = DFA_V2_POLY_MASK;

__host__ __device__ constexpr uint32_t col_s(int s) { return 64u * s; }
__host__ __device__ constexpr uint32_t col_o(int s) { return 256u + 64u * s; }

struct __align__(1024) Smem {
  uint8_t q[kSlots][kQTile];
  uint8_t k[kKStages][kKVTile];
  uint8_t v[kVStages][kKVTile];
  uint8_t ostage[2][kQTile];
  uint8_t zero[kQTile];
  uint64_t q_full[kSlots], q_empty[kSlots];
  uint64_t k_full[kKStages], k_empty[kKStages];
  uint64_t v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[kSlots], p_full[kSlots], s_free[kSlots], pv_done[kSlots];
  uint64_t o_full[kSlots], o_empty[kSlots], stat_full[kSlots], stat_empty[kSlots];
  float stat_l[2][kSlots][kBM], stat_m[2][kSlots][kBM];
  uint32_t tmem_base;
};

struct FastDiv {
  uint32_t d, mul, shift;
  __device__ __forceinline__ int32_t div(int32_t n) const {
    return (int32_t)((__umulhi((uint32_t)n, mul) + (uint32_t)n) >> shift);
  }
};
FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t shift = 0;
  while ((1ull << shift) < d) ++shift;
  f.shift = shift;
  f.mul = (uint32_t)((((1ull << 32) * ((1ull << shift) - d)) / d) + 1);
  if (d == 1) f.mul = 0;
  return f;
}

struct Params {
  int32_t N, T, m, r, h, n_units, n_blocks;  // n_blocks: units per (b, j) stream
  float c, scale;
  FastDiv div_blocks, div_h, div_m;
  int32_t offsets[kMaxHeads];
};

struct Unit {
  int32_t b, j, gamma, t0, kv_lo, rounds;
  int32_t kt0[kSlots], len[kSlots];  // first key tile (relative to kv_lo) and tile count; len 0 = no rows
  __device__ __forceinline__ bool active(int s, int32_t rho) const { return s >= 0 && s < kSlots && rho < len[s]; }
  // first active slot of its group in round rho: loads the group's key tile
  __device__ __forceinline__ bool lead(int s, int32_t rho) const {
    return active(s, rho) && (s == 0 || kt0[s] != kt0[s - 1] || !active(s - 1, rho));
  }
  // last active slot of its group in round rho: releases the tile
  __device__ __forceinline__ bool last(int s, int32_t rho) const {
    return active(s, rho) && (s == kSlots - 1 || kt0[s + 1] != kt0[s] || !active(s + 1, rho));
  }
};

__device__ __forceinline__ Unit make_unit(const Params& p, int32_t u) {
  Unit x;
  const int32_t bp = p.div_h.div(u);  // head-major: the h CTAs side by side share token rows
  x.j = u - bp * p.h;
  x.b = p.div_blocks.div(bp);
  const int32_t blk = bp - x.b * p.n_blocks;
  x.gamma = p.offsets[x.j];
  x.t0 = blk * kUnit;
  x.kv_lo = p.div_m.div(x.t0) * p.m;
  x.rounds = 0;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    const int32_t r0 = x.t0 + s * kBM, r1 = min(r0 + kBM, p.T);
    if (r0 < r1) {
      const int32_t lo = p.div_m.div(r0) * p.m;
      const int32_t hi = min((p.div_m.div(r1 - 1) + 1) * p.m, p.T);
      x.kt0[s] = (lo - x.kv_lo) / kBN;  // lo - kv_lo is a multiple of m, not of kBN: floor
      x.len[s] = (hi - x.kv_lo + kBN - 1) / kBN - x.kt0[s];
    } else {
      x.kt0[s] = 0;
      x.len[s] = 0;
    }
    x.rounds = max(x.rounds, x.len[s]);
  }
  return x;
}

__global__ void __launch_bounds__(kThreads, 1)
    dfa_sm100_v2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                        float* __restrict__ lse, const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  for (uint32_t i = threadIdx.x; i < kQTile / 16; i += kThreads) ptx::st_shared_v4(ptx::smem_u32(sm.zero) + 16 * i, 0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kSlots; ++s) {
      ptx::mbar_init(&sm.q_full[s], 1);
      ptx::mbar_init(&sm.q_empty[s], 1);
      ptx::mbar_init(&sm.s_full[s], 1);
      ptx::mbar_init(&sm.p_full[s], kBM);
      ptx::mbar_init(&sm.s_free[s], 1);
      ptx::mbar_init(&sm.pv_done[s], 1);
      ptx::mbar_init(&sm.o_full[s], 1);
      ptx::mbar_init(&sm.o_empty[s], kBM);
      ptx::mbar_init(&sm.stat_full[s], kBM);
      ptx::mbar_init(&sm.stat_empty[s], kBM);
    }
    for (int s = 0; s < kKStages; ++s) {
      ptx::mbar_init(&sm.k_full[s], 1);
      ptx::mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      ptx::mbar_init(&sm.v_full[s], 1);
      ptx::mbar_init(&sm.v_empty[s], 1);
    }
    ptx::fence_barrier_init();
  } else if (warp == 2) {
    ptx::tmem_alloc<512>(&sm.tmem_base);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (warp < 4) {
    ptx::setmaxnreg_dec<48>();
    if (warp == 0) {
      // ------------------------------------------------- Q / K producer
      if (ptx::elect_one()) {
        const uint64_t pol = ptx::policy_evict_first();
        uint32_t g = 0, qpar = 0;  // K loads issued; bit s: parity of slot s's Q-stage reuse
        for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
          const Unit x = make_unit(p, u);
#pragma unroll
          for (int s = 0; s < kSlots; ++s) {
            if (x.len[s] == 0) continue;
            ptx::mbar_wait(&sm.q_empty[s], ((qpar >> s) & 1u) ^ 1u);
            qpar ^= 1u << s;
            ptx::mbar_arrive_expect_tx(&sm.q_full[s], kQTile);
            ptx::tma_load_5d(sm.q[s], &tm_q, &sm.q_full[s], 0, x.j, x.gamma, x.t0 + s * kBM, x.b, pol);
          }
          for (int32_t rho = 0; rho < x.rounds; ++rho) {
#pragma unroll
            for (int s = 0; s < kSlots; ++s) {
              if (!x.lead(s, rho)) continue;
              const uint32_t st = g % kKStages;
              ptx::mbar_wait(&sm.k_empty[st], ((g / kKStages) & 1) ^ 1);
              ptx::mbar_arrive_expect_tx(&sm.k_full[st], kKVTile);
              ptx::tma_load_5d(sm.k[st], &tm_k, &sm.k_full[st], 0, x.j, x.gamma,
                               x.kv_lo + (x.kt0[s] + rho) * kBN, x.b, pol);
              ++g;
            }
          }
        }
      }
    } else if (warp == 3) {
      // ------------------------------------------------------ V producer
      if (ptx::elect_one()) {
        const uint64_t pol = ptx::policy_evict_first();
        uint32_t g = 0;
        for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
          const Unit x = make_unit(p, u);
          for (int32_t rho = 0; rho < x.rounds; ++rho) {
#pragma unroll
            for (int s = 0; s < kSlots; ++s) {
              if (!x.lead(s, rho)) continue;
              const uint32_t st = g % kVStages;
              ptx::mbar_wait(&sm.v_empty[st], ((g / kVStages) & 1) ^ 1);
              ptx::mbar_arrive_expect_tx(&sm.v_full[st], kKVTile);
              ptx::tma_load_5d(sm.v[st], &tm_v, &sm.v_full[st], 0, x.j, x.gamma,
                               x.kv_lo + (x.kt0[s] + rho) * kBN, x.b, pol);
              ++g;
            }
          }
        }
      }
    } else if (warp == 1) {
      // ------------------------------------------------- Q K^T issuer
      if (ptx::elect_one()) {
        constexpr uint32_t idesc = ptx::idesc_bf16(kBM, kBN, 0, 0);
        const uint64_t qdesc0 = ptx::sdesc_sw128(ptx::smem_u32(sm.q[0]));
        const uint64_t kdesc0 = ptx::sdesc_sw128(ptx::smem_u32(sm.k[0]));
        uint32_t g = 0, qpar = 0;
        uint32_t used = 0;    // bit s: S_s written before (s_free phases to wait for)
        uint32_t frpar = 0;   // bit s: parity of the next s_free[s] completion
        for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
          const Unit x = make_unit(p, u);
          for (int32_t rho = 0; rho < x.rounds; ++rho) {
            uint64_t kd = 0;
#pragma unroll
            for (int s = 0; s < kSlots; ++s) {
              if (!x.active(s, rho)) continue;
              if (rho == 0) {
                ptx::mbar_wait(&sm.q_full[s], (qpar >> s) & 1u);
                qpar ^= 1u << s;
              }
              if (x.lead(s, rho)) {
                const uint32_t st = g % kKStages;
                ptx::mbar_wait(&sm.k_full[st], (g / kKStages) & 1);
                kd = kdesc0 + (uint64_t)(st * (kKVTile >> 4));
              }
              if ((used >> s) & 1u) {  // S_s is free once the slot's previous P V completed
                ptx::mbar_wait(&sm.s_free[s], (frpar >> s) & 1u);
                frpar ^= 1u << s;
              }
              used |= 1u << s;
              ptx::tc_fence_after();
              const uint64_t qd = qdesc0 + (uint64_t)(s * (kQTile >> 4));
#pragma unroll
              for (int kk = 0; kk < kD / 16; ++kk)
                ptx::mma_ss(tbase + col_s(s), qd + 2 * kk, kd + 2 * kk, idesc, kk > 0);
              ptx::tc_commit(&sm.s_full[s]);
              if (rho == x.len[s] - 1) ptx::tc_commit(&sm.q_empty[s]);
              if (x.last(s, rho)) {
                ptx::tc_commit(&sm.k_empty[g % kKStages]);
                ++g;
              }
            }
          }
        }
      }
    } else {
      // --------------------------------------------------- P V issuer
      if (ptx::elect_one()) {
        constexpr uint32_t idesc = ptx::idesc_bf16(kBM, kD, 0, 1);
        const uint64_t vdesc0 = ptx::sdesc_sw128(ptx::smem_u32(sm.v[0]));
        uint32_t g = 0;
        uint32_t ppar = 0;  // bit s: parity of the next p_full[s] phase
        uint32_t opar = 0;  // bit s: parity of slot s's completed-unit count (o_empty)
        for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
          const Unit x = make_unit(p, u);
          for (int32_t rho = 0; rho < x.rounds; ++rho) {
            uint64_t vd = 0;
#pragma unroll
            for (int s = 0; s < kSlots; ++s) {
              if (!x.active(s, rho)) continue;
              ptx::mbar_wait(&sm.p_full[s], (ppar >> s) & 1u);
              ppar ^= 1u << s;
              if (rho == 0) ptx::mbar_wait(&sm.o_empty[s], ((opar >> s) & 1u) ^ 1u);
              if (x.lead(s, rho)) {
                const uint32_t st = g % kVStages;
                ptx::mbar_wait(&sm.v_full[st], (g / kVStages) & 1);
                vd = vdesc0 + (uint64_t)(st * (kKVTile >> 4));
              }
              ptx::tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < kBN / 16; ++kk)
                ptx::mma_ts(tbase + col_o(s), tbase + col_s(s) + kk * 8, vd + (uint64_t)(kk * 128), idesc,
                            (rho > 0 || kk > 0) ? 1u : 0u);
              ptx::tc_commit(&sm.pv_done[s]);
              ptx::tc_commit(&sm.s_free[s]);
              if (rho == x.len[s] - 1) {
                ptx::tc_commit(&sm.o_full[s]);
                opar ^= 1u << s;
              }
              if (x.last(s, rho)) {
                ptx::tc_commit(&sm.v_empty[g % kVStages]);
                ++g;
              }
            }
          }
        }
      }
    }
  } else if (warp < 20) {
    // ------------------------------------------------------- softmax
    ptx::setmaxnreg_inc<96>();
    const int s = (warp - 4) / 4;
    const uint32_t row = (warp % 4) * 32 + lane;
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const uint32_t tS = tbase + lane_base + col_s(s), tO = tbase + lane_base + col_o(s);
    uint32_t steps = 0, published = 0;
    for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      const Unit x = make_unit(p, u);
      const int32_t n = x.len[s];
      if (n == 0) continue;
      const int32_t tq = x.t0 + s * kBM + (int32_t)row;
      const bool valid_q = tq < p.T;
      const int32_t seg_lo = valid_q ? p.div_m.div(tq) * p.m : 0;
      const int32_t seg_hi = valid_q ? min(seg_lo + p.m, p.T) : 0;
      const int32_t kbase = x.kv_lo + x.kt0[s] * kBN;
      float mref = -INFINITY, l = 0.0f;
      for (int32_t rho = 0; rho < n; ++rho) {
        ptx::mbar_wait(&sm.s_full[s], steps & 1);
        ptx::tc_fence_after();
        uint32_t sr[2][32];
        ptx::tmem_ld32(tS, sr[0]);
        ptx::tmem_ld32(tS + 32, sr[1]);
        ptx::tmem_ld_wait();
        const int32_t k0 = kbase + rho * kBN;
        const int32_t lo = min(max(seg_lo - k0, 0), kBN), hi = min(max(seg_hi - k0, 0), kBN);
        if (!(lo == 0 && hi == kBN)) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              const int col = 32 * c + e;
              if (col < lo || col >= hi) sr[c][e] = __float_as_uint(-INFINITY);
            }
        }
        float mx[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx[e] = -INFINITY;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e) mx[e & 7] = fmaxf(mx[e & 7], __uint_as_float(sr[c][e]));
        const float tmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                 fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        // Lazy rescale (warp-uniform): a new reference only when the tile max
        // exceeds it by 2^thr; O_s and l are rescaled after the exp pass (sr dead).
        const bool move = tmax > mref && (mref == -INFINITY || (tmax - mref) * p.c > kThr);
        const bool fix_o = move && mref != -INFINITY;
        const float corr = fix_o ? ptx::ex2((mref - tmax) * p.c) : 1.0f;
        if (move) mref = tmax;
        const float neg = (mref == -INFINITY) ? 0.0f : -mref * p.c;
        const float2 c2 = make_float2(p.c, p.c), n2 = make_float2(neg, neg);
        float2 ls2[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
        // 8 pairs (16 columns) at a time keeps the softmax within its 96 registers
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float2 xv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int col = 16 * c + 2 * e;
            xv[e] = ptx::ffma2(make_float2(__uint_as_float(sr[col >> 5][col & 31]),
                                           __uint_as_float(sr[col >> 5][(col & 31) + 1])), c2, n2);
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            if ((kPolyMask >> (8 * (c & 1) + e)) & 1u) {
              xv[e] = ptx::ex2_poly2(xv[e]);
            } else {
              xv[e].x = ptx::ex2(xv[e].x);
              xv[e].y = ptx::ex2(xv[e].y);
            }
          }
          uint32_t pk[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            ls2[e & 1] = ptx::fadd2(ls2[e & 1], xv[e]);
            pk[e] = ptx::pack_bf16x2(xv[e].x, xv[e].y);
          }
          ptx::tmem_st8(tS + 8 * c, pk);
        }
        const float2 lsum = ptx::fadd2(ls2[0], ls2[1]);
        l = fmaf(l, corr, lsum.x + lsum.y);
        // S_s was written after the slot's previous P V completed (s_free), so
        // O_s is final here; the pv_done wait (its latest phase has completed)
        // only makes the ordering explicit.
        if (__any_sync(0xffffffffu, fix_o)) {
          ptx::mbar_wait(&sm.pv_done[s], (steps - 1) & 1);
          ptx::tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            uint32_t orow[32];
            ptx::tmem_ld32(tO + 32 * c, orow);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) orow[e] = __float_as_uint(__uint_as_float(orow[e]) * corr);
            ptx::tmem_st32(tO + 32 * c, orow);
          }
        }
        ++steps;
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&sm.p_full[s]);
      }
      // row statistics to the epilogue, double-buffered by the published count;
      // publish unit n only after the epilogue consumed unit n-1 (see v1)
      sm.stat_l[published & 1][s][row] = l;
      sm.stat_m[published & 1][s][row] = mref;
      if (published > 0) ptx::mbar_wait(&sm.stat_empty[s], (published - 1) & 1);
      ptx::mbar_arrive(&sm.stat_full[s]);
      ++published;
    }
  } else {
    // ------------------------------------------------------ epilogue
    ptx::setmaxnreg_dec<48>();
    const uint32_t row = (warp % 4) * 32 + lane;
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const bool leader = warp == 20 && lane == 0;
    uint32_t par = 0;  // bit s: parity of slot s's completed-unit count
    uint32_t nst = 0;  // tiles stored (staging rotation)
    for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      const Unit x = make_unit(p, u);
#pragma unroll 1
      for (int s = 0; s < kSlots; ++s) {
        if (x.len[s] == 0) continue;
        const int32_t ts0 = x.t0 + s * kBM, tq = ts0 + (int32_t)row;
        const bool valid_q = tq < p.T;
        const uint32_t ph = (par >> s) & 1u;
        par ^= 1u << s;
        uint8_t* stage = sm.ostage[nst & 1];
        ++nst;
        if (leader) ptx::tma_store_wait_read<1>();  // the store issued two tiles ago finished reading `stage`
        ptx::mbar_wait(&sm.o_full[s], ph);
        ptx::mbar_wait(&sm.stat_full[s], ph);
        ptx::tc_fence_after();
        const float l = sm.stat_l[ph][s][row], mref = sm.stat_m[ph][s][row];
        const float inv = valid_q ? 1.0f / l : 0.0f;
        ptx::named_bar_sync(1, kBM);  // staging free (leader's wait) before anyone writes it
        const uint32_t sa = ptx::smem_u32(stage);
        const uint32_t tO = tbase + lane_base + col_o(s);
#pragma unroll 1
        for (int hh = 0; hh < 4; ++hh) {  // 16 columns at a time (48 registers)
          uint32_t orow[16];
          ptx::tmem_ld16(tO + 16 * hh, orow);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int c = 2 * hh + cc;
            const float* f = reinterpret_cast<const float*>(&orow[cc * 8]);
            ptx::st_shared_v4(sa + row * 128 + ((c ^ (row & 7)) * 16), ptx::pack_bf16x2(f[0] * inv, f[1] * inv),
                              ptx::pack_bf16x2(f[2] * inv, f[3] * inv), ptx::pack_bf16x2(f[4] * inv, f[5] * inv),
                              ptx::pack_bf16x2(f[6] * inv, f[7] * inv));
          }
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&sm.stat_empty[s]);  // stats buffer `ph` may be reused
        ptx::mbar_arrive(&sm.o_empty[s]);     // O_s may be overwritten by the next unit
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(1, kBM);
        if (leader) {
          ptx::tma_store_5d(&tm_o, stage, 0, x.j, x.gamma, ts0, x.b);
          for (int32_t gz = 0; gz < p.r; ++gz)
            if (gz != x.gamma) ptx::tma_store_5d(&tm_o, sm.zero, 0, x.j, gz, ts0, x.b);
          ptx::tma_store_commit();
        }
        if (lse && valid_q) {
          float* lb = lse + ((int64_t)x.b * p.h + x.j) * p.N + (int64_t)tq * p.r;
          const float lse_new = mref * p.scale + __logf(l);
          for (int32_t gz = 0; gz < p.r; ++gz) lb[gz] = (gz == x.gamma) ? lse_new : -INFINITY;
        }
      }
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

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// The t'-stream view [B][N/r][r][h][64] of a [B, N, h, *] tensor with token
// stride ld (elements), box (64, 1, 1, rows, 1), 128B swizzle (as v1's make_map).
bool map5(CUtensorMap* map, const void* base, const Geometry& g, int64_t ld, uint32_t rows) {
  static EncodeTiledFn enc = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  if (!enc) return false;
  cuuint64_t dims[5] = {(cuuint64_t)kD, (cuuint64_t)g.h, (cuuint64_t)g.r, (cuuint64_t)(g.N / g.r), (cuuint64_t)g.B};
  cuuint64_t strides[4] = {(cuuint64_t)kD * 2, (cuuint64_t)ld * 2, (cuuint64_t)(g.r * ld * 2),
                           (cuuint64_t)(g.N * ld * 2)};
  cuuint32_t box[5] = {kD, 1, 1, rows, 1}, es[5] = {1, 1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int64_t sm100_v2_units(const Geometry& g) {
  const int64_t T = g.N / g.r;
  return g.B * g.h * ((T + kUnit - 1) / kUnit);
}

int launch_sm100_v2(const Geometry& g, const void* q, const void* k, const void* v, void* o, float* lse,
                    cudaStream_t stream, cudaError_t* err, const char** why) {
  ensure_context();
  CUtensorMap mq, mk, mv, mo;
  if (!map5(&mq, q, g, g.ldq, kBM) || !map5(&mk, k, g, g.ldk, kBN) || !map5(&mv, v, g, g.ldv, kBN) ||
      !map5(&mo, o, g, g.ldo, kBM)) {
    *why = "cuTensorMapEncodeTiled failed (v2)";
    *err = cudaErrorInvalidValue;
    return 0;
  }
  Params p;
  p.N = (int32_t)g.N;
  p.T = (int32_t)(g.N / g.r);
  p.m = (int32_t)(g.w / g.r);
  p.r = (int32_t)g.r;
  p.h = (int32_t)g.h;
  p.n_blocks = (p.T + kUnit - 1) / kUnit;
  p.n_units = (int32_t)(g.B * g.h * p.n_blocks);
  p.scale = g.scale;
  p.c = g.scale * kLog2e;
  p.div_blocks = make_fastdiv((uint32_t)p.n_blocks);
  p.div_h = make_fastdiv((uint32_t)p.h);
  p.div_m = make_fastdiv((uint32_t)p.m);
  for (int i = 0; i < kMaxHeads; ++i) p.offsets[i] = i < g.h ? g.offsets[i] : 0;
  const size_t smem = sizeof(Smem) + 1024;
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [&] {
    attr = cudaFuncSetAttribute(dfa_sm100_v2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (attr != cudaSuccess) {
    *err = attr;
    *why = "cudaFuncSetAttribute failed (v2)";
    return 0;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(p.n_units, sms);
  dfa_sm100_v2_kernel<<<grid, kThreads, smem, stream>>>(mq, mk, mv, mo, lse, p);
  *err = cudaGetLastError();
  return 1;
}

}  // namespace dfa_impl
