// Backward of the Dilated Flash Attention core on sm_100a: TMA + tcgen05 +
// TMEM (bf16 in/out, fp32 accumulate), for segments whose view holds
// m = w / r in {128, 256} rows (r | w, w | N, d = d_v = 64) -- e.g. the
// headline (512, 2) and every m = 256 branch of BASELINE config 4.  Other
// geometries take the SIMT kernels in dfa_bwd.cu.
//
// Math (same as dfa_bwd.cu; the reference's tape for the dilated branch of
// attention_mix, encoder.hpp:204-219): with P = exp(S sc - lse),
// Delta = rowsum(dO o O) (delta_kernel), dS = P o (dP - Delta):
//   dV = P^T dO,  dK = sc dS^T Q,  dQ = sc dS K.
//
// Persistent CTAs (one per SM) loop over units = (image, head, segment); a
// unit's whole view (Q, K, V, dO: m x 64 each) is TMA-loaded once into shared
// memory as 128-row SW128 tiles of the t'-stream (the forward's index
// mapping: no gather), and the next unit's loads are issued as soon as this
// unit's MMAs complete, overlapping its dQ epilogue and output stores.  For key block kb and
// query block qb (128 each), one elected thread issues
//   S^T  = K_kb Q_qb^T            (M=128 keys, N=128 queries)  -> TMEM [0,128)
//   dP^T = V_kb dO_qb^T                                         -> TMEM [128,256)
// two gradient warpgroups (thread = key row = TMEM lane, half the queries each) turn them
// into P^T (bf16 over S^T's columns) and dS^T (bf16 over dP^T's columns, and
// into shared memory as the MN-major A operand of dQ), then
//   dV_kb += P^T dO_qb   (A = P^T from TMEM, B = dO MN-major)   -> TMEM [256,320)
//   dK_kb += dS^T Q_qb   (A = dS^T from TMEM, B = Q MN-major)   -> TMEM [320,384)
//   dQ_qb += dS K_kb     (A = dS from smem, MN-major; B = K MN-major) -> TMEM [384 + 64 qb, ...)
// dK/dV leave after a key block, dQ after the last one: TMEM -> bf16 -> SW128
// staging -> TMA store, plus zero boxes for the rows of the other offset
// classes (their gradient is 0).  Deterministic: no atomics, every output
// element written once.
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
constexpr int kB = 128;                // rows per tile (keys / queries)
constexpr int kTile = 128 * 128;       // 128 rows x 128 B (64 bf16), SW128
constexpr int kMaxBlk = 2;             // m <= 256
constexpr int kThreads = 384;          // warp 0: TMA + MMA, warp 1: TMEM alloc, warps 4-11: gradient WGs
constexpr float kLog2e = 1.4426950408889634f;
#ifndef DFA_BWD_POLY_MASK
#define DFA_BWD_POLY_MASK 0x8080u
#endif
// bit e: pair e of each 16-pair (32-query) chunk of the gradient warpgroups
// takes the FMA-pipe exp2 polynomial (ptx::ex2_poly2) instead of MUFU.EX2
constexpr uint32_t kBwdPolyMask = DFA_BWD_POLY_MASK;
// the m >= 512 pair (dkdv_long / dq_long) keeps more of its exps on the FMA
// pipe: 4 of 16 pairs measured 2.7% faster than 2 of 16 at (1024, 2)
#ifndef DFA_BWD_POLY_MASK_LONG
#define DFA_BWD_POLY_MASK_LONG 0x8888u
#endif
constexpr uint32_t kBwdPolyMaskLong = DFA_BWD_POLY_MASK_LONG;
#ifndef DFA_BWD_LONG_FROM
#define DFA_BWD_LONG_FROM 3  // view blocks (m / 128) from which the dkdv + dq pair replaces the fused kernel
#endif

struct __align__(1024) BwdSmem {
  uint8_t q[kMaxBlk][kTile];
  uint8_t k[kMaxBlk][kTile];
  uint8_t v[kMaxBlk][kTile];
  uint8_t g[kMaxBlk][kTile];      // dO
  uint8_t ds[2][kTile];           // dS^T as the MN-major A operand: queries [0,64) | [64,128)
  uint8_t stage[2][kTile];        // output staging (dK | dV, then dQ blocks)
  uint8_t zero[kTile];
  float lse2[kMaxBlk * kB];       // -lse * log2(e) of the view's query rows
  float dlt[kMaxBlk * kB];        // -Delta of the view's query rows
  uint64_t load_full[kMaxBlk], kv_done, q_done;  // load_full[blk]: Q, K, V, dO of 128-row block blk
  uint64_t s_full[2], p_full[2];                 // per query half: S^T / dP^T ready, P^T / dS^T written
  uint64_t blk0_free;  // two-block views: every MMA reading block 0 (steps up to (1, 0)) completed
  uint32_t tmem_base;
};

struct BwdSm100Params {
  int32_t N, T, m, r, h, n_seg, nblk, n_units;
  int32_t mseg;  // segment view rows when < 128: 128 / mseg segments packed per tile, block-diagonal mask
  float c, scale;
  int32_t offsets[kMaxHeads];
};

__device__ __forceinline__ void wait(uint64_t* bar, uint32_t par) { ptx::mbar_wait(bar, par); }

// kPacked: m < 128, 128 / m segments per tile with the block-diagonal mask --
// a separate instantiation so the common path carries no mask code in its
// inner loop (a runtime test there left one body with per-pair mask
// arithmetic whenever the compiler declined to unswitch it: 12-15% slower)
template <bool kPacked>
__global__ void __launch_bounds__(kThreads, 1)
    dfa_bwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_g,
                         const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dk,
                         const __grid_constant__ CUtensorMap tm_dv, const float* __restrict__ lse,
                         const float* __restrict__ delta, const __grid_constant__ BwdSm100Params p) {
  extern __shared__ uint8_t smem_raw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const int nb = p.nblk;
  const int32_t n_units = p.n_units;
  // unit u = (b * h + j) * n_seg + seg
  struct View {
    int32_t b, j, gamma, t0;
  };
  auto view = [&](int32_t u) {
    View v;
    const int32_t seg = u % p.n_seg, bj = u / p.n_seg;
    v.j = bj % p.h;
    v.b = bj / p.h;
    v.gamma = p.offsets[v.j];
    v.t0 = seg * p.m;  // first t' of the view
    return v;
  };
  // Q, K, V, dO of unit u (the forward's t'-stream boxes) -> smem, one
  // barrier per 128-row block.  Views of one block (m <= 128, nb = 1) leave
  // the second block's tiles free: units alternate between the two (slot
  // `sl`), so the next unit's loads go out while this unit computes.
  auto issue_loads = [&](int32_t u, int sl, int b0 = 0, int b1 = -1) {
    const View x = view(u);
    const uint64_t pol = ptx::policy_evict_first();
    if (b1 < 0) b1 = nb;
    for (int blk = b0; blk < b1; ++blk) {  // block 0 first: the unit's first step needs only it
      const int32_t tb = x.t0 + blk * kB;
      const int t = blk + sl;
      uint64_t* bar = &sm.load_full[t];
      ptx::mbar_arrive_expect_tx(bar, 4 * kTile);
      ptx::tma_load_5d(sm.q[t], &tm_q, bar, 0, x.j, x.gamma, tb, x.b, pol);
      ptx::tma_load_5d(sm.k[t], &tm_k, bar, 0, x.j, x.gamma, tb, x.b, pol);
      ptx::tma_load_5d(sm.v[t], &tm_v, bar, 0, x.j, x.gamma, tb, x.b, pol);
      ptx::tma_load_5d(sm.g[t], &tm_g, bar, 0, x.j, x.gamma, tb, x.b, pol);
    }
  };

  if (warp == 0 && lane == 0) {
    for (int blk = 0; blk < kMaxBlk; ++blk) ptx::mbar_init(&sm.load_full[blk], 1);
    ptx::mbar_init(&sm.blk0_free, 1);
    for (int hf = 0; hf < 2; ++hf) {
      ptx::mbar_init(&sm.s_full[hf], 1);
      ptx::mbar_init(&sm.p_full[hf], kB);
    }
    ptx::mbar_init(&sm.kv_done, 1);
    ptx::mbar_init(&sm.q_done, 1);
    ptx::fence_barrier_init();
    issue_loads(blockIdx.x, 0);  // the first unit's loads go out before anything else
  } else if (warp == 1) {
    ptx::tmem_alloc<512>(&sm.tmem_base);
  }
  for (uint32_t i = threadIdx.x; i < kTile / 16; i += kThreads) ptx::st_shared_v4(ptx::smem_u32(sm.zero) + 16 * i, 0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = sm.tmem_base;
  constexpr uint32_t cS = 0, cDP = 128, cDV = 256, cDK = 320, cDQ = 384;

  if (warp == 0) {
    if (ptx::elect_one()) {
      // ------------------------------------------------------------ MMA
      constexpr uint32_t id_sh = ptx::idesc_bf16(kB, kB / 2, 0, 0);  // S^T, dP^T per query half: K-major A and B
      constexpr uint32_t id_ts = ptx::idesc_bf16(kB, kD, 0, 1);   // dV, dK: A from TMEM, B MN-major
      constexpr uint32_t id_dq = ptx::idesc_bf16(kB, kD, 1, 1);   // dQ: A (dS) MN-major, B (K) MN-major
      const uint64_t dsd = ptx::sdesc_sw128(ptx::smem_u32(sm.ds[0]), 1024, kTile);  // LBO: next 64 queries
      uint32_t step = 0;
      int it = 0;
      // One-block views: operands double-buffered across units.  Measured: -16%
      // at r = 2; at r >= 4 the units are dominated by the zero-box stores and
      // the extra loads in flight cost 2-8%, so they keep the single buffer.
      const bool dbl = nb == 1 && p.r <= 2;
      // Two-block views (r <= 2, same measurement): block 0 of the next unit
      // is loaded as soon as its last reader (step (1, 0)) has completed.
      const bool early0 = nb == 2 && p.r <= 2;
      for (int32_t u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
        const int sl = dbl ? (it & 1) : 0;
        wait(&sm.load_full[sl], dbl ? ((it >> 1) & 1) : (it & 1));
        ptx::tc_fence_after();
        if (dbl && u + (int32_t)gridDim.x < n_units) {
          // the other slot held unit it-1, whose MMAs are done once q_done(it-1) fired
          if (it > 0) wait(&sm.q_done, (it - 1) & 1);
          issue_loads(u + gridDim.x, sl ^ 1);
        }
        for (int kb = 0; kb < nb; ++kb) {
          const uint64_t kd = ptx::sdesc_sw128(ptx::smem_u32(sm.k[kb + sl]));
          const uint64_t vd = ptx::sdesc_sw128(ptx::smem_u32(sm.v[kb + sl]));
          for (int qb = 0; qb < nb; ++qb, ++step) {
            if (kb == 0 && qb == 1) {  // first step touching block 1 (Q1, dO1; K1, V1 follow)
              wait(&sm.load_full[1], it & 1);
              ptx::tc_fence_after();
            }
            const uint64_t qd = ptx::sdesc_sw128(ptx::smem_u32(sm.q[qb + sl]));
            const uint64_t gd = ptx::sdesc_sw128(ptx::smem_u32(sm.g[qb + sl]));
            // S^T / dP^T in two query halves (N = 64; the half's Q / dO rows
            // start 64 x 128 B into the tile): gradient warpgroup hf starts
            // on its half while the other half's products are still running
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
              for (int kk = 0; kk < kD / 16; ++kk) {
                ptx::mma_ss(tbase + cS + 64 * hf, kd + 2 * kk, qd + 512 * hf + 2 * kk, id_sh, kk > 0);
                ptx::mma_ss(tbase + cDP + 64 * hf, vd + 2 * kk, gd + 512 * hf + 2 * kk, id_sh, kk > 0);
              }
              ptx::tc_commit(&sm.s_full[hf]);
            }
            if (early0 && kb == 1 && qb == 1 && u + (int32_t)gridDim.x < n_units) {
              // block 0 of the next unit loads under this unit's last step
              wait(&sm.blk0_free, it & 1);
              issue_loads(u + gridDim.x, 0, 0, 1);
            }
            // dV / dK per half as soon as that warpgroup has written P^T / dS^T
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              wait(&sm.p_full[hf], step & 1);
              ptx::tc_fence_after();
#pragma unroll
              for (int kk = 4 * hf; kk < 4 * hf + 4; ++kk) {
                // K-step of 16 queries: 8 packed TMEM columns of P^T / dS^T, 16 rows (2048 B) of dO / Q
                ptx::mma_ts(tbase + cDV, tbase + cS + 32 * hf + kk * 8, gd + kk * 128, id_ts, (qb > 0 || kk > 0) ? 1u : 0u);
                ptx::mma_ts(tbase + cDK, tbase + cDP + 32 * hf + kk * 8, qd + kk * 128, id_ts, (qb > 0 || kk > 0) ? 1u : 0u);
              }
            }
#pragma unroll
            for (int kk = 0; kk < kB / 16; ++kk)  // K-step of 16 keys: 16 rows of dS / K
              ptx::mma_ss(tbase + cDQ + 64 * qb, dsd + kk * 128, kd + kk * 128, id_dq, (kb > 0 || kk > 0) ? 1u : 0u);
            if (early0 && kb == 1 && qb == 0) ptx::tc_commit(&sm.blk0_free);  // last reader of Q0 / dO0 / K0 / V0
          }
          ptx::tc_commit(&sm.kv_done);
        }
        ptx::tc_commit(&sm.q_done);
        // the unit's operands are free once its MMAs complete: the next
        // unit's loads overlap this unit's dQ epilogue and output stores
        if (!dbl && u + (int32_t)gridDim.x < n_units) {
          wait(&sm.q_done, it & 1);
          issue_loads(u + gridDim.x, 0, early0 ? 1 : 0);  // early0: block 0 went out already
        }
      }
    }
  } else if (warp >= 4) {
    // ----------------------------------------------- gradient warpgroups
    // Two warpgroups share every step: WG0 takes queries [0, 64) of the
    // block, WG1 [64, 128) (thread = key row = TMEM lane in both); in the
    // epilogues WG0 writes dK, WG1 dV, and they alternate the dQ blocks.
    const int wg = (warp - 4) / 4;
    const uint32_t row = ((warp - 4) % 4) * 32 + lane;  // key row (TMEM lane) / query row for dQ
    const uint32_t lane_base = (((warp - 4) % 4) * 32) << 16;
    // packed views: this key row's segment covers queries [seg_lo, seg_lo + seg_len)
    const uint32_t seg_len = (uint32_t)p.mseg, seg_lo = kPacked ? row / seg_len * seg_len : 0u;
    const bool leader = warp % 4 == 0 && lane == 0;
    const uint32_t bar_id = 1 + wg;
    uint32_t step = 0, kvn = 0;
    // The leader's last bulk-store group was zero boxes only (they read the
    // zero tile, not the staging tile): a staging reuse then needs all but
    // that one group to have finished reading.
    bool zeros_last = false;
    auto wait_stage = [&]() {
      if (leader) {
        if (zeros_last) ptx::tma_store_wait_read<1>();
        else ptx::tma_store_wait_read<0>();
      }
    };
    auto stage_store = [&](uint8_t* st, const uint32_t (&v)[2][32], float mul) {
      const uint32_t a0 = ptx::smem_u32(st);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float* f = reinterpret_cast<const float*>(&v[c >> 2][(c & 3) * 8]);
        ptx::st_shared_v4(a0 + row * 128 + ((c ^ (row & 7)) * 16), ptx::pack_bf16x2(f[0] * mul, f[1] * mul),
                          ptx::pack_bf16x2(f[2] * mul, f[3] * mul), ptx::pack_bf16x2(f[4] * mul, f[5] * mul),
                          ptx::pack_bf16x2(f[6] * mul, f[7] * mul));
      }
    };
    // The view's lse (log2 units) and Delta, one query row per thread (nb * 128
    // <= 256 rows): fetched into registers one unit ahead -- the next unit's
    // loads go out after this unit's last step, so their latency hides behind
    // the dK / dV / dQ epilogues -- and copied to shared memory (both
    // warpgroups read all of it) at the start of the unit.
    const int t_row = threadIdx.x - 128;
    float pre_l = 0.0f, pre_d = 0.0f;
    auto fetch_stats = [&](int32_t uu) {
      const View y = view(uu);
      if (t_row < nb * kB) {
        const int64_t n = (int64_t)(y.t0 + t_row) * p.r + y.gamma;
        const int64_t off = ((int64_t)y.b * p.h + y.j) * p.N + n;
        pre_l = lse[off];  // raw: scaled / negated at the smem store, so nothing waits on the load here
        pre_d = delta[off];
      }
    };
    fetch_stats(blockIdx.x);
    int it = 0;
    for (int32_t u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
      const View x = view(u);
      ptx::named_bar_sync(4, 2 * kB);  // previous unit's steps are done with lse2 / dlt
      if (t_row < nb * kB) {
        sm.lse2[t_row] = -pre_l * kLog2e;  // negated: the gradient loop adds them with packed FFMA2 / FADD2
        sm.dlt[t_row] = -pre_d;
      }
      ptx::named_bar_sync(4, 2 * kB);
      for (int kb = 0; kb < nb; ++kb) {
        for (int qb = 0; qb < nb; ++qb, ++step) {
          wait(&sm.s_full[wg], step & 1);
          ptx::tc_fence_after();
          const float* l2 = sm.lse2 + qb * kB;
          const float* dl = sm.dlt + qb * kB;
          const uint32_t dsa = ptx::smem_u32(sm.ds[0]);
#pragma unroll 1
          for (int c = 2 * wg; c < 2 * wg + 2; ++c) {  // 32 queries per chunk
            uint32_t s[32], dp[32];
            ptx::tmem_ld32(tbase + lane_base + cS + 32 * c, s);
            ptx::tmem_ld32(tbase + lane_base + cDP + 32 * c, dp);
            ptx::tmem_ld_wait();
            uint32_t pp[16], dd[16];
            const float2 c2 = make_float2(p.c, p.c);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int q0 = 32 * c + 2 * e;
              // packed pairs: x = s c - lse log2e (FFMA2), dS = P (dP - Delta) (FADD2, FMUL2)
              const float2 nl = *reinterpret_cast<const float2*>(l2 + q0);
              const float2 nd = *reinterpret_cast<const float2*>(dl + q0);
              const float2 x = ptx::ffma2(make_float2(__uint_as_float(s[2 * e]), __uint_as_float(s[2 * e + 1])), c2, nl);
              float2 pr;
              if ((kBwdPolyMask >> e) & 1u) {  // FMA-pipe exp2 for a share of the pairs (MUFU-bound otherwise)
                pr = ptx::ex2_poly2(x);
              } else {
                pr = make_float2(ptx::ex2(x.x), ptx::ex2(x.y));
              }
              if (kPacked) {  // packed short segments: no interaction across segments
                if ((uint32_t)q0 - seg_lo >= seg_len) pr.x = 0.0f;
                if ((uint32_t)q0 + 1u - seg_lo >= seg_len) pr.y = 0.0f;
              }
              const float2 dsv =
                  ptx::fmul2(pr, ptx::fadd2(make_float2(__uint_as_float(dp[2 * e]), __uint_as_float(dp[2 * e + 1])), nd));
              pp[e] = ptx::pack_bf16x2(pr.x, pr.y);
              dd[e] = ptx::pack_bf16x2(dsv.x, dsv.y);
            }
            // Packed P^T / dS^T of chunk c land on the first 32 columns of its
            // own half's fp32 region (chunk 2h + e on 64 h + 16 e): each
            // warpgroup only overwrites scores it has already loaded
            ptx::tmem_st16(tbase + lane_base + cS + 16 * c + 32 * (c >> 1), pp);
            ptx::tmem_st16(tbase + lane_base + cDP + 16 * c + 32 * (c >> 1), dd);
            // dS^T row `row` (key) -> MN-major A of dQ: queries 32c..32c+31 are
            // 16-byte chunks 4(c&1)..4(c&1)+3 of sub-tile c>>1, SW128-swizzled
            const uint32_t sub = dsa + (c >> 1) * kTile + row * 128;
#pragma unroll
            for (int h4 = 0; h4 < 4; ++h4) {
              const uint32_t chunk = 4 * (c & 1) + h4;
              ptx::st_shared_v4(sub + ((chunk ^ (row & 7)) * 16), dd[4 * h4], dd[4 * h4 + 1], dd[4 * h4 + 2],
                                dd[4 * h4 + 3]);
            }
          }
          ptx::tmem_st_wait();
          ptx::fence_proxy_async_smem();
          ptx::tc_fence_before();
          // The first dV / dK product of key block kb > 0 (issued once WG0's
          // half arrives) overwrites the accumulators: WG1 must have read the
          // previous block's dV first (WG0 read dK before this step)
          if (wg == 0 && kb > 0 && qb == 0) ptx::named_bar_sync(5, 2 * kB);
          ptx::mbar_arrive(&sm.p_full[wg]);
        }
        if (kb == nb - 1 && u + (int32_t)gridDim.x < n_units) fetch_stats(u + gridDim.x);  // next unit's stats
        // dK (WG0) / dV (WG1) of key block kb
        wait(&sm.kv_done, kvn & 1);
        ++kvn;
        ptx::tc_fence_after();
        uint32_t a[2][32];
        wait_stage();
        ptx::named_bar_sync(bar_id, 128);
        const uint32_t col = wg == 0 ? cDK : cDV;
        ptx::tmem_ld32(tbase + lane_base + col, a[0]);
        ptx::tmem_ld32(tbase + lane_base + col + 32, a[1]);
        ptx::tmem_ld_wait();
        if (wg == 1 && kb + 1 < nb) ptx::named_bar_arrive(5, 2 * kB);  // dV of block kb is in registers
        stage_store(sm.stage[wg], a, wg == 0 ? p.scale : 1.0f);
        ptx::tc_fence_before();
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(bar_id, 128);
        if (leader) {
          const int32_t tb = x.t0 + kb * kB;
          const CUtensorMap* mo = wg == 0 ? &tm_dk : &tm_dv;
          ptx::tma_store_5d(mo, sm.stage[wg], 0, x.j, x.gamma, tb, x.b);
          ptx::tma_store_commit();  // the staging tile's group
          if (p.r > 1) {
            for (int32_t gz = 0; gz < p.r; ++gz)
              if (gz != x.gamma) {
                ptx::tma_store_5d(mo, sm.zero, 0, x.j, gz, tb, x.b);
                if (wg == 0) ptx::tma_store_5d(&tm_dq, sm.zero, 0, x.j, gz, tb, x.b);
              }
            ptx::tma_store_commit();  // zero boxes
          }
        }
        zeros_last = p.r > 1;
      }
      // dQ blocks (TMEM lanes = query rows), alternating between the warpgroups
      wait(&sm.q_done, it & 1);
      ptx::tc_fence_after();
      for (int qb = wg; qb < nb; qb += 2) {
        uint32_t a[2][32];
        wait_stage();
        ptx::named_bar_sync(bar_id, 128);
        ptx::tmem_ld32(tbase + lane_base + cDQ + 64 * qb, a[0]);
        ptx::tmem_ld32(tbase + lane_base + cDQ + 64 * qb + 32, a[1]);
        ptx::tmem_ld_wait();
        stage_store(sm.stage[wg], a, p.scale);
        ptx::tc_fence_before();
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(bar_id, 128);
        if (leader) {
          ptx::tma_store_5d(&tm_dq, sm.stage[wg], 0, x.j, x.gamma, x.t0 + qb * kB, x.b);
          ptx::tma_store_commit();
        }
        zeros_last = false;
      }
    }
    if (leader) ptx::tma_store_wait_all<0>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tbase);
  }
}

// ============================================================================
// Long segments (m = w / r >= 512, m % 128 == 0): the accumulators of a whole
// view no longer fit TMEM next to S / dP, so the backward splits FA2-style
// into two tcgen05 kernels, each deterministic:
//   dkdv_long: unit = (b, j, segment, key block kb); K_kb, V_kb resident, the
//              view's (Q, dO) blocks streamed through a 2-stage ring;
//              S^T, dP^T -> P^T, dS^T (TMEM, bf16) -> dV += P^T dO, dK += dS^T Q.
//   dq_long:   unit = (b, j, segment, query block qb); Q_qb, dO_qb resident,
//              (K, V) blocks streamed; S = Q K^T, dP = dO V^T (lanes = queries,
//              so lse / Delta are per-thread scalars) -> dS (TMEM, bf16) ->
//              dQ += dS K.
// 7 GEMM-shaped products per (kb, qb) pair instead of the fused kernel's 5.
struct LongParams {
  int32_t N, m, r, h, n_seg, nblk, n_units;
  float c, scale;
  int32_t offsets[kMaxHeads];
};

struct LongView {
  int32_t b, j, gamma, t0, blk;  // t0: first t' of the view; blk: kb or qb
};
__device__ __forceinline__ LongView long_view(const LongParams& p, int32_t u) {
  LongView v;
  v.blk = u % p.nblk;
  const int32_t rest = u / p.nblk;
  const int32_t seg = rest % p.n_seg, bj = rest / p.n_seg;
  v.j = bj % p.h;
  v.b = bj / p.h;
  v.gamma = p.offsets[v.j];
  v.t0 = seg * p.m;
  return v;
}

struct __align__(1024) DkdvSmem {
  uint8_t k[kTile], v[kTile];
  uint8_t q[2][kTile], g[2][kTile];  // (Q, dO) ring
  uint8_t stage[2][kTile];
  uint8_t zero[kTile];
  float lse2[2][kB], dlt[2][kB];     // per step, double-buffered (prefetched one step ahead)
  uint64_t kv_full, kv_done, ring_full[2], ring_empty[2], s_full, p_full;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kThreads, 1)
    dfa_bwd_dkdv_long_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_g,
                             const __grid_constant__ CUtensorMap tm_dk, const __grid_constant__ CUtensorMap tm_dv,
                             const float* __restrict__ lse, const float* __restrict__ delta,
                             const __grid_constant__ LongParams p) {
  extern __shared__ uint8_t smem_raw[];
  DkdvSmem& sm = *reinterpret_cast<DkdvSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const int nq = p.nblk;
  if (warp == 0 && lane == 0) {
    ptx::mbar_init(&sm.kv_full, 1);
    ptx::mbar_init(&sm.kv_done, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&sm.ring_full[i], 1);
      ptx::mbar_init(&sm.ring_empty[i], 1);
    }
    ptx::mbar_init(&sm.s_full, 1);
    ptx::mbar_init(&sm.p_full, 2 * kB);
    ptx::fence_barrier_init();
  } else if (warp == 1) {
    ptx::tmem_alloc<512>(&sm.tmem_base);
  }
  for (uint32_t i = threadIdx.x; i < kTile / 16; i += kThreads) ptx::st_shared_v4(ptx::smem_u32(sm.zero) + 16 * i, 0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = sm.tmem_base;
  constexpr uint32_t cS = 0, cDP = 128, cDV = 256, cDK = 320;

  if (warp == 3) {
    // ------------------------------------------------------- TMA producer
    if (ptx::elect_one()) {
      const uint64_t pol = ptx::policy_evict_first();
      uint32_t gstep = 0;
      int it = 0;
      for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
        const LongView x = long_view(p, u);
        if (it > 0) wait(&sm.kv_done, (it - 1) & 1);  // previous unit's MMAs finished with K / V
        ptx::mbar_arrive_expect_tx(&sm.kv_full, 2 * kTile);
        const int32_t tk = x.t0 + x.blk * kB;
        ptx::tma_load_5d(sm.k, &tm_k, &sm.kv_full, 0, x.j, x.gamma, tk, x.b, pol);
        ptx::tma_load_5d(sm.v, &tm_v, &sm.kv_full, 0, x.j, x.gamma, tk, x.b, pol);
        for (int qb = 0; qb < nq; ++qb, ++gstep) {
          const uint32_t st = gstep & 1;
          wait(&sm.ring_empty[st], ((gstep >> 1) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&sm.ring_full[st], 2 * kTile);
          const int32_t tq = x.t0 + qb * kB;
          ptx::tma_load_5d(sm.q[st], &tm_q, &sm.ring_full[st], 0, x.j, x.gamma, tq, x.b, pol);
          ptx::tma_load_5d(sm.g[st], &tm_g, &sm.ring_full[st], 0, x.j, x.gamma, tq, x.b, pol);
        }
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------- MMA
    if (ptx::elect_one()) {
      constexpr uint32_t id_ss = ptx::idesc_bf16(kB, kB, 0, 0);
      constexpr uint32_t id_ts = ptx::idesc_bf16(kB, kD, 0, 1);
      const uint64_t kd = ptx::sdesc_sw128(ptx::smem_u32(sm.k));
      const uint64_t vd = ptx::sdesc_sw128(ptx::smem_u32(sm.v));
      uint32_t step = 0;
      int it = 0;
      for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
        wait(&sm.kv_full, it & 1);
        ptx::tc_fence_after();
        for (int qb = 0; qb < nq; ++qb, ++step) {
          const uint32_t st = step & 1;
          wait(&sm.ring_full[st], (step >> 1) & 1);
          ptx::tc_fence_after();
          const uint64_t qd = ptx::sdesc_sw128(ptx::smem_u32(sm.q[st]));
          const uint64_t gd = ptx::sdesc_sw128(ptx::smem_u32(sm.g[st]));
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk) {
            ptx::mma_ss(tbase + cS, kd + 2 * kk, qd + 2 * kk, id_ss, kk > 0);
            ptx::mma_ss(tbase + cDP, vd + 2 * kk, gd + 2 * kk, id_ss, kk > 0);
          }
          ptx::tc_commit(&sm.s_full);
          wait(&sm.p_full, step & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kB / 16; ++kk) {
            ptx::mma_ts(tbase + cDV, tbase + cS + kk * 8, gd + kk * 128, id_ts, (qb > 0 || kk > 0) ? 1u : 0u);
            ptx::mma_ts(tbase + cDK, tbase + cDP + kk * 8, qd + kk * 128, id_ts, (qb > 0 || kk > 0) ? 1u : 0u);
          }
          ptx::tc_commit(&sm.ring_empty[st]);
        }
        ptx::tc_commit(&sm.kv_done);
      }
    }
  } else if (warp >= 4) {
    // ----------------------------------------------- gradient warpgroups
    const int wg = (warp - 4) / 4;
    const uint32_t row = ((warp - 4) % 4) * 32 + lane;
    const uint32_t lane_base = (((warp - 4) % 4) * 32) << 16;
    const bool leader = warp % 4 == 0 && lane == 0;
    const int t = threadIdx.x - 128;  // 0..255: entry t % 128 of lse (t < 128) or Delta
    // this CTA's step sequence: (unit it, qb) -> lse / Delta of query block qb
    auto fetch = [&](int32_t u, int qb) -> float {
      const LongView x = long_view(p, u);
      const int64_t n = (int64_t)(x.t0 + qb * kB + (t & 127)) * p.r + x.gamma;
      const int64_t base = ((int64_t)x.b * p.h + x.j) * p.N;
      return t < 128 ? -lse[base + n] * kLog2e : -delta[base + n];  // negated for packed FFMA2 / FADD2
    };
    auto put = [&](int buf, float val) {
      if (t < 128) sm.lse2[buf][t] = val;
      else sm.dlt[buf][t - 128] = val;
    };
    if ((int32_t)blockIdx.x < p.n_units) put(0, fetch(blockIdx.x, 0));
    ptx::named_bar_sync(4, 2 * kB);
    uint32_t step = 0;
    int it = 0;
    for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
      const LongView x = long_view(p, u);
      for (int qb = 0; qb < nq; ++qb, ++step) {
        // prefetch the next step's lse / Delta (stored after this step's work)
        int32_t nu = u;
        int nqb = qb + 1;
        if (nqb == nq) {
          nqb = 0;
          nu = u + gridDim.x;
        }
        const bool has_next = nu < p.n_units;
        const float nxt = has_next ? fetch(nu, nqb) : 0.0f;
        const int buf = step & 1;
        wait(&sm.s_full, step & 1);
        ptx::tc_fence_after();
#pragma unroll 1
        for (int c = 2 * wg; c < 2 * wg + 2; ++c) {
          uint32_t sv[32], dp[32];
          ptx::tmem_ld32(tbase + lane_base + cS + 32 * c, sv);
          ptx::tmem_ld32(tbase + lane_base + cDP + 32 * c, dp);
          ptx::tmem_ld_wait();
          if (c == 1) ptx::named_bar_arrive(3, 2 * kB);  // see dfa_bwd_sm100_kernel
          uint32_t pp[16], dd[16];
          const float2 c2 = make_float2(p.c, p.c);
#pragma unroll
          for (int e = 0; e < 16; ++e) {  // packed pairs, as dfa_bwd_sm100_kernel
            const int q0 = 32 * c + 2 * e;
            const float2 nl = *reinterpret_cast<const float2*>(&sm.lse2[buf][q0]);
            const float2 nd = *reinterpret_cast<const float2*>(&sm.dlt[buf][q0]);
            const float2 x =
                ptx::ffma2(make_float2(__uint_as_float(sv[2 * e]), __uint_as_float(sv[2 * e + 1])), c2, nl);
            const float2 pr = ((kBwdPolyMaskLong >> e) & 1u) ? ptx::ex2_poly2(x) : make_float2(ptx::ex2(x.x), ptx::ex2(x.y));
            const float2 dsv =
                ptx::fmul2(pr, ptx::fadd2(make_float2(__uint_as_float(dp[2 * e]), __uint_as_float(dp[2 * e + 1])), nd));
            pp[e] = ptx::pack_bf16x2(pr.x, pr.y);
            dd[e] = ptx::pack_bf16x2(dsv.x, dsv.y);
          }
          if (c == 2) ptx::named_bar_sync(3, 2 * kB);
          ptx::tmem_st16(tbase + lane_base + cS + 16 * c, pp);
          ptx::tmem_st16(tbase + lane_base + cDP + 16 * c, dd);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&sm.p_full);
        if (has_next) put(buf ^ 1, nxt);
        ptx::named_bar_sync(4, 2 * kB);
      }
      // dK (WG0, scaled) / dV (WG1) of this key block, + zero boxes of the other classes
      wait(&sm.kv_done, it & 1);
      ptx::tc_fence_after();
      uint32_t a[2][32];
      if (leader) ptx::tma_store_wait_read<0>();
      ptx::named_bar_sync(1 + wg, 128);
      const uint32_t col = wg == 0 ? cDK : cDV;
      ptx::tmem_ld32(tbase + lane_base + col, a[0]);
      ptx::tmem_ld32(tbase + lane_base + col + 32, a[1]);
      ptx::tmem_ld_wait();
      const float mul = wg == 0 ? p.scale : 1.0f;
      const uint32_t a0 = ptx::smem_u32(sm.stage[wg]);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float* f = reinterpret_cast<const float*>(&a[c >> 2][(c & 3) * 8]);
        ptx::st_shared_v4(a0 + row * 128 + ((c ^ (row & 7)) * 16), ptx::pack_bf16x2(f[0] * mul, f[1] * mul),
                          ptx::pack_bf16x2(f[2] * mul, f[3] * mul), ptx::pack_bf16x2(f[4] * mul, f[5] * mul),
                          ptx::pack_bf16x2(f[6] * mul, f[7] * mul));
      }
      ptx::tc_fence_before();
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(1 + wg, 128);
      if (leader) {
        const int32_t tk = x.t0 + x.blk * kB;
        const CUtensorMap* mo = wg == 0 ? &tm_dk : &tm_dv;
        ptx::tma_store_5d(mo, sm.stage[wg], 0, x.j, x.gamma, tk, x.b);
        for (int32_t gz = 0; gz < p.r; ++gz)
          if (gz != x.gamma) ptx::tma_store_5d(mo, sm.zero, 0, x.j, gz, tk, x.b);
        ptx::tma_store_commit();
      }
    }
    if (leader) ptx::tma_store_wait_all<0>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tbase);
  }
}

struct __align__(1024) DqSmem {
  uint8_t q[kTile], g[kTile];
  uint8_t k[2][kTile], v[2][kTile];  // (K, V) ring
  uint8_t stage[kTile];
  uint8_t zero[kTile];
  uint64_t qg_full, q_done, ring_full[2], ring_empty[2], s_full, p_full;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kThreads, 1)
    dfa_bwd_dq_long_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_g,
                           const __grid_constant__ CUtensorMap tm_dq, const float* __restrict__ lse,
                           const float* __restrict__ delta, const __grid_constant__ LongParams p) {
  extern __shared__ uint8_t smem_raw[];
  DqSmem& sm = *reinterpret_cast<DqSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const int nk = p.nblk;
  if (warp == 0 && lane == 0) {
    ptx::mbar_init(&sm.qg_full, 1);
    ptx::mbar_init(&sm.q_done, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&sm.ring_full[i], 1);
      ptx::mbar_init(&sm.ring_empty[i], 1);
    }
    ptx::mbar_init(&sm.s_full, 1);
    ptx::mbar_init(&sm.p_full, 2 * kB);
    ptx::fence_barrier_init();
  } else if (warp == 1) {
    ptx::tmem_alloc<512>(&sm.tmem_base);
  }
  for (uint32_t i = threadIdx.x; i < kTile / 16; i += kThreads) ptx::st_shared_v4(ptx::smem_u32(sm.zero) + 16 * i, 0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = sm.tmem_base;
  constexpr uint32_t cS = 0, cDP = 128, cDQ = 256;

  if (warp == 3) {
    if (ptx::elect_one()) {
      const uint64_t pol = ptx::policy_evict_first();
      uint32_t gstep = 0;
      int it = 0;
      for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
        const LongView x = long_view(p, u);
        if (it > 0) wait(&sm.q_done, (it - 1) & 1);  // previous unit's MMAs finished with Q / dO
        ptx::mbar_arrive_expect_tx(&sm.qg_full, 2 * kTile);
        const int32_t tq = x.t0 + x.blk * kB;
        ptx::tma_load_5d(sm.q, &tm_q, &sm.qg_full, 0, x.j, x.gamma, tq, x.b, pol);
        ptx::tma_load_5d(sm.g, &tm_g, &sm.qg_full, 0, x.j, x.gamma, tq, x.b, pol);
        for (int kb = 0; kb < nk; ++kb, ++gstep) {
          const uint32_t st = gstep & 1;
          wait(&sm.ring_empty[st], ((gstep >> 1) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&sm.ring_full[st], 2 * kTile);
          const int32_t tk = x.t0 + kb * kB;
          ptx::tma_load_5d(sm.k[st], &tm_k, &sm.ring_full[st], 0, x.j, x.gamma, tk, x.b, pol);
          ptx::tma_load_5d(sm.v[st], &tm_v, &sm.ring_full[st], 0, x.j, x.gamma, tk, x.b, pol);
        }
      }
    }
  } else if (warp == 0) {
    if (ptx::elect_one()) {
      constexpr uint32_t id_ss = ptx::idesc_bf16(kB, kB, 0, 0);  // S = Q K^T, dP = dO V^T (K-major)
      constexpr uint32_t id_ts = ptx::idesc_bf16(kB, kD, 0, 1);  // dQ += dS K (A TMEM, B = K MN-major)
      const uint64_t qd = ptx::sdesc_sw128(ptx::smem_u32(sm.q));
      const uint64_t gd = ptx::sdesc_sw128(ptx::smem_u32(sm.g));
      uint32_t step = 0;
      int it = 0;
      for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
        wait(&sm.qg_full, it & 1);
        ptx::tc_fence_after();
        for (int kb = 0; kb < nk; ++kb, ++step) {
          const uint32_t st = step & 1;
          wait(&sm.ring_full[st], (step >> 1) & 1);
          ptx::tc_fence_after();
          const uint64_t kd = ptx::sdesc_sw128(ptx::smem_u32(sm.k[st]));
          const uint64_t vd = ptx::sdesc_sw128(ptx::smem_u32(sm.v[st]));
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk) {
            ptx::mma_ss(tbase + cS, qd + 2 * kk, kd + 2 * kk, id_ss, kk > 0);
            ptx::mma_ss(tbase + cDP, gd + 2 * kk, vd + 2 * kk, id_ss, kk > 0);
          }
          ptx::tc_commit(&sm.s_full);
          wait(&sm.p_full, step & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kB / 16; ++kk)  // K-step of 16 keys: 8 packed dS columns, 16 rows of K
            ptx::mma_ts(tbase + cDQ, tbase + cDP + kk * 8, kd + kk * 128, id_ts, (kb > 0 || kk > 0) ? 1u : 0u);
          ptx::tc_commit(&sm.ring_empty[st]);
        }
        ptx::tc_commit(&sm.q_done);
      }
    }
  } else if (warp >= 4) {
    const int wg = (warp - 4) / 4;
    const uint32_t row = ((warp - 4) % 4) * 32 + lane;  // query row (TMEM lane)
    const uint32_t lane_base = (((warp - 4) % 4) * 32) << 16;
    const bool leader = warp == 4 && lane == 0;
    uint32_t step = 0;
    int it = 0;
    for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++it) {
      const LongView x = long_view(p, u);
      const int32_t tq = x.t0 + x.blk * kB;
      const int64_t n = (int64_t)(tq + row) * p.r + x.gamma;
      const int64_t base = ((int64_t)x.b * p.h + x.j) * p.N;
      const float l2 = lse[base + n] * kLog2e, dl = delta[base + n];
      for (int kb = 0; kb < nk; ++kb, ++step) {
        wait(&sm.s_full, step & 1);
        ptx::tc_fence_after();
#pragma unroll  // both chunks: the second's TMEM loads overlap the first's math (-1-3%)
        for (int c = 2 * wg; c < 2 * wg + 2; ++c) {
          uint32_t sv[32], dp[32];
          ptx::tmem_ld32(tbase + lane_base + cS + 32 * c, sv);
          ptx::tmem_ld32(tbase + lane_base + cDP + 32 * c, dp);
          ptx::tmem_ld_wait();
          if (c == 1) ptx::named_bar_arrive(3, 2 * kB);
          uint32_t dd[16];
          const float2 c2 = make_float2(p.c, p.c), nl = make_float2(-l2, -l2), nd = make_float2(-dl, -dl);
#pragma unroll
          for (int e = 0; e < 16; ++e) {  // packed pairs, as dfa_bwd_sm100_kernel
            const float2 x =
                ptx::ffma2(make_float2(__uint_as_float(sv[2 * e]), __uint_as_float(sv[2 * e + 1])), c2, nl);
            const float2 pr = ((kBwdPolyMaskLong >> e) & 1u) ? ptx::ex2_poly2(x) : make_float2(ptx::ex2(x.x), ptx::ex2(x.y));
            const float2 dsv =
                ptx::fmul2(pr, ptx::fadd2(make_float2(__uint_as_float(dp[2 * e]), __uint_as_float(dp[2 * e + 1])), nd));
            dd[e] = ptx::pack_bf16x2(dsv.x, dsv.y);
          }
          if (c == 2) ptx::named_bar_sync(3, 2 * kB);
          ptx::tmem_st16(tbase + lane_base + cDP + 16 * c, dd);
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&sm.p_full);
      }
      if (wg == 0) {  // dQ of this query block (scaled) + zero boxes of the other classes
        wait(&sm.q_done, it & 1);
        ptx::tc_fence_after();
        uint32_t a[2][32];
        if (leader) ptx::tma_store_wait_read<0>();
        ptx::named_bar_sync(1, 128);
        ptx::tmem_ld32(tbase + lane_base + cDQ, a[0]);
        ptx::tmem_ld32(tbase + lane_base + cDQ + 32, a[1]);
        ptx::tmem_ld_wait();
        const uint32_t a0 = ptx::smem_u32(sm.stage);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float* f = reinterpret_cast<const float*>(&a[c >> 2][(c & 3) * 8]);
          ptx::st_shared_v4(a0 + row * 128 + ((c ^ (row & 7)) * 16), ptx::pack_bf16x2(f[0] * p.scale, f[1] * p.scale),
                            ptx::pack_bf16x2(f[2] * p.scale, f[3] * p.scale),
                            ptx::pack_bf16x2(f[4] * p.scale, f[5] * p.scale),
                            ptx::pack_bf16x2(f[6] * p.scale, f[7] * p.scale));
        }
        ptx::tc_fence_before();
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(1, 128);
        if (leader) {
          ptx::tma_store_5d(&tm_dq, sm.stage, 0, x.j, x.gamma, tq, x.b);
          for (int32_t gz = 0; gz < p.r; ++gz)
            if (gz != x.gamma) ptx::tma_store_5d(&tm_dq, sm.zero, 0, x.j, gz, tq, x.b);
          ptx::tma_store_commit();
        }
      }
    }
    if (leader) ptx::tma_store_wait_all<0>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tbase);
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

// The forward's t'-stream view [B][N/r][r][h][64], box (64, 1, 1, 128, 1), SW128.
bool map5(CUtensorMap* map, const void* base, const Geometry& g) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const int64_t ld = g.h * kD;
  cuuint64_t dims[5] = {(cuuint64_t)kD, (cuuint64_t)g.h, (cuuint64_t)g.r, (cuuint64_t)(g.N / g.r), (cuuint64_t)g.B};
  cuuint64_t strides[4] = {(cuuint64_t)kD * 2, (cuuint64_t)ld * 2, (cuuint64_t)(g.r * ld * 2),
                           (cuuint64_t)(g.N * ld * 2)};
  cuuint32_t box[5] = {kD, 1, 1, 128, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool bwd_sm100_supported(const Geometry& g, int dtype, const void* const* ptrs, int n_ptrs) {
  if (dtype != 1 || g.d != kD || g.dv != kD) return false;
  if (g.N % g.w != 0 || g.w % g.r != 0) return false;
  const int64_t m = g.w / g.r;
  // 128, 256: fused kernel; >= 512: the dkdv_long + dq_long pair; 16..64
  // (dividing 128): fused kernel on 128-row tiles of packed segments
  const bool packed = m < 128 && 128 % m == 0 && m >= 16 && (g.N / g.r) % 128 == 0;
  if (m % 128 != 0 && !packed) return false;
  if (g.h > kMaxHeads || g.N > (int64_t)INT32_MAX / 2 || g.B * g.h * (g.N / g.w) > (int64_t)INT32_MAX) return false;
  for (int i = 0; i < n_ptrs; ++i)
    if (reinterpret_cast<uintptr_t>(ptrs[i]) & 15u) return false;
  return true;
}

int launch_bwd_sm100(const Geometry& g, const void* q, const void* k, const void* v, const void* dout,
                     const float* lse, const float* delta, void* dq, void* dk, void* dv, cudaStream_t stream,
                     cudaError_t* err, const char** why) {
  ensure_context();
  CUtensorMap mq, mk, mv, mg, mdq, mdk, mdv;
  if (!map5(&mq, q, g) || !map5(&mk, k, g) || !map5(&mv, v, g) || !map5(&mg, dout, g) || !map5(&mdq, dq, g) ||
      !map5(&mdk, dk, g) || !map5(&mdv, dv, g)) {
    *why = "cuTensorMapEncodeTiled failed";
    *err = cudaErrorInvalidValue;
    return 0;
  }
  BwdSm100Params p;
  p.N = (int32_t)g.N;
  p.T = (int32_t)(g.N / g.r);
  p.m = (int32_t)(g.w / g.r);
  p.mseg = p.m;
  if (p.m < kB) p.m = kB;  // packed: a "view" is 128 t'-rows holding 128 / mseg segments
  p.r = (int32_t)g.r;
  p.h = (int32_t)g.h;
  p.n_seg = (int32_t)((g.N / g.r) / p.m);  // units of p.m t'-rows per (b, j) stream
  p.nblk = p.m / kB;
  p.n_units = (int32_t)(g.B * g.h * p.n_seg);
  p.scale = g.scale;
  p.c = g.scale * kLog2e;
  for (int i = 0; i < kMaxHeads; ++i) p.offsets[i] = i < g.h ? g.offsets[i] : 0;
  const int sms = device_sms();
  if (p.nblk > kMaxBlk || p.nblk >= DFA_BWD_LONG_FROM) {
    LongParams lp;
    lp.N = p.N;
    lp.m = p.m;
    lp.r = p.r;
    lp.h = p.h;
    lp.n_seg = p.n_seg;
    lp.nblk = p.nblk;
    lp.n_units = (int32_t)(g.B * g.h * p.n_seg * p.nblk);
    lp.c = p.c;
    lp.scale = p.scale;
    for (int i = 0; i < kMaxHeads; ++i) lp.offsets[i] = p.offsets[i];
    const size_t s1 = sizeof(DkdvSmem) + 1024, s2 = sizeof(DqSmem) + 1024;
    cudaError_t attr_l = ensure_smem_attr(reinterpret_cast<const void*>(dfa_bwd_dkdv_long_kernel), s1);
    if (attr_l == cudaSuccess) attr_l = ensure_smem_attr(reinterpret_cast<const void*>(dfa_bwd_dq_long_kernel), s2);
    if (attr_l != cudaSuccess) {
      *err = attr_l;
      *why = "cudaFuncSetAttribute failed";
      return 0;
    }
    const unsigned grid = (unsigned)std::min<int64_t>(lp.n_units, sms);
    dfa_bwd_dkdv_long_kernel<<<grid, kThreads, s1, stream>>>(mq, mk, mv, mg, mdk, mdv, lse, delta, lp);
    dfa_bwd_dq_long_kernel<<<grid, kThreads, s2, stream>>>(mq, mk, mv, mg, mdq, lse, delta, lp);
    *err = cudaGetLastError();
    return 2;
  }
  const size_t smem = sizeof(BwdSmem) + 1024;
  const bool packed = p.mseg < kB;
  const void* kfn = packed ? reinterpret_cast<const void*>(dfa_bwd_sm100_kernel<true>)
                           : reinterpret_cast<const void*>(dfa_bwd_sm100_kernel<false>);
  const cudaError_t attr = ensure_smem_attr(kfn, smem);
  if (attr != cudaSuccess) {
    *err = attr;
    *why = "cudaFuncSetAttribute failed";
    return 0;
  }
  const unsigned grid = (unsigned)std::min<int64_t>(p.n_units, sms);  // persistent: one CTA per SM
  if (packed) dfa_bwd_sm100_kernel<true><<<grid, kThreads, smem, stream>>>(mq, mk, mv, mg, mdq, mdk, mdv, lse, delta, p);
  else dfa_bwd_sm100_kernel<false><<<grid, kThreads, smem, stream>>>(mq, mk, mv, mg, mdq, mdk, mdv, lse, delta, p);
  *err = cudaGetLastError();
  return 1;
}

}  // namespace dfa_impl
