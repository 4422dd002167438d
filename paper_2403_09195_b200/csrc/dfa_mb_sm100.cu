// Fused multi-(w, r) Dilated Flash Attention forward for sm_100a: every
// branch of a LongNet-style set and their LSE-weighted combine in ONE
// persistent tcgen05 kernel, with the output written once.
//
// Extension (the reference has a single (w, r) per call; SPEC.md:204 lists
// multi-(w, r) as a non-goal).  Semantics = oracle_multibranch_f64
// (oracle/dfa_oracle.c): for every query row the keys of every branch whose
// view contains the row (attention.hpp:84-98 per branch), one softmax over
// that multiset.  Algebraically O = sum_b e^{lse_b} O_b / sum_b e^{lse_b},
// i.e. the north_star's "fused epilogue that weights branches by their
// log-sum-exp denominators" -- computed here as ONE online softmax per row
// that simply continues across the branches' key tiles, so no per-branch
// normalised output, no intermediate rounding and no combine pass exist.
//
// Layout.  R = lcm of the branch intervals (every r_b | R, R | N); the
// [B, N, h, 64] tensors are viewed as [B][N/R][R][h][64] ("R-stream": row
// n = R t + c sits at (t, class c)).  A query tile = 128 rows made of G
// class groups of gr = 128/G rows: group g holds class c + g R/G at
// t in [t0, t0 + gr) of the R-stream -- G TMA boxes of gr rows.  All rows of
// a group have the same n mod r_b for every branch, so a branch either
// selects a whole group or none of it; with G > 1 a tile spans
// L = gr R < 128 R original rows, which keeps the short-segment branches
// (w < 128 R) from paying for keys outside their segment.  Key tiles are
// 128-row boxes of the branch's own r_b-stream (as in dfa_sm100.cu).
//
// Schedule (host, build_plan): each work unit = head j + two query tiles
// (slots A / B, paired for equal step counts and shared key tiles) + an
// ordered list of key tiles, each tagged (branch, t', slot mask).  A key
// tile used by both slots is loaded once.  Units are replicated over the
// batch into one list, most expensive first, which the persistent CTAs
// claim dynamically (global counter, handed to the roles through a
// shared-memory ring), so the mixed unit costs of a branch set balance.
//
// Warp roles, TMEM (3 S buffers + O_A, O_B), barriers and the softmax are
// those of dfa_sm100_kernel; what changes is that every role walks the
// unit's key-tile list, the softmax derives each row's segment per branch,
// and rows no branch selects come out as exact zeros (epilogue: 1/l -> 0).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <mutex>
#include <numeric>
#include <queue>
#include <vector>

#include "dfa_internal.h"
#include "sm100_ptx.cuh"

namespace dfa_impl {
namespace {

constexpr int kD = 64;
constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kSC = kBN / 32;
constexpr int kTileBytes = 128 * 128;
constexpr int kQStages = 2, kKStages = 3, kVStages = 3, kOStages = 2;
constexpr int kThreads = 512;
constexpr uint32_t kTmemCols = 512;
constexpr int kSBufs = 3;
// Dynamic scheduling: the producer claims work units from a global counter
// (most expensive first) and hands each to the other roles through a
// shared-memory ring that also holds the unit's descriptor (bulk-copied from
// global memory, so no role waits on an L2 round trip per unit or reads the
// key-tile list from global memory per step).  A role frees its slot when it
// takes the next unit; consumers = Q K^T issuer, P V issuer, V producer, 8
// softmax warps and 4 epilogue warps.
constexpr int kSchedDepth = 6;
constexpr uint32_t kSchedConsumers = 15;
__host__ __device__ constexpr uint32_t col_s(int buf) { return (uint32_t)kBN * buf; }
__host__ __device__ constexpr uint32_t col_o(int slot) { return 384u + 64u * slot; }
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;
constexpr float kSumBound = 256.0f;  // sum-checked fast path: p <= sum <= 2^8 keeps the lazy-rescale bound
#ifndef DFA_MB_SUMCHECK
#define DFA_MB_SUMCHECK -1  // -1: by geometry (launch_mb_sm100), 0: never, 1: always
#endif
constexpr uint32_t kPolyMask = 0x0888u;  // as dfa_sm100.cu (3 of 16 pairs on the FMA pipe)
constexpr uint32_t kPolyMaskSumCheck = 0x0808u;  // sum-checked instantiation: 2 of 16 (-2% on {(2048, 2), (4096, 4)})

struct FastDivMb {
  uint32_t d, mul, shift;
  __device__ __forceinline__ int32_t div(int32_t n) const {
    return (int32_t)((__umulhi((uint32_t)n, mul) + (uint32_t)n) >> shift);
  }
};
FastDivMb make_fastdiv_mb(uint32_t d) {
  FastDivMb f;
  f.d = d;
  uint32_t shift = 0;
  while ((1ull << shift) < d) ++shift;
  f.shift = shift;
  f.mul = (uint32_t)((((1ull << 32) * ((1ull << shift) - d)) / d) + 1);
  if (d == 1) f.mul = 0;
  return f;
}

// One work unit (replicated over the batch).  tile[i] = t' (bits 0-23, in
// the branch's r-stream) | branch (bits 24-26) | slot mask (bits 28-29).
struct alignas(16) MbDesc {  // sizeof % 16 == 0: bulk-copied into shared memory
  int32_t j;
  int32_t n_tiles;
  int32_t steps;                      // sum of the tiles' slot counts
  int32_t qt[2];                      // R-stream t' of the slot's rows; -1: slot absent
  int32_t first[2], last[2];          // first / last key tile of slot s (-1: slot has no steps)
  int16_t cls[2][kMbMaxGroups];       // class of group g of slot s (< R <= 1024)
  uint8_t sel[2][kMaxBranches];       // bit g: group g of slot s selected by branch b
  uint8_t anysel[2];                  // bit g: group g selected by some branch
  uint8_t pad[2];
  int32_t gamma[kMaxBranches];        // offset of head j in branch b
  uint32_t tile[kMbMaxTiles];
  // the softmax's view: slot s's steps in order, t' (bits 0-19) | branch
  // (20-22) | step index within the unit (23-30)
  int32_t sn[2];
  uint32_t sstep[2][kMbMaxTiles];
};

static_assert(sizeof(MbDesc) % 16 == 0, "bulk copy size");

struct MbParams {
  int32_t N, h, R, TR;     // TR = N / R
  int32_t gr_shift;        // log2(rows per class group)
  float c, scale;
  int32_t br_m[kMaxBranches], br_T[kMaxBranches], br_map[kMaxBranches];
  FastDivMb br_divr[kMaxBranches], br_divm[kMaxBranches];
  const MbDesc* desc;
  const int2* work;        // (desc index, image), most expensive first
  int32_t n_work;
  int32_t* counters;       // [0] next unit to claim, [1] CTAs done (both 0 between launches)
};

struct MbMaps {
  CUtensorMap q, o;                   // R-stream, box (64, 1, 1, gr, 1)
  CUtensorMap k[kMbMaxMaps], v[kMbMaxMaps];  // per distinct interval, box rows 128
};

struct __align__(1024) MbSmem {
  uint8_t q[kQStages][2][kTileBytes];
  uint8_t k[kKStages][kTileBytes];
  uint8_t v[kVStages][kTileBytes];
  uint8_t ostage[kOStages][kTileBytes];
  uint8_t zero[kTileBytes];
  uint64_t q_full[kQStages], q_empty[kQStages];
  uint64_t k_full[kKStages], k_empty[kKStages];
  uint64_t v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[2][kSBufs];
  uint64_t p_full[kSBufs];
  uint64_t s_free[kSBufs];
  uint64_t pv_done[2];
  uint64_t o_full[2], o_empty[2];
  uint64_t stat_full[2], stat_empty[2];
  uint64_t sched_full[kSchedDepth], sched_empty[kSchedDepth];
  int32_t sched[kSchedDepth];    // claimed work-list index per ring slot (-1: no more work)
  int32_t sched_b[kSchedDepth];  // its image
  MbDesc dring[kSchedDepth];     // its descriptor, bulk-copied by the producer
  float stat_l[2][2][kBM];
  float stat_m[2][2][kBM];
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t tile_tp(uint32_t w) { return w & 0xFFFFFFu; }
__device__ __forceinline__ int32_t tile_br(uint32_t w) { return (int32_t)((w >> 24) & 7u); }
__device__ __forceinline__ uint32_t tile_mask(uint32_t w) { return (w >> 28) & 3u; }

// Optional timeline trace (kTrace instantiation, profiling only): CTA 0
// records (event << 56 | clock64) per role into trace[seg * 4096]; same
// events and layout as dfa_sm100.cu (decoded by scripts/trace_timeline.py).
constexpr int kTraceCap = 4096;
#define MB_TRACE(seg, ev)                                                                          \
  do {                                                                                             \
    if constexpr (kTrace) {                                                                        \
      if (tr_on && tr_n < kTraceCap)                                                               \
        trace[(seg) * kTraceCap + tr_n++] = ((uint64_t)(ev) << 56) | (clock64() & 0xFFFFFFFFFFFFFFull); \
    }                                                                                              \
  } while (0)

// Consumer side of the ring: free the previous unit's slot (n > 0), wait for
// unit n; returns its slot (the work index is sm.sched[slot], -1 = done).
// kWarp: a whole warp takes the unit and its lane 0 frees the slot.
template <bool kWarp>
__device__ __forceinline__ uint32_t next_slot(MbSmem& sm, uint32_t n) {
  if (n > 0) {
    const uint32_t prev = (n - 1) % kSchedDepth;
    if constexpr (kWarp) {
      __syncwarp();
      if (ptx::lane_id() == 0) ptx::mbar_arrive(&sm.sched_empty[prev]);
    } else {
      ptx::mbar_arrive(&sm.sched_empty[prev]);
    }
  }
  const uint32_t slot = n % kSchedDepth;
  ptx::mbar_wait(&sm.sched_full[slot], (n / kSchedDepth) & 1u);
  return slot;
}

template <bool kTrace, bool kSumCheck = false>
__global__ void __launch_bounds__(kThreads, 1)
    dfa_mb_sm100_kernel(const __grid_constant__ MbMaps maps, float* __restrict__ lse,
                        const __grid_constant__ MbParams p, uint64_t* __restrict__ trace) {
  extern __shared__ uint8_t smem_raw[];
  MbSmem& sm = *reinterpret_cast<MbSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();

  for (uint32_t i = threadIdx.x; i < kTileBytes / 16; i += kThreads)
    ptx::st_shared_v4(ptx::smem_u32(sm.zero) + 16 * i, 0u, 0u, 0u, 0u);
  ptx::fence_proxy_async_smem();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kQStages; ++s) {
      ptx::mbar_init(&sm.q_full[s], 1);
      ptx::mbar_init(&sm.q_empty[s], 1);
    }
    for (int s = 0; s < kKStages; ++s) {
      ptx::mbar_init(&sm.k_full[s], 1);
      ptx::mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      ptx::mbar_init(&sm.v_full[s], 1);
      ptx::mbar_init(&sm.v_empty[s], 1);
    }
    for (int b = 0; b < kSBufs; ++b) {
      ptx::mbar_init(&sm.s_full[0][b], 1);
      ptx::mbar_init(&sm.s_full[1][b], 1);
      ptx::mbar_init(&sm.p_full[b], kBM);
      ptx::mbar_init(&sm.s_free[b], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&sm.pv_done[s], 1);
      ptx::mbar_init(&sm.o_full[s], 1);
      ptx::mbar_init(&sm.o_empty[s], kBM);
      ptx::mbar_init(&sm.stat_full[s], kBM);
      ptx::mbar_init(&sm.stat_empty[s], kBM);
    }
    for (int i = 0; i < kSchedDepth; ++i) {
      ptx::mbar_init(&sm.sched_full[i], 1);
      ptx::mbar_init(&sm.sched_empty[i], kSchedConsumers);
    }
    ptx::fence_barrier_init();
    ptx::tma_prefetch_desc(&maps.q);
    ptx::tma_prefetch_desc(&maps.o);
  } else if (warp == 2) {
    ptx::tmem_alloc<kTmemCols>(&sm.tmem_base);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = sm.tmem_base;
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();
  if constexpr (kTrace) {
    if (threadIdx.x == 0) trace[6 * kTraceCap + 2 * blockIdx.x] = ptx::globaltimer();
  }

  // Registers: producers / MMA issuers 64, softmax 2 x 192, epilogue 64
  // (sum 65536); the work-list bounds are read inside each role so nothing
  // lives across the re-allocation.
  if (warp < 4) ptx::setmaxnreg_dec<64>();
  if (warp == 0) {
    // ============================================================ producer
    if (ptx::elect_one()) {
      const int32_t gr = 1 << p.gr_shift;
      const uint64_t pol = ptx::policy_evict_normal();  // key tiles are shared by several units
      const bool tr_on = blockIdx.x == 0;
      uint32_t tr_n = 0;
      uint32_t i = 0, g = 0;
      for (uint32_t n = 0;; ++n) {
        // claim the next unit once a Q stage is free (claimed work waits as little as possible)
        const uint32_t qs = i % kQStages;
        ptx::mbar_wait(&sm.q_empty[qs], ((i / kQStages) & 1) ^ 1);
        const uint32_t slot = n % kSchedDepth;
        ptx::mbar_wait(&sm.sched_empty[slot], ((n / kSchedDepth) & 1u) ^ 1u);
        int32_t wi = atomicAdd(&p.counters[0], 1);
        if (wi >= p.n_work) wi = -1;
        sm.sched[slot] = wi;
        if (wi < 0) {
          ptx::mbar_arrive(&sm.sched_full[slot]);
          break;
        }
        const int2 wk = p.work[wi];
        sm.sched_b[slot] = wk.y;
        ptx::mbar_arrive_expect_tx(&sm.sched_full[slot], (uint32_t)sizeof(MbDesc));
        ptx::bulk_g2s(&sm.dring[slot], p.desc + wk.x, (uint32_t)sizeof(MbDesc), &sm.sched_full[slot]);
        ptx::mbar_wait(&sm.sched_full[slot], (n / kSchedDepth) & 1u);
        const MbDesc& D = sm.dring[slot];
        const int32_t n_tiles = D.n_tiles;
        if (n_tiles == 0) continue;
        const int32_t b = wk.y, j = D.j;
        MB_TRACE(0, 1);
        const int act = (D.first[0] >= 0 ? 1 : 0) + (D.first[1] >= 0 ? 1 : 0);
        ptx::mbar_arrive_expect_tx(&sm.q_full[qs], act * kTileBytes);
        for (int s = 0; s < 2; ++s) {
          if (D.first[s] < 0) continue;
          for (int32_t gi = 0; gi < (kBM >> p.gr_shift); ++gi)
            ptx::tma_load_5d(sm.q[qs][s] + gi * gr * 128, &maps.q, &sm.q_full[qs], 0, j, D.cls[s][gi], D.qt[s],
                             b, pol);
        }
        ++i;
        for (int32_t t = 0; t < n_tiles; ++t, ++g) {
          const uint32_t w = D.tile[t];
          const int32_t br = tile_br(w);
          const uint32_t st = g % kKStages;
          MB_TRACE(0, 2);
          ptx::mbar_wait(&sm.k_empty[st], ((g / kKStages) & 1) ^ 1);
          MB_TRACE(0, 3);
          ptx::mbar_arrive_expect_tx(&sm.k_full[st], kTileBytes);
          ptx::tma_load_5d(sm.k[st], &maps.k[p.br_map[br]], &sm.k_full[st], 0, j, D.gamma[br], (int32_t)tile_tp(w),
                           b, pol);
        }
      }
    }
  } else if (warp == 3) {
    // ========================================================== V producer
    if (ptx::elect_one()) {
      const uint64_t pol = ptx::policy_evict_normal();
      uint32_t g = 0;
      for (uint32_t n = 0;; ++n) {
        const uint32_t slot = next_slot<false>(sm, n);
        if (sm.sched[slot] < 0) break;
        const MbDesc& D = sm.dring[slot];
        const int32_t n_tiles = D.n_tiles, j = D.j, img = sm.sched_b[slot];
        for (int32_t t = 0; t < n_tiles; ++t, ++g) {
          const uint32_t w = D.tile[t];
          const int32_t br = tile_br(w);
          const uint32_t st = g % kVStages;
          ptx::mbar_wait(&sm.v_empty[st], ((g / kVStages) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&sm.v_full[st], kTileBytes);
          ptx::tma_load_5d(sm.v[st], &maps.v[p.br_map[br]], &sm.v_full[st], 0, j, D.gamma[br], (int32_t)tile_tp(w),
                           img, pol);
        }
      }
    }
  } else if (warp == 1) {
    // ======================================================= Q K^T issuer
    if (ptx::elect_one()) {
      constexpr uint32_t idesc_qk = ptx::idesc_bf16(kBM, kBN, 0, 0);
      const uint64_t qdesc0 = ptx::sdesc_sw128(ptx::smem_u32(sm.q[0][0]));
      const uint64_t kdesc0 = ptx::sdesc_sw128(ptx::smem_u32(sm.k[0]));
      uint32_t b = 0, steps = 0, sfree_par = 0, gs = 0, gpar = 0, i = 0;
      const bool tr_on = blockIdx.x == 0;
      uint32_t tr_n = 0;
      for (uint32_t n = 0;; ++n) {
        const uint32_t slot = next_slot<false>(sm, n);
        if (sm.sched[slot] < 0) break;
        const MbDesc& D = sm.dring[slot];
        const int32_t n_tiles = D.n_tiles;
        if (n_tiles == 0) continue;
        const uint32_t qs = i & 1;
        MB_TRACE(1, 7);
        ptx::mbar_wait(&sm.q_full[qs], (i >> 1) & 1);
        MB_TRACE(1, 19);
        ++i;
        for (int32_t t = 0; t < n_tiles; ++t) {
          const uint32_t mask = tile_mask(D.tile[t]);
          ptx::mbar_wait(&sm.k_full[gs], gpar);
          ptx::tc_fence_after();
          MB_TRACE(1, 17);
          const uint64_t kd = kdesc0 + (uint64_t)(gs * (kTileBytes >> 4));
#pragma unroll 1
          for (int sl = 0; sl < 2; ++sl) {
            if (!((mask >> sl) & 1u)) continue;
            if (steps >= (uint32_t)kSBufs) {
              ptx::mbar_wait(&sm.s_free[b], (sfree_par >> b) & 1u);
              ptx::tc_fence_after();
            }
            sfree_par ^= (steps >= (uint32_t)kSBufs ? 1u : 0u) << b;
            const uint64_t qd = qdesc0 + (uint64_t)((qs * 2 + sl) * (kTileBytes >> 4));
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk)
              ptx::mma_ss(tbase + col_s(b), qd + (uint64_t)(2 * kk), kd + (uint64_t)(2 * kk), idesc_qk, kk > 0);
            ptx::tc_commit(&sm.s_full[sl][b]);
            MB_TRACE(1, 8);
            b = (b == kSBufs - 1) ? 0 : b + 1;
            ++steps;
          }
          ptx::tc_commit(&sm.k_empty[gs]);
          if (++gs == kKStages) {
            gs = 0;
            gpar ^= 1u;
          }
        }
        ptx::tc_commit(&sm.q_empty[qs]);
      }
    }
  } else if (warp == 2) {
    // ========================================================= P V issuer
    if (ptx::elect_one()) {
      constexpr uint32_t idesc_pv = ptx::idesc_bf16(kBM, kD, 0, 1);
      const uint64_t vdesc0 = ptx::sdesc_sw128(ptx::smem_u32(sm.v[0]));
      uint32_t b = 0, p_par = 0, oc_par = 0, gs = 0, gpar = 0;
      const bool tr_on = blockIdx.x == 0;
      uint32_t tr_n = 0;
      for (uint32_t n = 0;; ++n) {
        const uint32_t slot = next_slot<false>(sm, n);
        if (sm.sched[slot] < 0) break;
        const MbDesc& D = sm.dring[slot];
        const int32_t n_tiles = D.n_tiles;
        const int32_t first0 = D.first[0], first1 = D.first[1], last0 = D.last[0], last1 = D.last[1];
        for (int32_t t = 0; t < n_tiles; ++t) {
          const uint32_t mask = tile_mask(D.tile[t]);
          bool have_v = false;
          const uint64_t vdesc = vdesc0 + (uint64_t)(gs * (kTileBytes >> 4));
#pragma unroll 1
          for (int sl = 0; sl < 2; ++sl) {
            if (!((mask >> sl) & 1u)) continue;
            const bool first = t == (sl ? first1 : first0);
            MB_TRACE(5, 4);
            ptx::mbar_wait(&sm.p_full[b], (p_par >> b) & 1u);
            MB_TRACE(5, 5);
            p_par ^= 1u << b;
            if (first) ptx::mbar_wait(&sm.o_empty[sl], ((oc_par >> sl) & 1u) ^ 1u);
            if (!have_v) {
              ptx::mbar_wait(&sm.v_full[gs], gpar);
              have_v = true;
            }
            ptx::tc_fence_after();
            MB_TRACE(5, 18);
#pragma unroll
            for (int kk = 0; kk < kBN / 16; ++kk)
              ptx::mma_ts(tbase + col_o(sl), tbase + col_s(b) + kk * 8, vdesc + (uint64_t)(kk * (2048 >> 4)),
                          idesc_pv, (!first || kk > 0) ? 1u : 0u);
            ptx::tc_commit(&sm.pv_done[sl]);
            ptx::tc_commit(&sm.s_free[b]);
            MB_TRACE(5, 6);
            if (t == (sl ? last1 : last0)) {
              ptx::tc_commit(&sm.o_full[sl]);
              oc_par ^= 1u << sl;
            }
            b = (b == kSBufs - 1) ? 0 : b + 1;
          }
          ptx::tc_commit(&sm.v_empty[gs]);
          if (++gs == kVStages) {
            gs = 0;
            gpar ^= 1u;
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ====================================================== softmax slots
    ptx::setmaxnreg_inc<192>();
    const int s = (warp - 4) / 4;
    const uint32_t row = (warp % 4) * 32 + lane;
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const uint32_t tO = tbase + lane_base + col_o(s);
    const int32_t grp = (int32_t)row >> p.gr_shift;
    const int32_t rin = (int32_t)row & ((1 << p.gr_shift) - 1);
    uint32_t use_par = 0, pvc = 0, steps = 0, published = 0;
    uint32_t kbase = 0;  // CTA-global index of the unit's first step
    const bool tr_on = blockIdx.x == 0 && row == 0;
    uint32_t tr_n = 0;
    for (uint32_t n = 0;; ++n) {
      const uint32_t slot = next_slot<true>(sm, n);
      if (sm.sched[slot] < 0) break;
      const MbDesc& D = sm.dring[slot];
      const uint32_t k_unit = kbase;
      kbase += (uint32_t)D.steps;
      if (D.first[s] < 0) continue;
      // this thread's query row: class group grp, R-stream t = qt + rin
      const int32_t t_row = D.qt[s] + rin;
      const bool valid = t_row < p.TR;
      const int32_t n_row = t_row * p.R + D.cls[s][grp];
      const uint32_t sel_row = valid ? 0xFFu : 0u;
      float mref = -INFINITY, l = 0.0f;
      int32_t cur_br = -1, seg_lo = 0, seg_hi = 0;
      const int32_t ns = D.sn[s];
      const uint32_t k_unit3 = k_unit % kSBufs;
      for (int32_t si = 0; si < ns; ++si) {
        const uint32_t w = D.sstep[s][si];
        const uint32_t here = w >> 23;  // step index within the unit
        const int32_t br = (int32_t)((w >> 20) & 7u);
        if (br != cur_br) {
          cur_br = br;
          const bool sel = (sel_row & D.sel[s][br]) >> grp & 1u;
          if (sel) {
            const int32_t tk = p.br_divr[br].div(n_row);  // row's t' in the branch's r-stream
            seg_lo = p.br_divm[br].div(tk) * p.br_m[br];
            seg_hi = min(seg_lo + p.br_m[br], p.br_T[br]);
          } else {
            seg_lo = seg_hi = 0;  // every key masked: this branch does not select the row
          }
        }
        const uint32_t b = (k_unit3 + here) % kSBufs;
        MB_TRACE(2 + s, 9);
        ptx::mbar_wait(&sm.s_full[s][b], (use_par >> b) & 1u);
        MB_TRACE(2 + s, 10);
        use_par ^= 1u << b;
        ptx::tc_fence_after();
        const uint32_t tS = tbase + lane_base + col_s(b);
        const int32_t k0 = (int32_t)(w & 0xFFFFFu);
        const int32_t lo = min(max(seg_lo - k0, 0), kBN);
        const int32_t hi = min(max(seg_hi - k0, 0), kBN);
        bool waited = false;
        if (__all_sync(0xffffffffu, lo >= hi)) {
          // no row of this warp has a key in this tile (branch does not select
          // the warp's class group, or keys outside its segments): P = 0
          uint32_t zp[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) zp[e] = 0u;
#pragma unroll
          for (int c = 0; c < kSC; ++c) ptx::tmem_st16(tS + 16 * c, zp);
        } else {
          uint32_t sr[kSC][32];
#pragma unroll
          for (int c = 0; c < kSC; ++c) ptx::tmem_ld32(tS + 32 * c, sr[c]);
          ptx::tmem_ld_wait();
          if (!(lo == 0 && hi == kBN)) {
#pragma unroll
            for (int c = 0; c < kSC; ++c)
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                const int col = 32 * c + e;
                if (col < lo || col >= hi) sr[c][e] = __float_as_uint(-INFINITY);
              }
          }
          auto exp_pass = [&](float neg, bool clamp_hi) -> float {
            float2 ls2[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
            const float2 c2 = make_float2(p.c, p.c), n2 = make_float2(neg, neg);
#pragma unroll
            for (int c = 0; c < kSC; ++c) {
              float2 xv[16];
#pragma unroll
              for (int e = 0; e < 16; ++e)
                xv[e] = ptx::ffma2(make_float2(__uint_as_float(sr[c][2 * e]), __uint_as_float(sr[c][2 * e + 1])), c2, n2);
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                if (((kSumCheck ? kPolyMaskSumCheck : kPolyMask) >> e) & 1u) {
                  // the polynomial's exponent add wraps for x >= 128: clamp so an
                  // overflowing tile shows up in the fast path's row sum
                  if (clamp_hi) xv[e] = make_float2(fminf(xv[e].x, 126.0f), fminf(xv[e].y, 126.0f));
                  xv[e] = ptx::ex2_poly2(xv[e]);
                } else {
                  xv[e].x = ptx::ex2(xv[e].x);
                  xv[e].y = ptx::ex2(xv[e].y);
                }
              }
              uint32_t pk[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                ls2[e & 1] = ptx::fadd2(ls2[e & 1], xv[e]);
                pk[e] = ptx::pack_bf16x2(xv[e].x, xv[e].y);
              }
              ptx::tmem_st16(tS + 16 * c, pk);
            }
            const float2 lsum = ptx::fadd2(ls2[0], ls2[1]);
            return lsum.x + lsum.y;
          };
          bool exact = true;
          if constexpr (kSumCheck) {
            // Fast path (every row of the warp already has a reference): no
            // row max; the tile is redone exactly when a row sum exceeds 2^8
            // against the reference (or is inf / NaN), P re-stored in place.
            if (__all_sync(0xffffffffu, mref != -INFINITY)) {
              const float fs = exp_pass(-mref * p.c, true);
              exact = __any_sync(0xffffffffu, !(fs <= kSumBound));
              if (!exact) l += fs;
            }
          }
          if (exact) {
            float mx[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) mx[e] = -INFINITY;
#pragma unroll
            for (int c = 0; c < kSC; ++c)
#pragma unroll
              for (int e = 0; e < 32; ++e) mx[e & 7] = fmaxf(mx[e & 7], __uint_as_float(sr[c][e]));
            const float tmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                     fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
            const bool move = tmax > mref && (mref == -INFINITY || (tmax - mref) * p.c > kRescaleThreshold);
            const bool fix_o = move && mref != -INFINITY;
            if (__any_sync(0xffffffffu, fix_o)) {
              if (steps > 0) {
                ptx::mbar_wait(&sm.pv_done[s], pvc & 1);
                ++pvc;
                waited = true;
              }
              ptx::tc_fence_after();
              const float corr = fix_o ? ptx::ex2((mref - tmax) * p.c) : 1.0f;
              l *= corr;
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
            MB_TRACE(2 + s, 11);
            if (move) mref = tmax;
            l += exp_pass((mref == -INFINITY) ? 0.0f : -mref * p.c, false);
          }
        }  // rows with keys in this tile
        MB_TRACE(2 + s, 12);
        if (!waited && steps > 0) {
          ptx::mbar_wait(&sm.pv_done[s], pvc & 1);
          ++pvc;
        }
        ++steps;
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&sm.p_full[b]);
        MB_TRACE(2 + s, 13);
      }
      // rows no branch of this unit selects: l = 0 -> exact zeros in the epilogue
      const bool any = valid && ((D.anysel[s] >> grp) & 1u);
      sm.stat_l[published & 1][s][row] = any ? l : 0.0f;
      sm.stat_m[published & 1][s][row] = mref;
      if (published > 0) ptx::mbar_wait(&sm.stat_empty[s], (published - 1) & 1);
      ptx::mbar_arrive(&sm.stat_full[s]);
      ++published;
    }
  } else if (warp >= 12) {
    // ============================================================ epilogue
    ptx::setmaxnreg_dec<64>();
    const uint32_t row = (warp % 4) * 32 + lane;
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const bool leader = warp == 12 && lane == 0;
    const int32_t grp = (int32_t)row >> p.gr_shift;
    const int32_t rin = (int32_t)row & ((1 << p.gr_shift) - 1);
    const int32_t n_groups = kBM >> p.gr_shift;
    uint32_t par = 0;
    const bool tr_on = blockIdx.x == 0 && leader;
    uint32_t tr_n = 0;
    for (uint32_t n = 0;; ++n) {
      const uint32_t slot = next_slot<true>(sm, n);
      if (sm.sched[slot] < 0) break;
      const MbDesc& D = sm.dring[slot];
      const int32_t b = sm.sched_b[slot], j = D.j;
#pragma unroll 1
      for (int s = 0; s < 2; ++s) {
        const int32_t qt = D.qt[s];
        if (qt < 0) continue;  // slot absent
        const int32_t t_row = qt + rin;
        const bool valid = t_row < p.TR;
        const int32_t n_row = t_row * p.R + D.cls[s][grp];
        float* lrow = (lse && valid) ? lse + ((int64_t)b * p.h + j) * p.N + n_row : nullptr;
        if (D.first[s] < 0) {
          // no branch selects any row of this tile: zeros, lse = -inf
          if (lrow) *lrow = -INFINITY;
          if (leader) {
            for (int32_t gi = 0; gi < n_groups; ++gi)
              ptx::tma_store_5d(&maps.o, sm.zero, 0, j, D.cls[s][gi], qt, b);
            ptx::tma_store_commit();
          }
          continue;
        }
        const uint32_t ph = (par >> s) & 1u;
        par ^= 1u << s;
        MB_TRACE(4, 14);
        ptx::mbar_wait(&sm.o_full[s], ph);
        MB_TRACE(4, 15);
        ptx::mbar_wait(&sm.stat_full[s], ph);
        ptx::tc_fence_after();
        const float l = sm.stat_l[ph][s][row];
        const float mref = sm.stat_m[ph][s][row];
        const uint32_t tO = tbase + lane_base + col_o(s);
        const float inv = l > 0.0f ? 1.0f / l : 0.0f;
        const uint32_t stage_addr = ptx::smem_u32(sm.ostage[s]);
        if (leader) ptx::tma_store_wait_read<0>();
        ptx::named_bar_sync(1, kBM);
        // O row in two 32-column halves (64 registers for the epilogue)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint32_t orow[32];
          ptx::tmem_ld32(tO + 32 * hf, orow);
          ptx::tmem_ld_wait();
          if (hf == 1) {
            ptx::tc_fence_before();
            ptx::mbar_arrive(&sm.stat_empty[s]);
            ptx::mbar_arrive(&sm.o_empty[s]);
          }
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const int c = hf * 4 + c4;
            const float* f = reinterpret_cast<const float*>(&orow[c4 * 8]);
            const uint32_t addr = stage_addr + row * 128 + ((c ^ (row & 7)) * 16);
            ptx::st_shared_v4(addr, ptx::pack_bf16x2(f[0] * inv, f[1] * inv), ptx::pack_bf16x2(f[2] * inv, f[3] * inv),
                              ptx::pack_bf16x2(f[4] * inv, f[5] * inv), ptx::pack_bf16x2(f[6] * inv, f[7] * inv));
          }
        }
        if (lrow) *lrow = l > 0.0f ? mref * p.scale + __logf(l) : -INFINITY;
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(1, kBM);
        if (leader) {
          for (int32_t gi = 0; gi < n_groups; ++gi)
            ptx::tma_store_5d(&maps.o, sm.ostage[s] + gi * (128 << p.gr_shift), 0, j, D.cls[s][gi], qt, b);
          ptx::tma_store_commit();
        }
        MB_TRACE(4, 16);
      }
    }
    if (leader) ptx::tma_store_wait_all<0>();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (kTrace) {
    if (threadIdx.x == 0) trace[6 * kTraceCap + 2 * blockIdx.x + 1] = ptx::globaltimer();
  }
  if (threadIdx.x == 0) ptx::rearm_counters(p.counters);  // every CTA has claimed past the end
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tbase);
  }
}

// ---------------------------------------------------------------- host side
bool stream_map(CUtensorMap* map, const void* base, int64_t B, int64_t N, int64_t r, int64_t h, int64_t ld,
                uint32_t rows) {
  return encode_stream_map(map, base, B, N, r, h, ld, rows);
}

int64_t gcd64(int64_t a, int64_t b) { return b ? gcd64(b, a % b) : a; }

// A query tile of the schedule: super-unit su, class base c; per branch the
// selected groups and the key range [lo, lo + 128 nt) in the branch's stream.
struct TileInfo {
  int32_t su, c, steps;
  uint8_t sel[kMaxBranches];
  int32_t lo[kMaxBranches], nt[kMaxBranches];
};

// A plan's work counters are claimed by one launch at a time: the key
// includes the stream (launches on one stream are ordered; PDL waits for the
// previous grid before any global access).
struct PlanKey {
  int dev;
  uintptr_t stream;
  int64_t N, h, B;
  int grid;
  std::vector<int64_t> br;  // w, r, offsets... per branch
  bool operator==(const PlanKey& o) const {
    return dev == o.dev && stream == o.stream && N == o.N && h == o.h && B == o.B && grid == o.grid && br == o.br;
  }
};

struct DevicePlan {
  PlanKey key;
  void* buf = nullptr;  // descs | work | counters
  const MbDesc* desc = nullptr;
  const int2* work = nullptr;
  int32_t* counters = nullptr;
  int32_t n_work = 0;
  int32_t R = 1, gr_shift = 7, grid = 1;
  int n_maps = 0;
  int64_t r_of_map[kMbMaxMaps] = {};
  int32_t br_map[kMaxBranches] = {};
  int64_t steps = 0;
};

// Build the schedule on the host.  Returns false (with why) when the set is
// outside the fused kernel's envelope; the caller then takes the per-branch path.
bool build_plan(const Geometry* gb, int nb, int grid, DevicePlan* out, std::vector<uint8_t>* blob,
                const char** why) {
  const Geometry& g0 = gb[0];
  const int64_t N = g0.N, h = g0.h, B = g0.B;
  int64_t R = 1;
  for (int b = 0; b < nb; ++b) {
    if (gb[b].w % gb[b].r != 0) return (*why = "an interval does not divide its segment length"), false;
    R = R / gcd64(R, gb[b].r) * gb[b].r;
    if (R > 1024) return (*why = "lcm of the intervals > 1024"), false;
  }
  if (N % R != 0) return (*why = "lcm of the intervals does not divide N"), false;
  if (N >= (1 << 20)) return (*why = "N >= 2^20 (key-tile t' is packed in 20 bits)"), false;
  // distinct intervals -> tensor-map slots
  out->n_maps = 0;
  for (int b = 0; b < nb; ++b) {
    int m = 0;
    while (m < out->n_maps && out->r_of_map[m] != gb[b].r) ++m;
    if (m == out->n_maps) {
      if (out->n_maps == kMbMaxMaps) return (*why = "more than 4 distinct intervals"), false;
      out->r_of_map[out->n_maps++] = gb[b].r;
    }
    out->br_map[b] = m;
  }
  const int64_t TR = N / R;
  // tiles of head j for G class groups per tile
  auto make_tiles = [&](int64_t G, int64_t j, std::vector<TileInfo>* tiles) {
    const int64_t gr = 128 / G, nsu = (TR + gr - 1) / gr, nc = R / G;
    tiles->clear();
    for (int64_t su = 0; su < nsu; ++su) {
      const int64_t tf = su * gr, tl = std::min(tf + gr, TR) - 1;
      for (int64_t c = 0; c < nc; ++c) {
        TileInfo t{};
        t.su = (int32_t)su;
        t.c = (int32_t)c;
        for (int b = 0; b < nb; ++b) {
          const Geometry& gbb = gb[b];
          const int64_t gam = gbb.offsets[j];
          uint8_t sel = 0;
          int64_t cmin = R, cmax = -1;
          for (int64_t gi = 0; gi < G; ++gi) {
            const int64_t cls = c + gi * nc;
            if (cls % gbb.r == gam) {
              sel |= (uint8_t)(1u << gi);
              cmin = std::min(cmin, cls);
              cmax = std::max(cmax, cls);
            }
          }
          t.sel[b] = sel;
          if (!sel) continue;
          const int64_t nmin = tf * R + cmin, nmax = tl * R + cmax;
          const int64_t m = gbb.w / gbb.r, T = N / gbb.r;
          const int64_t lo = (nmin / gbb.w) * m, hi = std::min((nmax / gbb.w + 1) * m, T);
          t.lo[b] = (int32_t)lo;
          t.nt[b] = (int32_t)((hi - lo + kBN - 1) / kBN);
          t.steps += t.nt[b];
        }
        tiles->push_back(t);
      }
    }
  };
  // pick G (class groups per tile) by total steps over all heads
  int64_t bestG = 0, best_steps = INT64_MAX;
  std::vector<TileInfo> tiles;
  for (int64_t G = 1; G <= kMbMaxGroups; G *= 2) {
    if (R % G != 0) break;
    int64_t st = 0;
    for (int64_t j = 0; j < h; ++j) {
      make_tiles(G, j, &tiles);
      for (const TileInfo& t : tiles) st += t.steps;
    }
    if (st < best_steps) {
      best_steps = st;
      bestG = G;
    }
  }
  const int64_t G = bestG, gr = 128 / G;
  int gs = 0;
  while ((1 << gs) < gr) ++gs;
  out->R = (int32_t)R;
  out->gr_shift = gs;
  // pair tiles per head into units
  std::vector<MbDesc> descs;
  std::vector<int32_t> desc_su;  // first super-unit a unit touches (for the time order)
  int64_t total_steps = 0;
  for (int64_t j = 0; j < h; ++j) {
    make_tiles(G, j, &tiles);
    const int nt = (int)tiles.size();
    std::vector<int> order(nt);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tiles[a].steps > tiles[b].steps; });
    std::vector<char> used(nt, 0);
    auto shared = [&](const TileInfo& a, const TileInfo& b) {
      int64_t s = 0;
      for (int k = 0; k < nb; ++k)
        if (a.sel[k] && b.sel[k] && a.lo[k] == b.lo[k]) s += std::min(a.nt[k], b.nt[k]);
      return s;
    };
    for (int oi = 0; oi < nt; ++oi) {
      const int a = order[oi];
      if (used[a]) continue;
      used[a] = 1;
      int bsel = -1;
      int64_t bscore = -1;
      for (int ok = oi + 1, seen = 0; ok < nt && seen < 64; ++ok) {
        const int c = order[ok];
        if (used[c]) continue;
        ++seen;
        if (tiles[c].steps != tiles[a].steps && bsel >= 0) break;
        const int64_t sc = shared(tiles[a], tiles[c]) * 4 - std::abs(tiles[c].steps - tiles[a].steps);
        if (sc > bscore) {
          bscore = sc;
          bsel = c;
        }
      }
      if (bsel >= 0) used[bsel] = 1;
      MbDesc d{};
      d.j = (int32_t)j;
      const TileInfo* ts[2] = {&tiles[a], bsel >= 0 ? &tiles[bsel] : nullptr};
      for (int s = 0; s < 2; ++s) {
        d.first[s] = d.last[s] = -1;
        d.qt[s] = -1;
        if (!ts[s]) continue;
        d.qt[s] = (int32_t)(ts[s]->su * gr);
        for (int64_t gi = 0; gi < G; ++gi) d.cls[s][gi] = (int16_t)(ts[s]->c + gi * (R / G));
        for (int k = 0; k < nb; ++k) {
          d.sel[s][k] = ts[s]->sel[k];
          d.anysel[s] |= ts[s]->sel[k];
        }
      }
      for (int k = 0; k < nb; ++k) d.gamma[k] = gb[k].offsets[j];
      auto push = [&](int k, int64_t tp, uint32_t mask) -> bool {
        if (d.n_tiles >= kMbMaxTiles) return false;
        for (int s = 0; s < 2; ++s)
          if ((mask >> s) & 1u) {
            if (d.first[s] < 0) d.first[s] = d.n_tiles;
            d.last[s] = d.n_tiles;
          }
        uint32_t at = (uint32_t)d.steps;  // step index of this tile's first step in the unit
        for (int s = 0; s < 2; ++s)
          if ((mask >> s) & 1u) d.sstep[s][d.sn[s]++] = (uint32_t)tp | ((uint32_t)k << 20) | (at++ << 23);
        d.tile[d.n_tiles++] = (uint32_t)tp | ((uint32_t)k << 24) | (mask << 28);
        d.steps += (int32_t)((mask & 1u) + (mask >> 1));
        return true;
      };
      for (int k = 0; k < nb; ++k) {
        const bool ua = ts[0]->sel[k] != 0, ub = ts[1] && ts[1]->sel[k] != 0;
        const int na = ua ? ts[0]->nt[k] : 0, nbt = ub ? ts[1]->nt[k] : 0;
        bool ok = true;
        if (ua && ub && ts[0]->lo[k] == ts[1]->lo[k]) {
          for (int i = 0; i < std::max(na, nbt); ++i)
            ok = ok && push(k, ts[0]->lo[k] + (int64_t)kBN * i, (i < na ? 1u : 0u) | (i < nbt ? 2u : 0u));
        } else {
          for (int i = 0; i < std::max(na, nbt); ++i) {
            if (i < na) ok = ok && push(k, ts[0]->lo[k] + (int64_t)kBN * i, 1u);
            if (i < nbt) ok = ok && push(k, ts[1]->lo[k] + (int64_t)kBN * i, 2u);
          }
        }
        if (!ok) return (*why = "more than 64 key tiles in a work unit"), false;
      }
      total_steps += d.steps;
      descs.push_back(d);
      desc_su.push_back(std::min(ts[0]->su, ts[1] ? ts[1]->su : ts[0]->su));
    }
  }
  // Replicate over the batch into ONE work list that the CTAs claim
  // dynamically (no cost model needed for balance).
  const int64_t n_desc = (int64_t)descs.size();
  const int64_t n_work = n_desc * B;
  if (n_work > INT32_MAX / 2) return (*why = "too many work units"), false;
  std::vector<int2> seq;
  seq.reserve((size_t)n_work);
  for (int64_t e = 0; e < n_desc; ++e)
    for (int64_t b = 0; b < B; ++b) seq.push_back(make_int2((int)e, (int)b));
  // Image-major blocks (image, super-unit, head; most expensive unit first in
  // a block), so the units that read a super-unit's key tiles run at about the
  // same time and their re-reads hit L2; the last ~1/8 of the images is
  // ordered most-expensive-first instead, so the claimed tail is short.
  const int64_t b_tail = B - std::max<int64_t>(1, B / 8);
  std::stable_sort(seq.begin(), seq.end(), [&](int2 x, int2 y) {
    const MbDesc &dx = descs[x.x], &dy = descs[y.x];
    const bool tx = x.y >= b_tail, ty = y.y >= b_tail;
    if (tx != ty) return ty;  // block-ordered images first
    if (tx && dx.steps != dy.steps) return dx.steps > dy.steps;
    if (x.y != y.y) return x.y < y.y;
    if (desc_su[x.x] != desc_su[y.x]) return desc_su[x.x] < desc_su[y.x];
    if (dx.j != dy.j) return dx.j < dy.j;
    return dx.steps > dy.steps;
  });
  grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid, n_work));
  const size_t desc_bytes = sizeof(MbDesc) * (size_t)n_desc;
  const size_t work_bytes = sizeof(int2) * (size_t)n_work;
  const size_t work_at = (desc_bytes + 255) & ~(size_t)255, cnt_at = (work_at + work_bytes + 255) & ~(size_t)255;
  blob->assign(cnt_at + 256, 0);  // counters start at 0
  memcpy(blob->data(), descs.data(), desc_bytes);
  memcpy(blob->data() + work_at, seq.data(), work_bytes);
  out->n_work = (int32_t)n_work;
  out->grid = grid;
  out->steps = total_steps * B;
  // offsets of the arrays inside the device buffer (patched by the caller)
  out->desc = reinterpret_cast<const MbDesc*>(0);
  out->work = reinterpret_cast<const int2*>(work_at);
  out->counters = reinterpret_cast<int32_t*>(cnt_at);
  return true;
}

std::mutex g_plan_mu;
std::atomic<uint64_t*> g_mb_trace{nullptr};
std::vector<DevicePlan> g_plans;  // small LRU (front = most recent)
constexpr size_t kMaxPlans = 16;

}  // namespace

void set_mb_trace(uint64_t* trace) { g_mb_trace.store(trace); }

// Host-only: the schedule build_plan makes for a branch set (test / debug
// hook; no CUDA call).  Copies up to `cap` bytes of descriptors.
int mb_plan_host(const Geometry* gb, int nb, int grid, void* out, size_t cap, int32_t* n_desc, int32_t* R,
                 int32_t* gr_shift, int32_t* desc_bytes, const char** why) {
  DevicePlan plan;
  std::vector<uint8_t> blob;
  if (!build_plan(gb, nb, grid, &plan, &blob, why)) return 0;
  const size_t work_at = reinterpret_cast<uintptr_t>(plan.work);  // descriptors end before the work list
  const size_t n = plan.n_work / std::max<int64_t>(1, gb[0].B);
  *n_desc = (int32_t)n;
  *R = plan.R;
  *gr_shift = plan.gr_shift;
  *desc_bytes = (int32_t)sizeof(MbDesc);
  const size_t bytes = std::min(cap, std::min(work_at, n * sizeof(MbDesc)));
  if (out) memcpy(out, blob.data(), bytes);
  return 1;
}

// Fused multi-branch forward: returns 1 (launch issued), 0 when the set is
// outside the kernel's envelope (why set, nothing launched) or -1 on a CUDA
// error (err set).
int launch_mb_sm100(const Geometry* gb, int nb, const void* q, const void* k, const void* v, void* o, float* lse,
                    cudaStream_t stream, cudaError_t* err, const char** why, int64_t* steps_out) {
  ensure_context();
  *err = cudaSuccess;
  if (nb < 2 || nb > kMaxBranches) return (*why = "fused multibranch needs 2..8 branches"), 0;
  for (int b = 0; b < nb; ++b)
    if (!sm100_supported(gb[b], 1, q, k, v, o)) return (*why = "a branch is outside the tcgen05 envelope"), 0;
  const Geometry& g0 = gb[0];
  PlanKey key;
  key.dev = current_device();
  key.stream = reinterpret_cast<uintptr_t>(stream);
  key.N = g0.N;
  key.h = g0.h;
  key.B = g0.B;
  key.grid = device_sms();
  for (int b = 0; b < nb; ++b) {
    key.br.push_back(gb[b].w);
    key.br.push_back(gb[b].r);
    for (int64_t j = 0; j < g0.h; ++j) key.br.push_back(gb[b].offsets[j]);
  }
  DevicePlan plan;
  // The lock is held through the launch: a plan's buffer is only freed (LRU
  // eviction, after a device-wide synchronize) by a thread holding it, so no
  // launch can be enqueued on a buffer being freed.
  std::lock_guard<std::mutex> lock(g_plan_mu);
  {
    bool found = false;
    for (size_t i = 0; i < g_plans.size(); ++i)
      if (g_plans[i].key == key) {
        plan = g_plans[i];
        std::rotate(g_plans.begin(), g_plans.begin() + i, g_plans.begin() + i + 1);
        found = true;
        break;
      }
    if (!found) {
      // the schedule is uploaded once per (geometry, branch set); not while
      // the stream is being captured (the caller falls back instead)
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return (*why = "schedule not cached and the stream is capturing"), 0;
      }
      std::vector<uint8_t> blob;
      if (!build_plan(gb, nb, key.grid, &plan, &blob, why)) return 0;
      plan.key = key;
      cudaError_t e = cudaMalloc(&plan.buf, blob.size());
      if (e == cudaSuccess) e = cudaMemcpy(plan.buf, blob.data(), blob.size(), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) {
        if (plan.buf) cudaFree(plan.buf);
        *err = e;
        *why = "schedule upload failed";
        return -1;
      }
      char* base = static_cast<char*>(plan.buf);
      plan.desc = reinterpret_cast<const MbDesc*>(base);
      plan.work = reinterpret_cast<const int2*>(base + reinterpret_cast<uintptr_t>(plan.work));
      plan.counters = reinterpret_cast<int32_t*>(base + reinterpret_cast<uintptr_t>(plan.counters));
      if (g_plans.size() == kMaxPlans) {
        cudaDeviceSynchronize();  // the evicted plan may be in flight on any stream
        cudaFree(g_plans.back().buf);
        g_plans.pop_back();
      }
      g_plans.insert(g_plans.begin(), plan);
    }
  }
  MbMaps maps;
  const uint32_t gr = 1u << plan.gr_shift;
  bool ok = stream_map(&maps.q, q, g0.B, g0.N, plan.R, g0.h, g0.ldq, gr) &&
            stream_map(&maps.o, o, g0.B, g0.N, plan.R, g0.h, g0.ldo, gr);
  for (int m = 0; m < kMbMaxMaps; ++m) {
    const int64_t r = plan.r_of_map[m < plan.n_maps ? m : 0];
    ok = ok && stream_map(&maps.k[m], k, g0.B, g0.N, r, g0.h, g0.ldk, kBN) &&
         stream_map(&maps.v[m], v, g0.B, g0.N, r, g0.h, g0.ldv, kBN);
  }
  if (!ok) {
    *why = "cuTensorMapEncodeTiled failed";
    *err = cudaErrorInvalidValue;
    return -1;
  }
  MbParams p{};
  p.N = (int32_t)g0.N;
  p.h = (int32_t)g0.h;
  p.R = plan.R;
  p.TR = (int32_t)(g0.N / plan.R);
  p.gr_shift = plan.gr_shift;
  p.scale = g0.scale;
  p.c = g0.scale * kLog2e;
  for (int b = 0; b < nb; ++b) {
    p.br_m[b] = (int32_t)(gb[b].w / gb[b].r);
    p.br_T[b] = (int32_t)(g0.N / gb[b].r);
    p.br_map[b] = plan.br_map[b];
    p.br_divr[b] = make_fastdiv_mb((uint32_t)gb[b].r);
    p.br_divm[b] = make_fastdiv_mb((uint32_t)p.br_m[b]);
  }
  p.desc = plan.desc;
  p.work = plan.work;
  p.counters = plan.counters;
  p.n_work = plan.n_work;
  const size_t smem = sizeof(MbSmem) + 1024;
  uint64_t* trace = g_mb_trace.load();
  // Sum-checked fast path only when every branch's view is long (m = w / r
  // >= 1024): measured -3% on {(2048, 2), (4096, 4)}, but +9% on the LongNet
  // set and +20% on {(256, 2), (512, 2), (1024, 4)} (short views: the
  // redone tiles land on the critical path).
  int64_t min_m = INT64_MAX;
  for (int b = 0; b < nb; ++b) min_m = std::min<int64_t>(min_m, gb[b].w / gb[b].r);
  const bool sumcheck = DFA_MB_SUMCHECK < 0 ? min_m >= 1024 : DFA_MB_SUMCHECK != 0;
  auto kfn = trace ? dfa_mb_sm100_kernel<true> : sumcheck ? dfa_mb_sm100_kernel<false, true>
                                                          : dfa_mb_sm100_kernel<false>;
  cudaError_t ae = ensure_smem_attr(reinterpret_cast<const void*>(kfn), smem);
  if (ae != cudaSuccess) {
    *err = ae;
    *why = "cudaFuncSetAttribute failed";
    return -1;
  }
  cudaError_t le = cudaSuccess;
  if (trace)
    dfa_mb_sm100_kernel<true><<<plan.grid, kThreads, smem, stream>>>(maps, lse, p, trace);
  else
    le = launch_pdl(kfn, plan.grid, kThreads, smem, stream, maps, lse, p, (uint64_t*)nullptr);
  *err = le != cudaSuccess ? le : cudaGetLastError();
  if (*err != cudaSuccess) {
    *why = "launch failed";
    return -1;
  }
  if (steps_out) *steps_out = plan.steps;
  return 1;
}

}  // namespace dfa_impl
