// Dilated Flash Attention forward for sm_100a: TMA + tcgen05 + TMEM,
// persistent and warp-specialised.
//
// Reference path: attnkit::dilated_attention (attention.hpp:280-301):
// per segment i and head offset gamma, gather rows i*w+gamma+t*r
// (make_segment_view :84-98, sparsify_segment :210-222), softmax attention
// among them (naive_attention :119-127 / tiled_attention :147-207), scatter
// back into a zero-initialised [N, d] (recompose :246-274).
//
// B200 restatement.  With N % r == 0 the [B, N, h, d] bf16 tensor IS the
// contiguous 5-D tensor [B][N/r][r][h][d]; row n of image b sits at
// (b, t' = n / r, gamma' = n % r).  For head j the view rows of ALL segments
// are the t'-stream at gamma' = gamma_j, and segment i is the contiguous block
// t' in [i*m, i*m+m) (m = w/r when r | w; the tail segment is shorter).  The
// segment + strided gather of the reference is therefore a plain TMA box
// (d=64, h=1, gamma'=1, t'=128, b=1) at (0, j, gamma_j, t'0, b): no index
// arrays, no gather kernel.  Attention is block-diagonal in t'-space.  The
// recompose scatter is the same box stored back, plus r-1 boxes of zeros for
// the other offset classes (attention.hpp:243-245, 270), so every output byte
// is written exactly once and no memset is needed.
//
// Work unit = 256 consecutive t'-rows of one (b, j) stream: query tile A
// (rows t0..t0+127) and query tile B (t0+128..t0+255).  Key tiles of 128
// t'-rows cover the union of the segments either tile touches and are loaded
// ONCE per unit (for m >= 256 both tiles share them).  Keys outside a query's
// own segment are masked (only when m is not a multiple of 128, or at tails).
//
// Warp roles (512 threads, one CTA per SM, persistent over units):
//   warp 0      TMA producer: Q_A/Q_B (2-deep), K tiles (3-deep ring, a stage
//               is freed as soon as its Q K^T completes)
//   warp 3      TMA producer: V tiles (3-deep ring, freed after P V)
//   warp 1      Q K^T issuer (one elected lane):
//                 S_x = Q_x K^T   tcgen05.mma M=128 N=128 K=64 -> TMEM (fp32)
//               into three rotating S buffers, up to three steps ahead
//   warp 2      TMEM allocator (512 columns), then P V issuer:
//                 O_x += P_x V    tcgen05.mma A = P_x from TMEM, B = V (MN-major)
//               Two issuing threads on different SMSPs halve the serial
//               barrier-wait + issue latency per step (the single-issuer
//               timeline showed it on the critical path); s_free orders the
//               reuse of an S buffer after the P V that read it.
//   warps 4-7   slot A softmax (TMEM lanes 0-127, thread = row)
//   warps 8-11  slot B softmax
//   warps 12-15 epilogue (O / l -> bf16 -> TMA store, zero boxes, lse)
// Softmax: tcgen05.ld of the 128-score row, exp2 with the 1/sqrt(d)*log2(e)
// fold, lazy (2^8 threshold) rescale of O in TMEM, P packed to bf16 and
// tcgen05.st over the consumed S columns.  Epilogue: O/l -> bf16 -> 128B-
// swizzled smem staging -> TMA store; zero rows by TMA store from a zero tile.
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

constexpr int kD = 64;                 // head_dim handled by this kernel
constexpr int kBM = 128;               // query rows per slot (MMA M)
#ifndef DFA_BN
#define DFA_BN 128
#endif
constexpr int kBN = DFA_BN;            // keys per tile (MMA N of Q K^T, K of P V): 128 or 64
constexpr int kSC = kBN / 32;          // 32-column chunks of an S tile
constexpr int kUnitRows = 2 * kBM;     // t'-rows per work unit
constexpr int kTileBytes = 128 * 128;  // 128 rows x 128 B (64 bf16), SW128
constexpr int kKVTileBytes = kBN * 128;  // key / value tile: kBN rows x 128 B
#ifndef DFA_K_STAGES
#define DFA_K_STAGES 3
#endif
#ifndef DFA_V_STAGES
#define DFA_V_STAGES 3
#endif
#ifndef DFA_O_STAGES
#define DFA_O_STAGES 2
#endif
constexpr int kQStages = 2;
constexpr int kKStages = DFA_K_STAGES;  // K ring depth (loads in flight ahead of Q K^T)
constexpr int kVStages = DFA_V_STAGES;  // V ring depth
constexpr int kOStages = DFA_O_STAGES;  // epilogue staging tiles (slot s uses s % kOStages)
#ifndef DFA_ZERO_ROWS
#define DFA_ZERO_ROWS 128
#endif
// Rows per zero box: a smaller zero tile (stored 128 / kZeroRows times per
// class) frees shared memory for deeper load rings.
constexpr int kZeroRows = DFA_ZERO_ROWS;
constexpr int kThreads = 512;
constexpr uint32_t kTmemCols = 512;
constexpr int kSBufs = 384 / kBN;                          // rotating S/P buffers (3 x 128 or 6 x 64 columns)
__host__ __device__ constexpr uint32_t col_s(int buf) { return (uint32_t)kBN * buf; }  // S buffers (P aliases)
__host__ __device__ constexpr uint32_t col_o(int slot) { return 384u + 64u * slot; }  // O_A, O_B
constexpr float kLog2e = 1.4426950408889634f;
#ifndef DFA_RESCALE_THR
#define DFA_RESCALE_THR 8.0f
#endif
#ifndef DFA_POLY_MASK
#define DFA_POLY_MASK 0x0888u
#endif
constexpr float kRescaleThreshold = DFA_RESCALE_THR;  // log2 units: p <= 2^8 between rescales
#ifndef DFA_SUMCHECK
#define DFA_SUMCHECK -1  // -1: by geometry (launch_sm100), 0: never, 1: always
#endif
// Sum-checked fast path (DFA_SUMCHECK): a tile whose row sum against the
// running reference stays <= 2^thr needs no row max.
constexpr float kSumBound = 256.0f;
// bit e: pair e of each 16-pair (32-column) chunk uses the FMA-pipe exp2
// polynomial instead of MUFU.EX2 (balances the MUFU and FMA/issue pipes;
// measured with the 192-register softmax: 3 of 16 (pairs 3, 7, 11) beats
// 2 and 4 of 16 by 1-3% and 6 of 16 by 5-8%)
constexpr uint32_t kPolyMask = DFA_POLY_MASK;
// The sum-checked kernel (no row max on most tiles) leaves less work on the
// FMA / ALU side: 2 of 16 pairs (3 and 11) on the polynomial measured 1.7-4%
// faster than 3 of 16 on (1024, 1) .. (4096, 2); 1 / 16 and 4 / 16 slower.
#ifndef DFA_POLY_MASK_SC
#define DFA_POLY_MASK_SC 0x0808u
#endif
constexpr uint32_t kPolyMaskSumCheck = DFA_POLY_MASK_SC;

// Geometry of one work unit, identical in every role.
struct Unit {
  int32_t b, j, gamma;
  int32_t t0;              // first t' of slot A
  int32_t kv_lo;           // first key t' (a segment start)
  int32_t n_kv;            // key tiles in the unit
  int32_t kt0a, kt1a, kt0b, kt1b;  // key-tile range [kt0, kt1) of slot A / B (empty if equal)
  __device__ __forceinline__ int32_t kt0(int s) const { return s ? kt0b : kt0a; }
  __device__ __forceinline__ int32_t kt1(int s) const { return s ? kt1b : kt1a; }
};

// kKSt K-ring stages; the V ring takes the rest of the kKStages + kVStages
// tiles (the same shared-memory footprint for every split).
template <int kKSt = kKStages>
struct __align__(1024) SmemLayoutT {
  static constexpr int kVSt = kKStages + kVStages - kKSt;
  uint8_t q[kQStages][2][kTileBytes];  // contiguous: tile (stage, slot) at index stage * 2 + slot
  uint8_t k[kKSt][kKVTileBytes];
  uint8_t v[kVSt][kKVTileBytes];
  uint8_t ostage[kOStages][kTileBytes];
  uint8_t zero[kZeroRows * 128];
  uint64_t q_full[kQStages], q_empty[kQStages];
  uint64_t k_full[kKSt], k_empty[kKSt];  // K ring: freed when its last Q K^T completes
  uint64_t v_full[kVSt], v_empty[kVSt];  // V ring: freed when its last P V completes
  uint64_t s_full[2][kSBufs];  // MMA -> slot s: S ready in buffer b
  uint64_t p_full[kSBufs];     // slot -> P V issuer: P written in buffer b (128 arrivals)
  uint64_t s_free[kSBufs];     // P V issuer -> Q K^T issuer: P V of buffer b completed
  uint64_t pv_done[2];         // MMA -> slot s: its latest P V completed
  uint64_t o_full[2], o_empty[2];
  uint64_t stat_full[2];       // slot -> epilogue: row stats of the finished unit written
  uint64_t stat_empty[2];      // epilogue -> slot: stats read (keeps stat_full <= 1 phase ahead)
  uint64_t oload_full[2];      // merge mode: running output rows landed in ostage[slot]
  float stat_l[2][2][kBM];     // [published parity][slot][row] normaliser l
  float stat_m[2][2][kBM];     // [published parity][slot][row] reference max (raw score units), for lse
  uint32_t tmem_base;
};

// n / d for 0 <= n < 2^31 by multiply-high (magic numbers from the host).
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

struct Sm100Params {
  int32_t N, T;      // T = N / r (t'-stream length per (b, j))
  int32_t m;         // t'-rows per full segment (w / r)
  int32_t r, h;
  int32_t n_pairs;   // ceil(T / unit_rows) work units per (b, j) stream
  int32_t unit_rows; // 256 (slots A + B) or 128 (slot A only: twice the units for small grids)
  int32_t n_units;   // B * h * n_pairs
  float c;           // scale * log2(e)
  float scale;
  int32_t merge;     // 1: merge into the running (o, lse) of earlier branches (no zero boxes)
  int32_t zero_rows; // 0: the caller zero-fills the rows no view keeps (host-resident o, kept rows only cross PCIe)
  FastDiv div_pairs, div_h, div_m;
  int32_t offsets[kMaxHeads];
};

// Profiling probes (variant builds only, results wrong): drop the
// exponentials / the zero boxes to measure what each costs.
#ifndef DFA_PROBE_NO_EXP
#define DFA_PROBE_NO_EXP 0
#endif
#ifndef DFA_PROBE_NO_ZERO
#define DFA_PROBE_NO_ZERO 0
#endif
#ifndef DFA_L2_PROMO
#define DFA_L2_PROMO CU_TENSOR_MAP_L2_PROMOTION_NONE  // TMA L2 sector promotion of the t'-stream maps
#endif
#ifndef DFA_HEAD_MAJOR
#define DFA_HEAD_MAJOR 1
#endif
// Unit order.  Head-major (default): u = (b * n_pairs + pair) * h + j, so the
// h CTAs running side by side read the h heads' 128-byte column blocks of the
// SAME token rows -- one DRAM page opened once instead of h times.
__device__ __forceinline__ Unit make_unit(const Sm100Params& p, int32_t u) {
  Unit x;
#if DFA_HEAD_MAJOR
  const int32_t bp = p.div_h.div(u);
  x.j = u - bp * p.h;
  x.b = p.div_pairs.div(bp);
  const int32_t pair = bp - x.b * p.n_pairs;
#else
  const int32_t bj = p.div_pairs.div(u);
  const int32_t pair = u - bj * p.n_pairs;
  x.b = p.div_h.div(bj);
  x.j = bj - x.b * p.h;
#endif
  x.gamma = p.offsets[x.j];
  x.t0 = pair * p.unit_rows;
  int32_t lo[2], hi[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int32_t r0 = x.t0 + s * kBM;
    // half units (small grids): slot B stays empty, every CTA gets one 128-row tile
    const int32_t r1 = (s == 1 && p.unit_rows == kBM) ? r0 : min(r0 + kBM, p.T);
    if (r0 < r1) {
      lo[s] = p.div_m.div(r0) * p.m;
      hi[s] = min((p.div_m.div(r1 - 1) + 1) * p.m, p.T);
    } else {
      lo[s] = hi[s] = -1;
    }
  }
  x.kv_lo = lo[0];
  const int32_t kv_hi = hi[1] >= 0 ? max(hi[0], hi[1]) : hi[0];
  x.n_kv = (kv_hi - x.kv_lo + kBN - 1) / kBN;
  x.kt0a = (lo[0] - x.kv_lo) / kBN;
  x.kt1a = (hi[0] - x.kv_lo + kBN - 1) / kBN;
  if (lo[1] < 0) {
    x.kt0b = x.kt1b = 0;
  } else {
    x.kt0b = (lo[1] - x.kv_lo) / kBN;
    x.kt1b = (hi[1] - x.kv_lo + kBN - 1) / kBN;
  }
  return x;
}

// Per-unit step order (identical in every role): key tiles kt ascending, and
// for each kt slot A then slot B if the slot uses kt.  The CTA-global step
// index k selects S buffer k % 3.
__device__ __forceinline__ bool uses(const Unit& x, int slot, int32_t kt) {
  return kt >= x.kt0(slot) && kt < x.kt1(slot);
}
__device__ __forceinline__ int32_t clamp_count(int32_t kt, int32_t lo, int32_t hi) {
  return min(max(kt, lo), hi) - lo;  // tiles of [lo, hi) before kt
}
// index of step (kt, slot) within its unit
__device__ __forceinline__ int32_t step_in_unit(const Unit& x, int32_t kt, int slot) {
  return clamp_count(kt, x.kt0a, x.kt1a) + clamp_count(kt, x.kt0b, x.kt1b) + (slot == 1 && uses(x, 0, kt) ? 1 : 0);
}
__device__ __forceinline__ int32_t steps_of_unit(const Unit& x) { return (x.kt1a - x.kt0a) + (x.kt1b - x.kt0b); }

// Optional timeline trace (profiling builds of the same kernel, kTrace=true):
// CTA 0 records (event << 56 | clock64) per role into trace[seg * kTraceCap]
// (seg: 0 producer, 1 Q K^T issuer, 2/3 softmax A/B, 4 epilogue, 5 P V issuer).
constexpr int kTraceCap = 4096;
enum TraceEvent : uint64_t {
  TR_Q_ISSUE = 1, TR_KV_WAIT, TR_KV_ISSUE,                          // producer  (seg 0)
  TR_P_WAIT, TR_P_READY, TR_PV_ISSUED, TR_QK_WAIT, TR_QK_ISSUED,    // MMA       (seg 1)
  TR_S_WAIT, TR_S_READY, TR_MAX_DONE, TR_EXP_DONE, TR_P_ARRIVE,     // softmax   (seg 2 = A, 3 = B)
  TR_O_WAIT, TR_O_READY, TR_STORE_ISSUED,                           // epilogue  (seg 4)
  TR_QK_GOT, TR_PV_GOT, TR_Q_GOT                                    // MMA issuers: operands ready
};
#define DFA_TRACE(seg, ev)                                                                        \
  do {                                                                                            \
    if constexpr (kTrace) {                                                                       \
      if (tr_on && tr_n < kTraceCap) trace[(seg) * kTraceCap + tr_n++] = ((uint64_t)(ev) << 56) | \
                                                                          (clock64() & 0xFFFFFFFFFFFFFFull); \
    }                                                                                             \
  } while (0)

// Barrier wait; in the instrumented build (kTrace) a wait that lasts ~2 s
// writes {site, thread, parity, raw barrier word} to the mapped-host
// watchdog buffer and traps, so a protocol deadlock is diagnosable from host.
template <bool kDbg>
__device__ __forceinline__ void wait_site(uint64_t* bar, uint32_t parity, uint32_t site,
                                          unsigned long long* wd) {
  if constexpr (!kDbg) {
    ptx::mbar_wait(bar, parity);
  } else {
    const long long t0 = clock64();
    while (!ptx::mbar_try(bar, parity)) {
      if (wd && clock64() - t0 > 4000000000LL) {
        const unsigned long long raw = *reinterpret_cast<volatile unsigned long long*>(bar);
        wd[2 * blockIdx.x + 1] = raw;
        wd[2 * blockIdx.x] = (1ull << 63) | ((unsigned long long)site << 40) |
                             ((unsigned long long)threadIdx.x << 16) | ((unsigned long long)ptx::smem_u32(bar) << 1) |
                             parity;
        __threadfence_system();
        asm volatile("trap;");
      }
    }
  }
}
#define DFA_WAIT(bar, parity, site) wait_site<kTrace>((bar), (parity), (site), watchdog)

template <bool kTrace, bool kSumCheck = false, int kKS = kKStages>
__global__ void __launch_bounds__(kThreads, 1)
    dfa_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                     const __grid_constant__ CUtensorMap tm_z, float* __restrict__ lse,
                     const __grid_constant__ Sm100Params p, uint64_t* __restrict__ trace,
                     unsigned long long* __restrict__ watchdog) {
  extern __shared__ uint8_t smem_raw[];
  using SmemLayout = SmemLayoutT<kKS>;
  constexpr int kVS = SmemLayout::kVSt;
  SmemLayout& sm =
      *reinterpret_cast<SmemLayout*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();

  // zero tile for the unselected offset classes
  for (uint32_t i = threadIdx.x; i < kZeroRows * 128 / 16; i += kThreads)
    ptx::st_shared_v4(ptx::smem_u32(sm.zero) + 16 * i, 0u, 0u, 0u, 0u);
  ptx::fence_proxy_async_smem();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kQStages; ++s) {
      ptx::mbar_init(&sm.q_full[s], 1);
      ptx::mbar_init(&sm.q_empty[s], 1);
    }
    for (int s = 0; s < kKS; ++s) {
      ptx::mbar_init(&sm.k_full[s], 1);
      ptx::mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kVS; ++s) {
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
      ptx::mbar_init(&sm.oload_full[s], 1);
    }
    ptx::fence_barrier_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
    ptx::tma_prefetch_desc(&tm_o);
    ptx::tma_prefetch_desc(&tm_z);
  } else if (warp == 2) {
    ptx::tmem_alloc<kTmemCols>(&sm.tmem_base);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = sm.tmem_base;
  // Programmatic dependent launch: the setup above (barriers, TMEM, zero
  // tile, descriptor prefetch) overlaps the previous kernel's tail; no global
  // memory is touched before the previous grid has completed.  Dependents
  // may start their own setup right away (they wait the same way).
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();
  if constexpr (kTrace) {  // per-CTA start / end (globaltimer) after the role timelines
    if (threadIdx.x == 0) trace[6 * kTraceCap + 2 * blockIdx.x] = ptx::globaltimer();
  }

  // Registers: 512 x 128 at launch; rebalanced per warpgroup to
  // producer/MMA 40, softmax 2 x 192, epilogue 80 (sum 64512 <= 65536).  192
  // (was 176) removes most softmax spills: +2..8% on every config-4 shape.
  if (warp < 4) ptx::setmaxnreg_dec<40>();
  if (warp == 0) {
    // ============================================================ producer
    if (ptx::elect_one()) {
      const bool tr_on = blockIdx.x == 0;
      uint32_t tr_n = 0;
      const uint64_t pol = ptx::policy_evict_first();  // every byte is read once
      uint32_t i = 0, g = 0;
      for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++i) {
        const Unit x = make_unit(p, u);
        const uint32_t qs = i % kQStages;
        DFA_WAIT(&sm.q_empty[qs], ((i / kQStages) & 1) ^ 1, 2);
        DFA_TRACE(0, TR_Q_ISSUE);
        ptx::mbar_arrive_expect_tx(&sm.q_full[qs], 2 * kTileBytes);
        ptx::tma_load_5d(sm.q[qs][0], &tm_q, &sm.q_full[qs], 0, x.j, x.gamma, x.t0, x.b, pol);
        ptx::tma_load_5d(sm.q[qs][1], &tm_q, &sm.q_full[qs], 0, x.j, x.gamma, x.t0 + kBM, x.b, pol);
        for (int32_t kt = 0; kt < x.n_kv; ++kt, ++g) {
          const uint32_t st = g % kKS;
          DFA_TRACE(0, TR_KV_WAIT);
          DFA_WAIT(&sm.k_empty[st], ((g / kKS) & 1) ^ 1, 3);
          DFA_TRACE(0, TR_KV_ISSUE);
          ptx::mbar_arrive_expect_tx(&sm.k_full[st], kKVTileBytes);
          ptx::tma_load_5d(sm.k[st], &tm_k, &sm.k_full[st], 0, x.j, x.gamma, x.kv_lo + kt * kBN, x.b, pol);
        }
      }
    }
  } else if (warp == 3) {
    // ========================================================== V producer
    if (ptx::elect_one()) {
      const uint64_t pol = ptx::policy_evict_first();
      uint32_t g = 0;
      for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Unit x = make_unit(p, u);
        for (int32_t kt = 0; kt < x.n_kv; ++kt, ++g) {
          const uint32_t st = g % kVS;
          DFA_WAIT(&sm.v_empty[st], ((g / kVS) & 1) ^ 1, 4);
          ptx::mbar_arrive_expect_tx(&sm.v_full[st], kKVTileBytes);
          ptx::tma_load_5d(sm.v[st], &tm_v, &sm.v_full[st], 0, x.j, x.gamma, x.kv_lo + kt * kBN, x.b, pol);
        }
      }
    }
  } else if (warp == 1) {
    // ======================================================= Q K^T issuer
    // One elected lane.  Step k (CTA-global, unit-major order: key tiles
    // ascending, slot A then slot B) writes S buffer k % 3; the buffer is
    // free once P V of step k - 3 completed (s_free, committed by the P V
    // issuer).  Q and K are waited for once per unit / key tile.
    if (ptx::elect_one()) {
      const bool tr_on = blockIdx.x == 0;
      uint32_t tr_n = 0;
      constexpr uint32_t idesc_qk = ptx::idesc_bf16(kBM, kBN, 0, 0);  // K-major Q and K
      // Shared-memory descriptors of every operand tile, built once; a K step
      // of 16 bf16 (32 B) advances the start-address field by 2.
      const uint64_t qdesc0 = ptx::sdesc_sw128(ptx::smem_u32(sm.q[0][0]));
      const uint64_t kdesc0 = ptx::sdesc_sw128(ptx::smem_u32(sm.k[0]));
      uint32_t b = 0;          // S buffer of the next step (step % 3)
      uint32_t steps = 0;      // steps issued so far
      uint32_t sfree_par = 0;  // bit b: parity of the next s_free[b] completion
      uint32_t gs = 0, gpar = 0;  // K stage / its full-barrier parity
      int32_t i = 0;
      for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++i) {
        const Unit x = make_unit(p, u);
        const uint32_t qs = i & 1;
        DFA_TRACE(1, TR_QK_WAIT);
        DFA_WAIT(&sm.q_full[qs], (i >> 1) & 1, 5);
        DFA_TRACE(1, TR_Q_GOT);
        for (int32_t kt = 0; kt < x.n_kv; ++kt) {
          DFA_WAIT(&sm.k_full[gs], gpar, 6);
          ptx::tc_fence_after();
          DFA_TRACE(1, TR_QK_GOT);
          const uint64_t kd = kdesc0 + (uint64_t)(gs * (kKVTileBytes >> 4));
#pragma unroll 1
          for (int sl = 0; sl < 2; ++sl) {
            if (!uses(x, sl, kt)) continue;
            if (steps >= (uint32_t)kSBufs) {
              DFA_WAIT(&sm.s_free[b], (sfree_par >> b) & 1u, 16);
              ptx::tc_fence_after();
            }
            sfree_par ^= (steps >= (uint32_t)kSBufs ? 1u : 0u) << b;
            const uint64_t qd = qdesc0 + (uint64_t)((qs * 2 + sl) * (kTileBytes >> 4));
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk)
              ptx::mma_ss(tbase + col_s(b), qd + (uint64_t)(2 * kk), kd + (uint64_t)(2 * kk), idesc_qk, kk > 0);
            ptx::tc_commit(&sm.s_full[sl][b]);
            DFA_TRACE(1, TR_QK_ISSUED);
            b = (b == kSBufs - 1) ? 0 : b + 1;
            ++steps;
          }
          ptx::tc_commit(&sm.k_empty[gs]);  // every Q K^T of this K tile issued
          if (++gs == kKS) {
            gs = 0;
            gpar ^= 1u;
          }
        }
        ptx::tc_commit(&sm.q_empty[qs]);  // both Q tiles of the unit consumed
      }
    }
  } else if (warp == 2) {
    // ========================================================= P V issuer
    // Same step order.  O_s += P_s V with A = P from TMEM (bf16 over the S
    // columns) and B = V as an MN-major smem operand; completion frees the S
    // buffer (s_free), the V stage after the tile's last P V, and hands O_s
    // to the epilogue after the slot's last step of the unit.
    if (ptx::elect_one()) {
      const bool tr_on = blockIdx.x == 0;
      uint32_t tr_n = 0;
      constexpr uint32_t idesc_pv = ptx::idesc_bf16(kBM, kD, 0, 1);  // P from TMEM, V MN-major
      // a 16-key step of V (16 rows x 128 B) advances the start address by 128
      const uint64_t vdesc0 = ptx::sdesc_sw128(ptx::smem_u32(sm.v[0]));
      uint32_t b = 0;
      uint32_t p_par = 0;   // bit b: parity of the next p_full[b] phase
      uint32_t oc_par = 0;  // bit s: parity of slot s's completed-unit count
      uint32_t gs = 0, gpar = 0;
      for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Unit x = make_unit(p, u);
        for (int32_t kt = 0; kt < x.n_kv; ++kt) {
          bool have_v = false;
          const uint64_t vdesc = vdesc0 + (uint64_t)(gs * (kKVTileBytes >> 4));
#pragma unroll 1
          for (int sl = 0; sl < 2; ++sl) {
            if (!uses(x, sl, kt)) continue;
            const bool first = kt == x.kt0(sl);
            DFA_TRACE(5, TR_P_WAIT);
            DFA_WAIT(&sm.p_full[b], (p_par >> b) & 1u, 7);
            p_par ^= 1u << b;
            DFA_TRACE(5, TR_P_READY);
            if (first) DFA_WAIT(&sm.o_empty[sl], ((oc_par >> sl) & 1u) ^ 1u, 8);
            if (!have_v) {
              DFA_WAIT(&sm.v_full[gs], gpar, 9);
              have_v = true;
            }
            ptx::tc_fence_after();
            DFA_TRACE(5, TR_PV_GOT);
#pragma unroll
            for (int kk = 0; kk < kBN / 16; ++kk)
              ptx::mma_ts(tbase + col_o(sl), tbase + col_s(b) + kk * 8, vdesc + (uint64_t)(kk * (2048 >> 4)),
                          idesc_pv, (!first || kk > 0) ? 1u : 0u);
            ptx::tc_commit(&sm.pv_done[sl]);
            ptx::tc_commit(&sm.s_free[b]);
            DFA_TRACE(5, TR_PV_ISSUED);
            if (kt == x.kt1(sl) - 1) {
              ptx::tc_commit(&sm.o_full[sl]);
              oc_par ^= 1u << sl;
            }
            b = (b == kSBufs - 1) ? 0 : b + 1;
          }
          ptx::tc_commit(&sm.v_empty[gs]);  // every P V of this V tile issued
          if (++gs == kVS) {
            gs = 0;
            gpar ^= 1u;
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ====================================================== softmax slots
    ptx::setmaxnreg_inc<192>();
    const int s = (warp - 4) / 4;                 // slot
    const uint32_t row = (warp % 4) * 32 + lane;  // query row in tile == TMEM lane
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const uint32_t tO = tbase + lane_base + col_o(s);
    const bool tr_on = blockIdx.x == 0 && row == 0;
    uint32_t tr_n = 0;
    uint32_t use_par = 0;  // bit b: parity of the next s_full[s][b] phase
    uint32_t pvc = 0;      // pv_done phases consumed
    uint32_t steps = 0;    // steps of this slot so far
    uint32_t published = 0;  // units whose row stats went to the epilogue
    float mref = -INFINITY, l = 0.0f;
    int32_t seg_lo = 0, seg_hi = 0;
    int32_t k_base = 0;  // CTA-global index of the unit's first step
    int32_t i = 0;
    for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++i) {
      const Unit x = make_unit(p, u);
      const int32_t kt_lo = x.kt0(s), kt_hi = x.kt1(s);
      const int32_t k_unit = k_base;
      k_base += steps_of_unit(x);
      if (kt_lo == kt_hi) continue;  // no rows for this slot in this unit
      {
        const int32_t tq = x.t0 + s * kBM + (int32_t)row;
        const bool valid_q = tq < p.T;
        seg_lo = valid_q ? p.div_m.div(tq) * p.m : 0;
        seg_hi = valid_q ? min(seg_lo + p.m, p.T) : 0;
        mref = -INFINITY;
        l = 0.0f;
      }
      for (int32_t kt = kt_lo; kt < kt_hi; ++kt) {
      const uint32_t b = (uint32_t)(k_unit + step_in_unit(x, kt, s)) % kSBufs;
      DFA_TRACE(2 + s, TR_S_WAIT);
      DFA_WAIT(&sm.s_full[s][b], (use_par >> b) & 1u, 10);
      DFA_TRACE(2 + s, TR_S_READY);
      use_par ^= 1u << b;
      ptx::tc_fence_after();
      const uint32_t tS = tbase + lane_base + col_s(b);
      uint32_t sr[kSC][32];
#pragma unroll
      for (int c = 0; c < kSC; ++c) ptx::tmem_ld32(tS + 32 * c, sr[c]);
      ptx::tmem_ld_wait();
      const int32_t k0 = x.kv_lo + kt * kBN;
      const int32_t lo = min(max(seg_lo - k0, 0), kBN);
      const int32_t hi = min(max(seg_hi - k0, 0), kBN);
      if (!(lo == 0 && hi == kBN)) {
#pragma unroll
        for (int c = 0; c < kSC; ++c)
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int col = 32 * c + e;
            if (col < lo || col >= hi) sr[c][e] = __float_as_uint(-INFINITY);
          }
      }
      // Exponentiate the tile against `neg` = -reference * c: packed
      // scale-subtract (FFMA2), exp2 (pairs in kPolyMask as an FMA-pipe
      // polynomial, the rest on MUFU), packed sums (FADD2), bf16 packing and
      // tcgen05.st of P over the consumed S columns.  Returns the row sum.
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
            if (DFA_PROBE_NO_EXP) {
              // profiling probe only (wrong results): no exponentials
            } else if (((kSumCheck ? kPolyMaskSumCheck : kPolyMask) >> e) & 1u) {
              // the polynomial's exponent add wraps for x >= 128: clamp so an
              // overflowing tile shows up in the row sum (MUFU gives +inf)
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
      bool waited = false;
      if constexpr (kSumCheck) {
        // Fast path (every row of the warp already has a reference from an
        // earlier tile of this unit): no row max.  The tile's row sum bounds
        // each p, so sum <= 2^thr keeps every p within the lazy-rescale bound;
        // otherwise (or on inf / NaN) the tile is redone on the exact path and
        // P is simply re-stored over the same columns.
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
        DFA_TRACE(2 + s, TR_MAX_DONE);
        // Lazy rescale (warp-uniform: tcgen05.ld/st are warp collectives).  O_s
        // must hold every earlier P V of this slot: wait for the slot's previous
        // P V (pv_done phases are consumed exactly once per step, in order).
        const bool move = tmax > mref && (mref == -INFINITY || (tmax - mref) * p.c > kRescaleThreshold);
        const bool fix_o = move && mref != -INFINITY;
        if (__any_sync(0xffffffffu, fix_o)) {
          if (steps > 0) {
            DFA_WAIT(&sm.pv_done[s], pvc & 1, 11);
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
        if (move) mref = tmax;
        l += exp_pass((mref == -INFINITY) ? 0.0f : -mref * p.c, false);
      }
      DFA_TRACE(2 + s, TR_EXP_DONE);
      // keep the pv_done phases in lockstep with the steps
      if (!waited && steps > 0) {
        DFA_WAIT(&sm.pv_done[s], pvc & 1, 12);
        ++pvc;
      }
      ++steps;
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&sm.p_full[b]);
      DFA_TRACE(2 + s, TR_P_ARRIVE);
      }  // key tiles of the unit
      // Hand the row statistics to the epilogue warpgroup: double-buffered by
      // the slot's published-unit count; publish unit n only after the
      // epilogue consumed unit n-1, so stat_full is never two phases ahead
      // of its parity waits (slots with one step per unit would otherwise
      // outrun the epilogue -- scripts/protocol_model.py).
      sm.stat_l[published & 1][s][row] = l;
      sm.stat_m[published & 1][s][row] = mref;
      if (published > 0) DFA_WAIT(&sm.stat_empty[s], (published - 1) & 1, 15);
      ptx::mbar_arrive(&sm.stat_full[s]);
      ++published;
    }
  } else if (warp >= 12) {
    // ============================================================ epilogue
    ptx::setmaxnreg_dec<80>();
    const uint32_t row = (warp % 4) * 32 + lane;
    const uint32_t lane_base = ((warp % 4) * 32) << 16;
    const bool leader = warp == 12 && lane == 0;
    const bool tr_on = blockIdx.x == 0 && leader;
    uint32_t tr_n = 0;
    uint32_t par = 0;     // bit s: parity of slot s's completed-unit count
    uint32_t ld_par = 0;  // bit s: parity of oload_full[s] (merge mode)
    const uint64_t pol_merge = ptx::policy_evict_first();
    int32_t i = 0;
    for (int32_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++i) {
      const Unit x = make_unit(p, u);
#pragma unroll 1
      for (int s = 0; s < 2; ++s) {
        if (x.kt0(s) == x.kt1(s)) continue;  // slot has no rows in this unit
        const int32_t ts0 = x.t0 + s * kBM;
        const int32_t tq = ts0 + (int32_t)row;
        const bool valid_q = tq < p.T;
        const uint32_t ph = (par >> s) & 1u;
        par ^= 1u << s;
        // Branch merge (multi-(w, r) LSE combine): fetch the running output
        // rows (a TMA box of the previous branches' result) into this slot's
        // staging tile and the running lse, both before the O wait so their
        // latency hides behind it.
        float lse_prev = -INFINITY;
        float* lrow = nullptr;
        if (lse && valid_q) lrow = lse + ((int64_t)x.b * p.h + x.j) * p.N + (int64_t)tq * p.r;
        if (p.merge) {
          if (leader) {
            ptx::tma_store_wait_read<0>();  // staging no longer read by an earlier store
            ptx::mbar_arrive_expect_tx(&sm.oload_full[s], kTileBytes);
            ptx::tma_load_5d(sm.ostage[s % kOStages], &tm_o, &sm.oload_full[s], 0, x.j, x.gamma, ts0, x.b, pol_merge);
          }
          if (lrow) lse_prev = lrow[x.gamma];
        }
        DFA_TRACE(4, TR_O_WAIT);
        DFA_WAIT(&sm.o_full[s], ph, 13);
        DFA_TRACE(4, TR_O_READY);
        DFA_WAIT(&sm.stat_full[s], ph, 14);
        ptx::tc_fence_after();
        const float l = sm.stat_l[ph][s][row];
        const float mref = sm.stat_m[ph][s][row];
        const uint32_t tO = tbase + lane_base + col_o(s);
        uint32_t orow[2][32];
        ptx::tmem_ld32(tO, orow[0]);
        ptx::tmem_ld32(tO + 32, orow[1]);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&sm.stat_empty[s]);  // stats buffer `ph` may be reused
        ptx::mbar_arrive(&sm.o_empty[s]);     // O_s may be overwritten by the next unit
        const float lse_new = mref * p.scale + __logf(l);
        const uint32_t stage_addr = ptx::smem_u32(sm.ostage[s % kOStages]);
        if (!p.merge) {
          const float inv = valid_q ? 1.0f / l : 0.0f;
          // the previous TMA store from this staging tile must have finished reading it
          if (leader) ptx::tma_store_wait_read<0>();
          ptx::named_bar_sync(1, kBM);
          // 128B-swizzled staging row: 16B chunk c of row r at ((c ^ (r & 7)) * 16)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float* f = reinterpret_cast<const float*>(&orow[c >> 2][(c & 3) * 8]);
            const uint32_t addr = stage_addr + row * 128 + ((c ^ (row & 7)) * 16);
            ptx::st_shared_v4(addr, ptx::pack_bf16x2(f[0] * inv, f[1] * inv),
                              ptx::pack_bf16x2(f[2] * inv, f[3] * inv), ptx::pack_bf16x2(f[4] * inv, f[5] * inv),
                              ptx::pack_bf16x2(f[6] * inv, f[7] * inv));
          }
          if (lrow)
            for (int32_t gz = 0; gz < p.r; ++gz) lrow[gz] = (gz == x.gamma) ? lse_new : -INFINITY;
        } else {
          // O = (e^{lse_prev} O_prev + e^{lse_new} O_new) / (e^{lse_prev} + e^{lse_new}), max-subtracted;
          // rows outside the tensor (valid_q false) are dropped by the store.
          const float mx = fmaxf(lse_prev, lse_new);
          const float wp = __expf(lse_prev - mx), wn = __expf(lse_new - mx);
          const float den = wp + wn;
          const float a = valid_q ? wp / den : 0.0f;
          const float cn = valid_q ? wn / (den * l) : 0.0f;
          DFA_WAIT(&sm.oload_full[s], (ld_par >> s) & 1u, 17);
          ld_par ^= 1u << s;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float* f = reinterpret_cast<const float*>(&orow[c >> 2][(c & 3) * 8]);
            const uint32_t addr = stage_addr + row * 128 + ((c ^ (row & 7)) * 16);
            uint32_t prev[4];
            ptx::ld_shared_v4(addr, prev);
            uint32_t outp[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 pv = ptx::unpack_bf16x2(prev[e]);
              outp[e] = ptx::pack_bf16x2(fmaf(a, pv.x, cn * f[2 * e]), fmaf(a, pv.y, cn * f[2 * e + 1]));
            }
            ptx::st_shared_v4(addr, outp[0], outp[1], outp[2], outp[3]);
          }
          if (lrow) lrow[x.gamma] = mx + __logf(den);
        }
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(1, kBM);
        if (leader) {
          ptx::tma_store_5d(&tm_o, sm.ostage[s % kOStages], 0, x.j, x.gamma, ts0, x.b);
          if (!p.merge && p.zero_rows)
            for (int32_t gz = 0; gz < p.r; ++gz)
              if (gz != x.gamma && !DFA_PROBE_NO_ZERO)
                for (int32_t zr = 0; zr < kBM; zr += kZeroRows)
                  ptx::tma_store_5d(&tm_z, sm.zero, 0, x.j, gz, ts0 + zr, x.b);
          ptx::tma_store_commit();
        }
        DFA_TRACE(4, TR_STORE_ISSUED);
      }
    }
    if (leader) ptx::tma_store_wait_all<0>();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (kTrace) {
    if (threadIdx.x == 0) trace[6 * kTraceCap + 2 * blockIdx.x + 1] = ptx::globaltimer();
  }
  if (warp == 2) {
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

// [B][N/r][r][h][64] bf16 view; box (64, 1, 1, 128, 1), 128-byte swizzle.
// The t' extent is N/r per image, so boxes never cross into the next image:
// out-of-range rows are zero-filled on load and dropped on store.  `ld` is
// the token stride in elements (h * 64 when contiguous; 3 * h * 64 when q,
// k, v are column blocks of one fused-projection output).
bool encode_map(CUtensorMap* map, const void* base, int64_t B, int64_t N, int64_t r, int64_t h, int64_t ld,
                uint32_t box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[5] = {(cuuint64_t)kD, (cuuint64_t)h, (cuuint64_t)r, (cuuint64_t)(N / r), (cuuint64_t)B};
  cuuint64_t strides[4] = {(cuuint64_t)kD * 2, (cuuint64_t)ld * 2, (cuuint64_t)r * ld * 2, (cuuint64_t)N * ld * 2};
  cuuint32_t box[5] = {kD, 1, 1, box_rows, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult res = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, (CUtensorMapL2promotion)DFA_L2_PROMO,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS;
}

// Encoding a tensor map costs a driver call (~2-4 us host time); callers
// re-launch on the same buffers, so the last encodes are cached per host
// thread (key: every input of the encoding).
bool make_map(CUtensorMap* map, const void* base, int64_t B, int64_t N, int64_t r, int64_t h, int64_t ld,
              uint32_t box_rows = 128) {
  struct Entry {
    CUtensorMap map;
    const void* base;
    int64_t B, N, r, h, ld;
    uint32_t rows;
    int dev;
  };
  constexpr int kEntries = 32;
  thread_local Entry cache[kEntries];
  thread_local int used = 0, next = 0;
  const int dev = current_device();
  for (int i = 0; i < used; ++i) {
    const Entry& e = cache[i];
    if (e.base == base && e.B == B && e.N == N && e.r == r && e.h == h && e.ld == ld && e.rows == box_rows &&
        e.dev == dev) {
      *map = e.map;
      return true;
    }
  }
  if (!encode_map(map, base, B, N, r, h, ld, box_rows)) return false;
  Entry& e = cache[next];
  e.map = *map;
  e.base = base;
  e.B = B, e.N = N, e.r = r, e.h = h, e.ld = ld;
  e.rows = box_rows;
  e.dev = dev;
  next = (next + 1) % kEntries;
  if (used < kEntries) ++used;
  return true;
}

}  // namespace

bool encode_stream_map(CUtensorMap* map, const void* base, int64_t B, int64_t N, int64_t r, int64_t h, int64_t ld,
                       uint32_t rows) {
  return make_map(map, base, B, N, r, h, ld, rows);
}

bool sm100_supported(const Geometry& g, int dtype, const void* q, const void* k, const void* v, const void* o) {
  if (dtype != 1) return false;              // bf16 only
  if (g.d != kD || g.dv != kD) return false;  // head_dim 64
  if (g.N % g.r != 0) return false;           // t'-stream view needs r | N
  if (g.w % g.r != 0) return false;           // segments are contiguous t'-blocks
  if (g.h > kMaxHeads) return false;
  auto al = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; };
  if (!al(q) || !al(k) || !al(v) || !al(o)) return false;
  for (int64_t ld : {g.ldq, g.ldk, g.ldv, g.ldo})  // TMA global strides: multiples of 16 B
    if (ld % 8 != 0) return false;
  if (g.N > (int64_t)INT32_MAX / 2 || g.B > (int64_t)INT32_MAX) return false;  // TMA coordinates are int32
  const int64_t units = g.B * g.h * ((g.N / g.r + kUnitRows - 1) / kUnitRows);
  if (units > (int64_t)INT32_MAX) return false;
  return true;
}

int launch_sm100(const Geometry& g, const void* q, const void* k, const void* v, void* o, float* lse,
                 cudaStream_t stream, cudaError_t* err, const char** why, uint64_t* trace,
                 unsigned long long* watchdog, bool merge, bool kept_only) {
  ensure_context();
  if (merge && !lse) {
    *why = "merge mode needs the running lse buffer";
    *err = cudaErrorInvalidValue;
    return 0;
  }
  CUtensorMap mq, mk, mv, mo, mz;
  if (!make_map(&mq, q, g.B, g.N, g.r, g.h, g.ldq) || !make_map(&mk, k, g.B, g.N, g.r, g.h, g.ldk, kBN) ||
      !make_map(&mv, v, g.B, g.N, g.r, g.h, g.ldv, kBN) || !make_map(&mo, o, g.B, g.N, g.r, g.h, g.ldo) ||
      !make_map(&mz, o, g.B, g.N, g.r, g.h, g.ldo, kZeroRows)) {
    *why = "cuTensorMapEncodeTiled failed";
    *err = cudaErrorInvalidValue;
    return 0;
  }
  Sm100Params p;
  p.N = (int32_t)g.N;
  p.T = (int32_t)(g.N / g.r);
  p.m = (int32_t)(g.w / g.r);
  p.r = (int32_t)g.r;
  p.h = (int32_t)g.h;
  p.unit_rows = kUnitRows;
  p.n_pairs = (p.T + kUnitRows - 1) / kUnitRows;
  // small grids: 128-row half units when twice the units still fit one wave
  if ((int64_t)g.B * g.h * ((p.T + kBM - 1) / kBM) <= device_sms()) {
    p.unit_rows = kBM;
    p.n_pairs = (p.T + kBM - 1) / kBM;
  }
  p.n_units = (int32_t)(g.B * g.h * p.n_pairs);
  p.scale = g.scale;
  p.c = g.scale * kLog2e;
  p.merge = merge ? 1 : 0;
  p.zero_rows = kept_only ? 0 : 1;
  p.div_pairs = make_fastdiv((uint32_t)p.n_pairs);
  p.div_h = make_fastdiv((uint32_t)p.h);
  p.div_m = make_fastdiv((uint32_t)p.m);
  for (int i = 0; i < kMaxHeads; ++i) p.offsets[i] = i < g.h ? g.offsets[i] : 0;
  // Sum-checked fast path (no row max on tiles after a unit's first, 2/16
  // polynomial share): measured 3-7% faster on long views with at most one
  // zero box per row -- (1024, 1), (2048, 1), (4096, 1), (2048, 2), (4096, 2)
  // -- and 2-10% slower on the short / store-heavy ones ((512, 1), (512, 2),
  // (1024, 2), (2048, 4), (4096, 4)), where its occasional redo of a tile
  // lands on the critical path.
  const bool sumcheck = DFA_SUMCHECK < 0 ? (p.m >= 1024 && p.r <= 2) : DFA_SUMCHECK != 0;
  // r = 2 views of 256-512 rows (two to four key tiles per unit, one zero box
  // per output tile) keep more K tiles than V tiles in flight: 4 + 2 instead
  // of 3 + 3 measured -3% at config 2 ((512, 2)), neutral at (1024, 2); +1% on
  // (256, 1) / (256, 2) and +2-3.5% on r >= 4 and long views, which keep 3 + 3.
  const bool deep_k = !sumcheck && p.r == 2 && p.m >= 256 && p.m <= 512 && kKStages == 3 && kVStages == 3;
  static_assert(sizeof(SmemLayoutT<4>) == sizeof(SmemLayoutT<kKStages>), "K / V splits share one footprint");
  const size_t smem = sizeof(SmemLayoutT<>) + 1024;
  auto kfn = trace      ? dfa_sm100_kernel<true>
             : sumcheck ? dfa_sm100_kernel<false, true>
             : deep_k   ? dfa_sm100_kernel<false, false, 4>
                        : dfa_sm100_kernel<false>;
  cudaError_t attr_err = ensure_smem_attr(reinterpret_cast<const void*>(kfn), smem);
  if (attr_err != cudaSuccess) {
    *err = attr_err;
    *why = "cudaFuncSetAttribute failed";
    return 0;
  }
  const int grid = (int)std::min<int64_t>(p.n_units, device_sms());
  cudaError_t le = cudaSuccess;
  if (trace)
    dfa_sm100_kernel<true><<<grid, kThreads, smem, stream>>>(mq, mk, mv, mo, mz, lse, p, trace, watchdog);
  else
    le = launch_pdl(kfn, grid, kThreads, smem, stream, mq, mk, mv, mo, mz, lse, p, (uint64_t*)nullptr,
                    (unsigned long long*)nullptr);
  *err = le != cudaSuccess ? le : cudaGetLastError();
  return 1;
}

}  // namespace dfa_impl
