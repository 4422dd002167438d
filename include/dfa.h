/* include/dfa.h -- C-ABI of the B200-native Dilated Flash Attention forward.
 *
 * Drop-in boundary for the reference's hot path
 *   attnkit::dilated_attention<S>(q, k, v, cfg, head_offset, workers)
 *     (/root/reference/proj/include/attnkit/attention.hpp:280-301)
 * and the helpers it is built from (AttentionConfig::validate :44-65,
 * make_segment_view :84-98, flop_count :370-387, the recompose fault hook
 * :237-241).  The reference exposes a header-only C++ template API with no
 * FFI; these entry points are what an FFI for that path binds (plain
 * pointers and sizes, no C++ or torch types).  include/dfa.hpp rebuilds the
 * reference-shaped C++ API (same names, same exception types) on top.
 *
 * Tensor layout (all device entry points): q, k are [B, N, h, d] and v, o are
 * [B, N, h, d_v], row-major and contiguous -- i.e. per image the reference's
 * multi-head concat layout [N, h*d] (attention.hpp:350-357).  The single-head
 * reference call is B = 1, h = 1.  Head j uses offset head_offsets[j]; rows
 * selected by no view of head j are written as exact zeros (attention.hpp:
 * 243-245, 270).
 *
 * Ownership: the caller owns every buffer; no entry point allocates device
 * memory on the hot path (dfa_workspace_* is the explicit exception, created
 * once up front).  Threading: reentrant and stream-ordered; the only global
 * state is the fault-injection flag (mirrors attention.hpp:240).
 */
#ifndef DFA_H_
#define DFA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error taxonomy: 1:1 with the reference's exception types
 * (common.hpp:13-30 and std::out_of_range at attention.hpp:87-90,287-288). */
typedef enum {
  DFA_OK = 0,
  DFA_ERR_CONFIG = 1,       /* attnkit::config_error    */
  DFA_ERR_DIMENSION = 2,    /* attnkit::dimension_error */
  DFA_ERR_OUT_OF_RANGE = 3, /* std::out_of_range        */
  DFA_ERR_CONTRACT = 4,     /* attnkit::contract_error  */
  DFA_ERR_CUDA = 5,         /* CUDA runtime/driver failure (no reference analogue) */
  DFA_ERR_UNSUPPORTED = 6,  /* valid config outside what the device kernels implement */
  DFA_ERR_IO = 7            /* attnkit::io_error (DTNSR1 tensor files)  */
} dfa_status_t;

/* F64: the reference's double instantiation (attention.hpp with Scalar =
 * double) -- forward only, on the SIMT kernel with double arithmetic. */
typedef enum { DFA_F32 = 0, DFA_BF16 = 1, DFA_F64 = 2 } dfa_dtype_t;

/* attention.hpp:15 Kernel{naive, tiled}.  Validated exactly as the reference
 * does (tile_size >= 1 when tiled); on the GPU every kernel streams keys in
 * tiles, so the flag selects nothing else. */
typedef enum { DFA_KERNEL_NAIVE = 0, DFA_KERNEL_TILED = 1 } dfa_kernel_t;

/* Which device path dfa_forward takes for a given call (dfa_query_path). */
typedef enum {
  DFA_PATH_NONE = 0,
  DFA_PATH_SM100_TCGEN05 = 1, /* bf16, TMA + tcgen05/TMEM (sm_100a)          */
  DFA_PATH_SIMT = 2           /* f32 validation / general-geometry kernel    */
} dfa_path_t;

/* attention.hpp:24-33 AttentionConfig. */
typedef struct {
  int64_t seq_len;             /* N                                         */
  int64_t segment_len;         /* w                                         */
  int64_t interval;            /* r                                         */
  int64_t num_heads;           /* h                                         */
  int64_t head_dim;            /* d   (q/k width)                           */
  int64_t value_dim;           /* d_v (v/o width); 0 means d_v = d          */
  const int64_t* head_offsets; /* h offsets gamma_j in [0, r)               */
  int32_t kernel;              /* dfa_kernel_t                              */
  int64_t tile_size;           /* tiled kernel only                         */
  int32_t scale_scores;        /* nonzero: scores *= 1/sqrt(d) after q.k    */
} dfa_config_t;

/* Thread-local message of the last failing call on this thread (the text the
 * reference's exception would carry, common.hpp:50-55 msg()). */
const char* dfa_last_error(void);

/* attention.hpp:44-65 AttentionConfig::validate(require_full_coverage). */
dfa_status_t dfa_validate(const dfa_config_t* cfg, int32_t require_full_coverage);

/* attention.hpp:84-98 make_segment_view: global rows {i*w+g, i*w+g+r, ...}
 * clipped to segment i.  Writes min(count, cap) indices; *count = full count.
 * Errors: DFA_ERR_OUT_OF_RANGE for a bad segment index or offset. */
dfa_status_t dfa_segment_view(int64_t seq_len, int64_t segment_len, int64_t interval, int64_t segment_index,
                              int64_t offset, int64_t* rows, int64_t cap, int64_t* count);

/* attention.hpp:370-387 flop_count (multiplications only). */
dfa_status_t dfa_flop_count(const dfa_config_t* cfg, uint64_t* dense_mults, uint64_t* dilated_mults,
                            double* ratio);

/* Device path dfa_forward would take (no launch).  *path = dfa_path_t. */
dfa_status_t dfa_query_path(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, int32_t* path);

/* Batched multi-head forward on DEVICE pointers (attention.hpp:280-301 run
 * for every image b and head j with gamma_j = head_offsets[j]).
 *   q, k: [B, N, h, d]; v, o: [B, N, h, d_v] of `dtype`;
 *   lse : optional fp32 [B, h, N] (natural-log log-sum-exp of the scaled
 *         scores of each kept row; -inf for rows no view selects).  NULL = off.
 *   stream: a cudaStream_t (NULL = legacy default stream).
 * Stream-ordered: returns after the launch, not after completion. */
dfa_status_t dfa_forward(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q, const void* k,
                         const void* v, void* o, float* lse, void* stream);

/* dfa_forward with explicit token (row) strides in elements: q row n of
 * image b at q + (b * N + n) * ldq (heads contiguous inside the row), same
 * for k / v / o.  ldq, ldk >= h * d; ldv, ldo >= h * d_v.  Lets the core read
 * q, k, v as column blocks of one fused QKV projection ([B, N, 3, h, d]:
 * ld = 3 h d) without a split pass. */
dfa_status_t dfa_forward_strided(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q,
                                 int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* o,
                                 int64_t ldo, float* lse, void* stream);

/* Reference-shaped single-head call on HOST buffers, synchronous:
 * q, k [N x d], v [N x d_v] -> out [N x d_v] (attention.hpp:280-282).
 * `workers` is accepted and ignored (the GPU grid replaces parallel_for).
 * Uses `ws` (see below) for device staging. */
typedef struct dfa_workspace dfa_workspace_t;
dfa_status_t dfa_workspace_create(size_t bytes, dfa_workspace_t** ws);
dfa_status_t dfa_workspace_destroy(dfa_workspace_t* ws);
dfa_status_t dfa_dilated_attention_host(const dfa_config_t* cfg, dfa_dtype_t dtype, const void* q, const void* k,
                                        const void* v, int64_t head_offset, int32_t workers, void* out,
                                        dfa_workspace_t* ws);

/* Batched forward on HOST buffers (the end-to-end call): q, k, v reach the
 * device, dfa_forward runs, o (and lse if non-NULL) come back, then a stream
 * synchronize -- pipelined over image chunks on two copy streams.  When q, k, v
 * are pinned (mapped) host memory and the call takes the tcgen05 path, the
 * kernel TMA-reads only the kept rows straight from host memory over PCIe
 * (no staging copy; dfa_host_transfer_bytes reports the bytes); otherwise
 * they are copied in.  When o is pinned mapped memory too, the kernel writes
 * the kept output rows straight into it and host threads zero-fill the rest
 * (dfa_set_host_kept_out); otherwise o comes back by chunked D2H copies.
 * Pageable buffers work, slower. */
dfa_status_t dfa_forward_host(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q,
                              const void* k, const void* v, void* o, float* lse, dfa_workspace_t* ws,
                              void* stream);

/* attention.hpp:237-241 fault::recompose_perturb: when armed, every forward
 * adds 1e-3 to output element 0 so the parity harness demonstrably fails. */
void dfa_set_fault_perturb(int32_t armed);
int32_t dfa_get_fault_perturb(void);

/* Zero-copy input mode of dfa_forward_host (default on; 0 forces the copy-in
 * pipeline).  Process-wide. */
void dfa_set_host_zero_copy(int32_t enabled);
/* Output mode of dfa_forward_host when o is also pinned mapped host memory
 * (default on): the kernel writes the kept rows straight into o over PCIe
 * and host threads zero-fill the rows no view keeps, so only kept output
 * rows cross the bus; 0 = device output + chunked D2H copies.  Process-wide. */
void dfa_set_host_kept_out(int32_t enabled);
/* Bytes dfa_forward_host moves host->device (h2d) and device->host (d2h) for
 * these buffers: kept rows of q, k, v in zero-copy mode, whole tensors
 * otherwise; kept rows of o when o is written in place (kept-out mode), the
 * whole of o otherwise (o may be null: counted as not mapped). */
dfa_status_t dfa_host_transfer_bytes(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q,
                                     const void* k, const void* v, const void* o, int32_t with_lse, size_t* h2d,
                                     size_t* d2h);

/* Bytes a dfa_forward_host call needs in its workspace. */
dfa_status_t dfa_workspace_bytes(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, int32_t with_lse,
                                 size_t* bytes);

/* Test hook: 0 = automatic dispatch (default), DFA_PATH_SIMT = force the SIMT
 * kernel, DFA_PATH_SM100_TCGEN05 = require the tcgen05 kernel (calls it does
 * not cover fail with DFA_ERR_UNSUPPORTED).  Process-wide. */
void dfa_set_path_override(int32_t path);

/* EXTENSION (no reference analogue; SPEC.md:204 lists multi-(w, r) as a
 * non-goal): several (w, r) branches over the same q, k, v, combined row by
 * row with weights e^{lse_b} (each branch's log-sum-exp), i.e. one softmax over
 * the union of the branches' key sets.  `base` supplies N, h, d, d_v,
 * scale_scores; branch b supplies (w_b, r_b, head_offsets_b).  Rows no branch
 * selects are 0.  With one branch the output equals dfa_forward bit for bit.
 * `workspace` (device) must hold dfa_multibranch_workspace_bytes bytes. */
typedef struct {
  int64_t segment_len;          /* w_b */
  int64_t interval;             /* r_b */
  const int64_t* head_offsets;  /* h offsets in [0, r_b) */
} dfa_branch_t;
dfa_status_t dfa_multibranch_workspace_bytes(const dfa_config_t* base, int32_t n_branches, dfa_dtype_t dtype,
                                             int64_t batch, size_t* bytes);
dfa_status_t dfa_forward_multibranch(const dfa_config_t* base, int32_t n_branches, const dfa_branch_t* branches,
                                     dfa_dtype_t dtype, int64_t batch, const void* q, const void* k, const void* v,
                                     void* o, float* lse, void* workspace, size_t workspace_bytes, void* stream);

/* Test / measurement hook for dfa_forward_multibranch (bf16, 2+ branches):
 * DFA_MB_AUTO (default) runs every branch and the combine in one tcgen05
 * kernel when the set fits it (intervals dividing their segment lengths,
 * <= 4 distinct intervals, lcm | N; else per-branch launches);
 * DFA_MB_PER_BRANCH forces one launch per branch with the LSE merge in each
 * epilogue.  Process-wide. */
enum { DFA_MB_AUTO = 0, DFA_MB_PER_BRANCH = 1 };
void dfa_set_multibranch_mode(int32_t mode);
/* Profiling hook: while `trace` (device, 6 x 4096 + 2 x #SMs uint64) is non-NULL, fused
 * multi-branch launches record CTA 0's timeline into it (dfa_forward_traced's
 * format; scripts/trace_timeline.py decodes it). */
void dfa_set_multibranch_trace(uint64_t* trace);
/* Test hook (host only, no CUDA call): the work-unit schedule the fused
 * multi-branch kernel uses for a branch set -- *n_desc descriptors of
 * *desc_bytes bytes each (layout: csrc/dfa_mb_sm100.cu MbDesc) copied into
 * `descs` (up to `capacity` bytes), the lcm R of the intervals and log2 of the
 * rows per offset-class group.  DFA_ERR_UNSUPPORTED when the set is outside
 * the fused kernel's envelope. */
dfa_status_t dfa_multibranch_plan(const dfa_config_t* base, int32_t n_branches, const dfa_branch_t* branches,
                                  int64_t batch, int32_t grid, void* descs, size_t capacity, int32_t* n_desc,
                                  int32_t* lcm_interval, int32_t* rows_per_group_log2, int32_t* desc_bytes);

/* Backward of the dilated core (the reference computes
 * it on its autodiff tape for the dilated branch of detail::attention_mix,
 * encoder.hpp:204-219, ops autodiff.hpp:99-179, 269-289): gradients of a loss
 * w.r.t. q, k, v given dO = dloss/do.  o and lse are dfa_forward's outputs for
 * the same inputs (lse required).  Layouts as dfa_forward; dq, dk [B,N,h,d],
 * dv [B,N,h,d_v]; rows no view selects get 0.  `workspace` (device) holds
 * dfa_backward_workspace_bytes bytes (per-row dO . O).  Deterministic. */
dfa_status_t dfa_backward_workspace_bytes(const dfa_config_t* cfg, int64_t batch, size_t* bytes);
dfa_status_t dfa_backward(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* q, const void* k,
                          const void* v, const void* o, const float* lse, const void* dout, void* dq, void* dk,
                          void* dv, void* workspace, size_t workspace_bytes, void* stream);

/* tensor.hpp:175-195 matmul (row-major, C = A B) on device buffers, with the
 * layers' epilogue: D[b] = epi(A[b] B[b] + bias + beta C[b]) for b < batch;
 * A [M, K] (row stride lda, batch stride sa), B [K, N] (ldb, sb), C / D
 * [M, N] (ldc / ldd, batch stride sd); bias [N] or NULL; C NULL for none;
 * gelu != 0 applies GELU in the reference's erf form (tensor.hpp:262-265).
 * bf16: the tcgen05 kernel (fp32 accumulate); f32: the SIMT validation
 * kernel (FFMA, no TF32).  Strides in elements; the building block of the
 * projections below, exported for parity tests. */
/* Measurement knob: force dfa_gemm's tile width (64 / 128 / 192 / 256; 0 = the
 * dispatcher's choice).  Process-wide; not for production use. */
void dfa_set_gemm_tile(int32_t bn);
dfa_status_t dfa_gemm(dfa_dtype_t dtype, int64_t batch, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                      int64_t sa, const void* B, int64_t ldb, int64_t sb, void* D, int64_t ldd, int64_t sd,
                      const void* C, int64_t ldc, float beta, const void* bias, int32_t gelu, void* stream);

/* attention.hpp:340-360 multi_head_dilated for a batch: x [B, N, D] with
 * D = h * d; wq, wk, wv [h, D, d] (the reference's per-head D x d
 * projections, stacked); wo [D, D]; out [B, N, D] = concat_j(head_j) wo,
 * head_j = dilated_attention(x wq_j, x wk_j, x wv_j) at offset gamma_j.
 * Requires full coverage (attention.hpp:343).  All tensors `dtype`, device.
 * The projections run as this library's own tcgen05 GEMM (dfa_gemm.cu)
 * against the weights packed [D, 3, h, d] (bf16 with r > 1: per offset class,
 * 1/r of the rows); the core reads q / k / v straight out of its output and
 * writes the concat layout the output projection consumes.  `workspace`
 * holds dfa_multi_head_workspace_bytes. */
dfa_status_t dfa_multi_head_workspace_bytes(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch,
                                            size_t* bytes);
dfa_status_t dfa_multi_head_dilated(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* x,
                                    const void* wq, const void* wk, const void* wv, const void* wo, void* out,
                                    void* workspace, size_t workspace_bytes, void* stream);

/* The same on HOST buffers, synchronous (device staging in `ws`, sized by
 * dfa_multi_head_host_workspace_bytes): the call include/dfa.hpp's
 * reference-shaped dfa::multi_head_dilated makes. */
dfa_status_t dfa_multi_head_host_workspace_bytes(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch,
                                                 size_t* bytes);
dfa_status_t dfa_multi_head_dilated_host(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* x,
                                         const void* wq, const void* wk, const void* wv, const void* wo, void* out,
                                         dfa_workspace_t* ws);

/* One pre-norm encoder block (encoder.hpp:241-248; parameters as
 * init_encoder_params names them, :287-304): x1 = x + attention_mix(LN1(x))
 * (attention_mix = multi_head_dilated + bias bo, encoder.hpp:189-223);
 * out = x1 + GELU(LN2(x1) w1 + b1) w2 + b2, GELU the erf form
 * (tensor.hpp:262-265), LayerNorm eps 1e-5 with population variance. */
typedef struct {
  const void *ln1_g, *ln1_b;   /* [D] */
  const void *wq, *wk, *wv;    /* [h, D, d] */
  const void *wo, *bo;         /* [D, D], [D] */
  const void *ln2_g, *ln2_b;   /* [D] */
  const void *w1, *b1;         /* [D, hidden], [hidden] */
  const void *w2, *b2;         /* [hidden, D], [D] */
  int64_t hidden;              /* mlp width (mlp_ratio * D) */
} dfa_block_weights_t;
dfa_status_t dfa_encoder_block_workspace_bytes(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch,
                                               int64_t hidden, size_t* bytes);
dfa_status_t dfa_encoder_block_forward(const dfa_config_t* cfg, dfa_dtype_t dtype, int64_t batch, const void* x,
                                       const dfa_block_weights_t* weights, void* out, void* workspace,
                                       size_t workspace_bytes, void* stream);

/* Profiling hook: dfa_forward (bf16, tcgen05 path only) of a build of the
 * kernel that records a timeline of CTA 0 into `trace` (6 x 4096 uint64, then each
 * CTA's start / end %globaltimer at [6 x 4096 + 2 cta]: 6 x 4096 + 2 x #SMs entries;
 * per role producer / QK issuer / softmax A / softmax B / epilogue / PV issuer, entries
 * (event << 56) | clock64).  scripts/trace_timeline.py decodes it. */
dfa_status_t dfa_forward_traced(const dfa_config_t* cfg, int64_t batch, const void* q, const void* k, const void* v,
                                void* o, uint64_t* trace, void* stream);

/* Debug hook: as dfa_forward_traced, plus a deadlock watchdog -- a barrier
 * wait lasting ~2 s writes {site, thread, parity, barrier word} per CTA into
 * `watchdog` (2 x gridDim uint64, host-mapped memory) and traps. */
dfa_status_t dfa_forward_debug(const dfa_config_t* cfg, int64_t batch, const void* q, const void* k, const void* v,
                               void* o, uint64_t* trace, unsigned long long* watchdog, void* stream);

/* DTNSR1 tensor files (tensor_io.hpp:15-19, 52-156): the reference's on-disk
 * format for golden vectors and datasets.  dtype codes 0 = f32, 1 = f64;
 * rank <= 8; dims are written as uint32 little-endian.  Errors: DFA_ERR_IO
 * with the reference's io_error text ("bad magic in tensor file: ...",
 * "truncated tensor file: ...", "unknown dtype code ..."). */
dfa_status_t dfa_tensor_header(const char* path, int32_t* dtype, int32_t* rank, int64_t* dims /* [8] */);
/* load_tensor<Scalar> (:147-153): payload converted to `dtype` (f32 <-> f64
 * like read_payload's cast); `capacity` = scalars `out` can hold. */
dfa_status_t dfa_tensor_load(const char* path, int32_t dtype, void* out, int64_t capacity);
/* save_tensor (:86-91) / write_tensor (:52-84). */
dfa_status_t dfa_tensor_save(const char* path, int32_t dtype, int32_t rank, const int64_t* dims, const void* data);

/* Number of device kernels the last dfa_forward on this thread launched
 * (evidence for bench.py's gpu_launches). */
int32_t dfa_last_launch_count(void);

/* Library version, e.g. 100 = 0.1.0. */
int32_t dfa_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DFA_H_ */
