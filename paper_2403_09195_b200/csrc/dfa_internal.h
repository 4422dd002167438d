// Internal declarations shared by the C-ABI layer (dfa_api.cpp) and the
// device kernels (dfa_simt.cu, dfa_sm100.cu).  Not installed.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdlib.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <vector>

namespace dfa_impl {

constexpr int kMaxHeads = 256;  // head offsets travel in the kernel parameter block

// Validated geometry of one dfa_forward call.
struct Geometry {
  int64_t B, N, w, r, h, d, dv;
  int64_t n_seg;  // ceil(N / w)            attention.hpp:35
  int64_t m_max;  // ceil(w / r): rows per full view
  float scale;    // 1/sqrt(d) or 1         attention.hpp:112-115
  int64_t ldq, ldk, ldv, ldo;  // token (row) strides in elements; h*d / h*dv when contiguous
  int32_t offsets[kMaxHeads];
};

// Bind the device's primary context to the calling thread (once per thread)
// before driver-API calls such as cuTensorMapEncodeTiled: a thread whose first
// CUDA call is one of those (e.g. PyTorch's autograd worker running a
// backward) has no current context otherwise.
inline void ensure_context() {
  static thread_local bool bound = false;
  if (!bound) {
    cudaFree(nullptr);
    bound = true;
  }
}

// Per-device facts.  A process may drive several GPUs (one host thread per
// device, or one thread switching devices), so every cache is keyed by the
// current device, never process-wide.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
inline int device_sms() {
  static std::atomic<int> cache[kMaxDevices];  // 0 = not queried yet
  const int dev = current_device();
  int n = (dev >= 0 && dev < kMaxDevices) ? cache[dev].load(std::memory_order_relaxed) : 0;
  if (n > 0) return n;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = 148;
  }
  if (dev >= 0 && dev < kMaxDevices) cache[dev].store(n, std::memory_order_relaxed);
  return n;
}
// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device attribute of
// the kernel: set it once per (kernel, device, size).
inline cudaError_t ensure_smem_attr(const void* fn, size_t smem) {
  struct Done {
    const void* fn;
    int dev;
    size_t smem;
  };
  static std::mutex mu;
  static std::vector<Done> done;
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(mu);
  for (const Done& d : done)
    if (d.fn == fn && d.dev == dev && d.smem >= smem) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) done.push_back({fn, dev, smem});
  return e;
}

// Launch with the programmatic-stream-serialization attribute (PDL): the
// kernel's prologue may overlap the previous kernel in the stream; kernels
// launched this way call griddepcontrol.wait before touching global memory.
// DFA_PDL=0 in the environment turns it off (measurement).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t stream,
                              Args... args) {
  static const bool on = [] {
    const char* e = getenv("DFA_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = on ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Generic SIMT kernel: any geometry, f32 (validation mode) or bf16 I/O,
// fp32 arithmetic, online softmax over key tiles.  Returns launches issued.
int launch_simt(const Geometry& g, int dtype, const void* q, const void* k, const void* v, void* o, float* lse,
                cudaStream_t stream, cudaError_t* err);

// [B][N/r][r][h][64] bf16 t'-stream tensor map (box 64 x rows, 128-byte
// swizzle), from a per-thread cache of recent encodes (dfa_sm100.cu).
bool encode_stream_map(CUtensorMap* map, const void* base, int64_t B, int64_t N, int64_t r, int64_t h, int64_t ld,
                       uint32_t rows);

// True when the tcgen05/TMA kernel covers this call.
bool sm100_supported(const Geometry& g, int dtype, const void* q, const void* k, const void* v, const void* o);

// tcgen05/TMEM/TMA kernel (bf16 in/out, fp32 accumulate).  Returns launches.
// trace: optional profiling buffer (6 x 4096 uint64 timeline events of CTA 0).
// merge: multi-(w, r) branch merge -- o and lse hold the running result of
// the earlier branches; the kept rows of this branch are LSE-combined into
// them in the epilogue (no zero boxes; lse required).
// kept_only: write the kept rows only -- the caller zero-fills the others
// (dfa_forward_host with a host-resident o).
int launch_sm100(const Geometry& g, const void* q, const void* k, const void* v, void* o, float* lse,
                 cudaStream_t stream, cudaError_t* err, const char** why, uint64_t* trace = nullptr,
                 unsigned long long* watchdog = nullptr, bool merge = false, bool kept_only = false);

// LSE-weighted combine of nb <= 8 branch outputs (dfa_combine.cu).
int launch_combine(int dtype, int64_t B, int64_t N, int64_t h, int64_t dv, int nb, const void* const* o,
                   const float* const* lse, void* out, float* lse_out, cudaStream_t stream, cudaError_t* err);
constexpr int kMaxBranches = 8;

// dfa_mb_sm100.cu: all branches of a multi-(w, r) set + their LSE combine in
// one persistent tcgen05 kernel.  Returns 1 (launched), 0 (set outside the
// kernel's envelope, why set, nothing launched), -1 (CUDA error, err set).
// steps_out (optional): 128x128 score tiles the launch computes.
constexpr int kMbMaxMaps = 4;     // distinct intervals in a set
constexpr int kMbMaxTiles = 64;   // key tiles per work unit
constexpr int kMbMaxGroups = 8;   // offset-class groups per query tile
void set_mb_trace(uint64_t* trace);  // profiling: trace CTA 0 of the next fused launches (nullptr = off)
int mb_plan_host(const Geometry* gb, int nb, int grid, void* out, size_t cap, int32_t* n_desc, int32_t* R,
                 int32_t* gr_shift, int32_t* desc_bytes, const char** why);
int launch_mb_sm100(const Geometry* gb, int nb, const void* q, const void* k, const void* v, void* o, float* lse,
                    cudaStream_t stream, cudaError_t* err, const char** why, int64_t* steps_out);

// Backward of the dilated core (dfa_bwd.cu): delta = workspace [B, h, N] fp32.
// allow_sm100: take the tcgen05 kernel (dfa_bwd_sm100.cu) when it covers the call.
int launch_backward(const Geometry& g, int dtype, const void* q, const void* k, const void* v, const void* o,
                    const void* dout, const float* lse, float* delta, void* dq, void* dk, void* dv,
                    cudaStream_t stream, cudaError_t* err, bool allow_sm100, const char** why);
bool bwd_sm100_supported(const Geometry& g, int dtype, const void* const* ptrs, int n_ptrs);
int launch_bwd_sm100(const Geometry& g, const void* q, const void* k, const void* v, const void* dout,
                     const float* lse, const float* delta, void* dq, void* dk, void* dv, cudaStream_t stream,
                     cudaError_t* err, const char** why);

// dfa_gemm.cu: row-major D = epi(A B + bias + beta C), strided batch (A rows
// at lda, batch stride sa; B at ldb / sb; C and D at ldc / ldd, batch stride
// sd); epi = GELU(erf) when gelu.  bf16 -> tcgen05 kernel, f32 -> SIMT
// (validation).  Returns 0 on failure (why set).
int gemm_rowmajor(int dtype, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int64_t sa, const void* B,
                  int64_t ldb, int64_t sb, void* D, int64_t ldd, int64_t sd, const void* C, int64_t ldc, float beta,
                  const void* bias, int batch, cudaStream_t stream, const char** why, bool gelu = false);
void set_gemm_tile(int bn);  // measurement: force the GEMM tile width (0 = auto)
// dfa_layers.cu: LayerNorm (eps 1e-5) and erf-GELU kernels, weight packing.
int launch_layer_norm(int dtype, const void* x, const void* g, const void* b, void* y, int64_t rows, int cols,
                      cudaStream_t stream);
int launch_gelu(int dtype, const void* xin, void* x, int64_t n, cudaStream_t stream);  // x = GELU(xin); may alias
// wq/wk/wv [h, D, d] -> packed [D, 3, h, d] (one QKV GEMM writes q|k|v per token).
// Offset-class packing for the class-split multi-head path: q/k/v columns and
// wo rows in class-major head order (heads grouped by offset).  Returns launches.
int launch_pack_class(int dtype, const void* wq, const void* wk, const void* wv, const void* wo, void* qkv_out,
                      void* wo_out, int64_t h, int64_t D, int64_t d, const int32_t* offsets, cudaStream_t stream);
int launch_pack_qkv(int dtype, const void* wq, const void* wk, const void* wv, void* out, int64_t h, int64_t D,
                    int64_t d, cudaStream_t stream);

// Fault hook (attention.hpp:272): out[0] += 1e-3.
int launch_perturb(int dtype, void* o, cudaStream_t stream);

}  // namespace dfa_impl
