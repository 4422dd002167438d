// Memory-pipeline ceiling of the forward's access pattern, with no compute:
// a persistent kernel (one CTA per SM, the same units and head-major order as
// dfa_sm100_kernel) TMA-loads each unit's Q (2 tiles), K and V (m/128 tiles
// each) from the [B][N/r][r][h][64] t'-stream view and TMA-stores 2 output
// tiles + (r - 1) x 2 zero boxes -- exactly the forward's algorithmic bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2403_09195_b200/csrc \
//        -o scripts/micro/tma_stream scripts/micro/tma_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "sm100_ptx.cuh"

using namespace dfa_impl;
constexpr int kTile = 128 * 128;
constexpr int kStages = 12;

struct P {
  int T, m, r, h, n_pairs, n_units;
};

__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap tq,
                                                        const __grid_constant__ CUtensorMap tk,
                                                        const __grid_constant__ CUtensorMap tv,
                                                        const __grid_constant__ CUtensorMap to, const P p) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* zero = base + kStages * kTile;
  __shared__ uint64_t full[kStages];
  for (int i = threadIdx.x; i < kTile / 16; i += blockDim.x) ptx::st_shared_v4(ptx::smem_u32(zero) + 16 * i, 0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) ptx::mbar_init(&full[s], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint64_t pol = ptx::policy_evict_first();
  uint32_t g = 0;  // tiles loaded so far (ring position)
  const int kv_tiles = p.m >= 256 ? 2 : 1;
  const int n_loads = 2 + 2 * kv_tiles;  // Q_A, Q_B, K..., V...
  // software-pipelined: unit i+1's loads are issued before unit i's stores
  auto issue = [&](int u) {
    const int j = u % p.h, bp = u / p.h, pair = bp % p.n_pairs, b = bp / p.n_pairs;
    const int gamma = j % p.r, t0 = pair * 256;
    for (int l = 0; l < n_loads; ++l, ++g) {
      const int st = g % kStages;
      if (g >= kStages) ptx::tma_store_wait_read<0>();
      ptx::mbar_arrive_expect_tx(&full[st], kTile);
      const CUtensorMap* m = l < 2 ? &tq : (l < 2 + kv_tiles ? &tk : &tv);
      const int row = l < 2 ? t0 + 128 * l : t0 + 128 * ((l - 2) % kv_tiles);
      ptx::tma_load_5d(base + st * kTile, m, &full[st], 0, j, gamma, row, b, pol);
    }
  };
  uint32_t first = 0;
  if ((int)blockIdx.x < p.n_units) issue(blockIdx.x);
  for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
    const uint32_t cur = first;
    if (u + (int)gridDim.x < p.n_units) issue(u + gridDim.x);
    first += n_loads;
    const int j = u % p.h, bp = u / p.h, pair = bp % p.n_pairs, b = bp / p.n_pairs;
    const int gamma = j % p.r, t0 = pair * 256;
    for (int l = 0; l < n_loads; ++l) {
      const uint32_t gg = cur + l;
      ptx::mbar_wait(&full[gg % kStages], (gg / kStages) & 1);
      if (l < 2) {
        ptx::tma_store_5d(&to, base + (gg % kStages) * kTile, 0, j, gamma, t0 + 128 * l, b);
        for (int gz = 0; gz < p.r; ++gz)
          if (gz != gamma) ptx::tma_store_5d(&to, zero, 0, j, gz, t0 + 128 * l, b);
      }
    }
    ptx::tma_store_commit();
  }
  ptx::tma_store_wait_all<0>();
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void map(Enc enc, CUtensorMap* mp, void* ptr, long B, long N, long r, long h) {
  cuuint64_t dims[5] = {64, (cuuint64_t)h, (cuuint64_t)r, (cuuint64_t)(N / r), (cuuint64_t)B};
  const long ld = h * 64;
  cuuint64_t strides[4] = {128, (cuuint64_t)ld * 2, (cuuint64_t)(r * ld * 2), (cuuint64_t)(N * ld * 2)};
  cuuint32_t box[5] = {64, 1, 1, 128, 1}, es[5] = {1, 1, 1, 1, 1};
  enc(mp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  Enc enc = (Enc)fn;
  const long B = 64, N = 4096, h = 6;
  const size_t bytes = (size_t)B * N * h * 64 * 2;
  void *q, *k, *v, *o;
  cudaMalloc(&q, bytes); cudaMalloc(&k, bytes); cudaMalloc(&v, bytes); cudaMalloc(&o, bytes);
  cudaMemset(q, 0, bytes); cudaMemset(k, 0, bytes); cudaMemset(v, 0, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = (kStages + 1) * kTile + 1024;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int r : {2, 8, 1}) {
    const int w = r == 1 ? 2048 : (r == 2 ? 512 : 256);
    CUtensorMap tq, tk, tv, to;
    map(enc, &tq, q, B, N, r, h); map(enc, &tk, k, B, N, r, h); map(enc, &tv, v, B, N, r, h); map(enc, &to, o, B, N, r, h);
    P p;
    p.T = N / r; p.m = w / r; p.r = r; p.h = h; p.n_pairs = (p.T + 255) / 256; p.n_units = B * h * p.n_pairs;
    for (int it = 0; it < 3; ++it) stream_kernel<<<sms, 128, smem>>>(tq, tk, tv, to, p);
    cudaEvent_t a, bb; cudaEventCreate(&a); cudaEventCreate(&bb);
    cudaEventRecord(a);
    for (int it = 0; it < 20; ++it) stream_kernel<<<sms, 128, smem>>>(tq, tk, tv, to, p);
    cudaEventRecord(bb); cudaEventSynchronize(bb);
    float ms; cudaEventElapsedTime(&ms, a, bb); ms /= 20;
    // algorithmic bytes of the forward: kept q/k/v rows + full output (the probe reads K/V once per unit pair
    // like the kernel: for m >= 256 each unit reads 2 K + 2 V tiles)
    const double rd = (double)p.n_units * (2 + 2 * (p.m >= 256 ? 2 : 1)) * kTile;
    const double wr = (double)bytes;
    printf("r=%d w=%d: %.1f us, read %.0f MB write %.0f MB -> %.0f GB/s (%s)\n", r, w, ms * 1e3, rd / 1e6, wr / 1e6,
           (rd + wr) / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
