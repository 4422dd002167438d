// Micro-benchmark: does the bf16 pack (F2FP.BF16.F32.PACK_AB, cvt.rn.bf16x2.f32)
// share the XU pipe with MUFU.EX2?  Throughput per SM of: ex2 alone, F2FP
// alone, the softmax mix (2 ex2 + 1 pack per pair), PRMT packing alone, and
// the softmax mix with PRMT-based packing.  Decides how P is packed in the
// forward's softmax.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 2048;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// mode 0: ex2 only; 1: pack only; 2: 2 ex2 + 1 pack; 3: prmt only; 4: 2 ex2 + prmt (+2 iadd rounding)
template <int MODE>
__global__ void k(float* out, float seed) {
  float x[8];
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + i) * 1e-9f - 0.5f;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      if (MODE == 0) {
        x[i] = ex2(x[i]);
        x[i + 1] = ex2(x[i + 1]);
      } else if (MODE == 1) {
        acc += pack(x[i], x[i + 1]);
        x[i] = __uint_as_float(__float_as_uint(x[i]) ^ acc);
      } else if (MODE == 2) {
        x[i] = ex2(x[i]);
        x[i + 1] = ex2(x[i + 1]);
        acc ^= pack(x[i], x[i + 1]);
      } else if (MODE == 3) {
        acc += prmt(__float_as_uint(x[i]), __float_as_uint(x[i + 1]));
        x[i] = __uint_as_float(__float_as_uint(x[i]) ^ acc);
      } else {
        x[i] = ex2(x[i]);
        x[i + 1] = ex2(x[i + 1]);
        acc ^= prmt(__float_as_uint(x[i]) + 0x8000u, __float_as_uint(x[i + 1]) + 0x8000u);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f || acc == 0x12345u) out[0] = s + acc;
}

template <int MODE>
void run(const char* name, double pairs_per_iter) {
  float* out;
  cudaMalloc(&out, 4);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  dim3 grid(sms * 4), block(256);
  k<MODE><<<grid, block>>>(out, 1.0f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<grid, block>>>(out, 1.0f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double pairs = (double)grid.x * block.x * kIters * pairs_per_iter;
  const double per_clk = pairs / sms / (ms * 1e-3) / (clk * 1e3);
  printf("%-22s %.3f ms  pairs/clk/SM %.2f  (elements/clk/SM %.2f)\n", name, ms, per_clk, 2 * per_clk);
  cudaFree(out);
}

int main() {
  run<0>("ex2 x2", 4);
  run<1>("cvt.rn.bf16x2 (F2FP)", 4);
  run<2>("2 ex2 + F2FP", 4);
  run<3>("prmt", 4);
  run<4>("2 ex2 + 2 iadd + prmt", 4);
  return 0;
}
