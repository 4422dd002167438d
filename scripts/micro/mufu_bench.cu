// Micro-benchmark: MUFU ex2 throughput per SM for f32, f16x2 and bf16x2
// (decides whether packed exp can relieve the softmax's MUFU bound).
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_f32(float* out, float seed) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + i) * 1e-9f - 1.0f;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_f16x2(float* out, float seed) {
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    __half2 h = __floats2half2_rn(seed * threadIdx.x * 1e-9f - 1.0f, -0.5f);
    x[i] = *reinterpret_cast<uint32_t*>(&h) + i;
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[i]));
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= x[i];
  if (s == 12345u) out[0] = (float)s;
}

__global__ void k_bf16x2(float* out, float seed) {
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(seed * threadIdx.x * 1e-9f - 1.0f, -0.5f);
    x[i] = *reinterpret_cast<uint32_t*>(&h) + i;
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x[i]));
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= x[i];
  if (s == 12345u) out[0] = (float)s;
}

template <typename F>
void run(const char* name, F kern, int elems_per_op) {
  float* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  dim3 grid(sms * 4), block(256);
  kern<<<grid, block>>>(out, 1.0f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<grid, block>>>(out, 1.0f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double ops = (double)grid.x * block.x * kIters * 8;
  double per_sm_per_s = ops / sms / (ms * 1e-3);
  printf("%-8s %.3f ms  %.2f warp-instr... lane-ops/clk/SM (at max clock %d MHz): %.2f, elems/clk/SM %.2f\n", name, ms,
         0.0, clk / 1000, per_sm_per_s / (clk * 1e3), per_sm_per_s * elems_per_op / (clk * 1e3));
  cudaFree(out);
}

int main() {
  run("f32", k_f32, 1);
  run("f16x2", k_f16x2, 2);
  run("bf16x2", k_bf16x2, 2);
  return 0;
}
