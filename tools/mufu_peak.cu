// Measured MUFU (SFU) throughput of this GPU: independent ex2.approx chains
// in every thread of a full grid; the blend roofline's peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_peak tools/mufu_peak.cu && ./mufu_peak
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr int kChains = 8, kIters = 4096;

__global__ void __launch_bounds__(256) mufu_kernel(float *out, float seed) {
  float v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; c++) v[c] = seed * (threadIdx.x + c) * 1e-9f - 0.5f;
  for (int i = 0; i < kIters; i++) {
#pragma unroll
    for (int c = 0; c < kChains; c++) v[c] = ex2(v[c]) - 1.0f;   // stays in (-0.5, 0]
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; c++) s += v[c];
  if (s == 12345.f) out[threadIdx.x] = s;   // keep the work alive
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out;
  cudaMalloc(&out, 1024 * sizeof(float));
  const int blocks = sms * 8;
  mufu_kernel<<<blocks, 256>>>(out, 1.f);   // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; r++) mufu_kernel<<<blocks, 256>>>(out, 1.f + r);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = (double)reps * blocks * 256 * kChains * kIters;
  const double gops = ops / (ms * 1e-3) / 1e9;
  printf("{\"mufu_ex2_gops\": %.1f, \"sms\": %d, \"clock_khz_attr\": %d, \"per_sm_per_clk_at_attr_clock\": %.2f}\n",
         gops, sms, clk, gops * 1e9 / sms / (clk * 1e3));
  return 0;
}
