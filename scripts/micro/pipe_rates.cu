// Microbenchmark: per-SM throughput of MUFU.RCP, FFMA (3-reg), FFMA2 on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float rcpa(float x) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__global__ void k_rcp(float* out, int iters) {
  float a[8];
  for (int j = 0; j < 8; ++j) a[j] = 1.0f + threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = rcpa(a[j] + 1.0f);
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void k_ffma(float* out, int iters, float b, float c) {
  float a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b, a[(j + 1) & 7]);
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, int iters, float b, float c) {
  unsigned long long a[8], bb;
  asm("mov.b64 %0, {%1,%2};" : "=l"(bb) : "f"(b), "f"(c));
  for (int j = 0; j < 8; ++j) { float x = threadIdx.x * 1e-3f + j; asm("mov.b64 %0, {%1,%1};" : "=l"(a[j]) : "f"(x)); }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(a[j]) : "l"(a[j]), "l"(bb), "l"(a[(j + 1) & 7]));
  }
  float s = 0, x, y; for (int j = 0; j < 8; ++j) { asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[j])); s += x + y; }
  if (s == 12345.f) out[threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  for (int w = 0; w < 3; ++w) {
    for (int kind = 0; kind < 3; ++kind) {
      cudaEventRecord(e0);
      if (kind == 0) k_rcp<<<blocks, threads>>>(out, iters);
      if (kind == 1) k_ffma<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
      if (kind == 2) k_ffma2<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 8 * (kind == 2 ? 2 : 1);
      double per_clk_sm = ops / (ms * 1e-3) / sms / (clk * 1e3);
      if (w == 2) printf("%s: %.1f ops/clk/SM (at nominal %d MHz), %.3f ms\n",
                         kind == 0 ? "MUFU.RCP" : kind == 1 ? "FFMA" : "FFMA2 (x2 lanes)", per_clk_sm, clk / 1000, ms);
    }
  }
  return 0;
}
