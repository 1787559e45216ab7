// Microbenchmark: per-SM global store / load bandwidth (1 CTA and 148 CTAs).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void k_store(float4* out, int per_cta_f4, int reps, unsigned long long* tt) {
  float4* o = out + (size_t)blockIdx.x * per_cta_f4;
  unsigned long long t0 = gt();
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < per_cta_f4; i += blockDim.x)
      o[i] = make_float4(r, i, 0, 1);
  __syncthreads();
  unsigned long long t1 = gt();
  if (threadIdx.x == 0) tt[blockIdx.x] = t1 - t0;
}
__global__ void k_load(const float4* in, int per_cta_f4, int reps, unsigned long long* tt, float* sink) {
  const float4* p = in + (size_t)blockIdx.x * per_cta_f4;
  unsigned long long t0 = gt();
  float s = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < per_cta_f4; i += blockDim.x) { float4 v = __ldcg(p + i); s += v.x + v.w; }
  __syncthreads();
  unsigned long long t1 = gt();
  if (threadIdx.x == 0) tt[blockIdx.x] = t1 - t0;
  if (s == 1234.5f) sink[0] = s;
}
int main() {
  const int per = 64 * 1024 / 16;       // 64 KB per CTA per rep
  float4* buf; cudaMalloc(&buf, (size_t)148 * per * 16);
  unsigned long long* tt; cudaMallocManaged(&tt, 148 * 8);
  float* sink; cudaMalloc(&sink, 4);
  for (int threads : {256, 1024}) for (int grid : {1, 148}) {
    for (int w = 0; w < 3; ++w) k_store<<<grid, threads>>>(buf, per, 16, tt);
    cudaDeviceSynchronize();
    double mx = 0; for (int b = 0; b < grid; ++b) mx = tt[b] > mx ? tt[b] : mx;
    printf("store threads %d grid %d: 1 MB per CTA in %.2f us -> %.1f GB/s per SM\n", threads, grid, mx / 1e3, 16.0 * 65536 / mx);
    for (int w = 0; w < 3; ++w) k_load<<<grid, threads>>>(buf, per, 16, tt, sink);
    cudaDeviceSynchronize();
    mx = 0; for (int b = 0; b < grid; ++b) mx = tt[b] > mx ? tt[b] : mx;
    printf("load  threads %d grid %d: 1 MB per CTA in %.2f us -> %.1f GB/s per SM\n", threads, grid, mx / 1e3, 16.0 * 65536 / mx);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
