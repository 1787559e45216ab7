// Microbenchmark: the GEMM epilogue's store pattern (8 warps, each 2 chunks of
// 32 rows x 32 fp32 columns transposed through smem, row-contiguous STG).
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda.h>
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void __launch_bounds__(320, 1) k_epi(float* c, long ldc, int M, int n, unsigned long long* tt, int variant, const __grid_constant__ CUtensorMap tmC) {
  extern __shared__ float dyn[];
  __shared__ float st_all[8][32 * 33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 2) return;
  float* st = st_all[warp - 2];
  const int quarter = warp & 3, half = (warp - 2) >> 2;
  const int m0 = (blockIdx.x % 2) * 128, n0 = (blockIdx.x / 2) * 128;
  const int row0 = m0 + quarter * 32;
  unsigned long long t0 = gt();
  for (int cch = 0; cch < 2; ++cch) {
    float v[32];
    for (int j = 0; j < 32; ++j) v[j] = lane * 0.5f + j + cch;
    const int nb = n0 + (half * 2 + cch) * 32;
#pragma unroll
    for (int j = 0; j < 32; ++j) st[lane * 33 + j] = v[j];
    __syncwarp();
    const int col = nb + lane;
    if (variant == 0) {
      for (int r = 0; r < 32; ++r) {
        const int row = row0 + r;
        if (row >= M) break;
        if (col < n) c[(long)row * ldc + col] = st[r * 33 + lane];
      }
    } else if (variant == 3) {
      // float4 per lane: 4 rows x 128 B per warp instruction
      const int rr = lane >> 3, cq = (lane & 7) * 4;
#pragma unroll
      for (int r = 0; r < 32; r += 4) {
        const int row = row0 + r + rr;
        if (row < M) {
          const float* q = st + (r + rr) * 33 + cq;
          *reinterpret_cast<float4*>(c + (long)row * ldc + nb + cq) = make_float4(q[0], q[1], q[2], q[3]);
        }
      }
    } else if (variant == 4) {
      // 2D TMA store of the 32x32 box from row-major smem
      float* sr = st_all[warp - 2];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        reinterpret_cast<float4*>(sr + lane * 32)[(j + lane) & 7] =
            make_float4(v[4*((j + lane) & 7)], v[4*((j + lane) & 7)+1], v[4*((j + lane) & 7)+2], v[4*((j + lane) & 7)+3]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(sr);
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                     :: "l"(&tmC), "r"(nb), "r"(row0), "r"(sa) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncwarp();
    } else if (variant == 2) {
      // row-major staging + one 128-byte bulk copy (TMA engine) per row
      float* sr = st_all[warp - 2];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        reinterpret_cast<float4*>(sr + lane * 32)[(j + lane) & 7] =
            make_float4(v[4*((j + lane) & 7)], v[4*((j + lane) & 7)+1], v[4*((j + lane) & 7)+2], v[4*((j + lane) & 7)+3]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      const int row = row0 + lane;
      if (row < M) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(sr + lane * 32);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;"
                     :: "l"(c + (long)row * ldc + nb), "r"(sa) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    } else {
      // lane = row: direct 32 consecutive floats per row (no transpose)
      const int row = row0 + lane;
      if (row < M) {
        float4* p = reinterpret_cast<float4*>(c + (long)row * ldc + nb);
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = make_float4(v[4*j], v[4*j+1], v[4*j+2], v[4*j+3]);
      }
    }
    __syncwarp();
  }
  unsigned long long t1 = gt();
  if (lane == 0 && blockIdx.x == 0) { tt[warp * 2] = t0; tt[warp * 2 + 1] = t1; }
}
int main() {
  const int M = 160, N = 4800;
  float* c; cudaMalloc(&c, (size_t)256 * N * 4);
  unsigned long long* tt; cudaMallocManaged(&tt, 64 * 8);
  const int smem = 193 * 1024;
  cudaFuncSetAttribute(k_epi, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  CUtensorMap tmC;
  {
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)N * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tmC, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, c, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("map rc %d\n", (int)r);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int grid : {1, 76}) for (int variant = 0; variant < 5; ++variant) {
    printf("grid %d ", grid);
    for (int i = 0; i < 3; ++i) k_epi<<<grid, 320, smem>>>(c, N, M, N, tt, variant, tmC);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) k_epi<<<grid, 320, smem>>>(c, N, M, N, tt, variant, tmC);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("variant %d: %.2f us/launch; CTA0 warp spans (us):", variant, ms * 1000 / 20);
    for (int w = 2; w < 10; ++w) printf(" %.2f", (tt[2 * w + 1] - tt[2 * w]) / 1000.0);
    printf("\n");
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
