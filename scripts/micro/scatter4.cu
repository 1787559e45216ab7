// Probe: TMA tile::scatter4 store semantics (tensor-map box and smem layout).
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
__global__ void k(const __grid_constant__ CUtensorMap tm, int r0, int r1, int r2, int r3) {
  __shared__ __align__(128) float s[4 * 32];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) s[i] = 1000.f * (i / 32) + (i % 32);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
      :: "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"((unsigned)__cvta_generic_to_shared(s)) : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  float* d; cudaMalloc(&d, 64 * 64 * 4);
  float h[64 * 64];
  for (int boxr : {1, 4}) {
    cudaMemset(d, 0, 64 * 64 * 4);
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, 64}; cuuint64_t str[1] = {64 * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)boxr}; cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 128>>>(tm, 5, 17, 3, 40);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("box rows %d: encode %d, err %s\n", boxr, (int)r, cudaGetErrorString(e));
    for (int row : {3, 5, 17, 40, 0, 6}) printf("  row %2d: %g %g ... %g | col32 %g\n", row, h[row * 64], h[row * 64 + 1], h[row * 64 + 31], h[row * 64 + 32]);
    if (e != cudaSuccess) break;
  }
}
