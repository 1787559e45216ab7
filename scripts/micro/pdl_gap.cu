// Microbenchmark: per-kernel cost of a chain of dependent small kernels inside
// a CUDA graph, plain stream order vs programmatic dependent launch (PDL).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_small(float* x, int n, int pdl) {
  if (pdl) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 1.0001f + 1.0f;
}
int main() {
  const int n = 148 * 256;
  float* x; cudaMalloc(&x, n * 4);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < 40; ++k) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148); cfg.blockDim = dim3(256); cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, k_small, x, n, pdl);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int w = 0; w < 20; ++w) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaStreamSynchronize(s);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl %d: %.2f us per kernel\n", pdl, ms * 1000 / (20 * 40));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
