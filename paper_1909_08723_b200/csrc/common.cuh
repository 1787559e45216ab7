// Shared helpers for the fusedbeam_b200 kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cmath>
#include <cstdlib>
#include <string>
#include <utility>

#include "fusedbeam_b200.h"

namespace fb {

// thread-local last-error message (fb_last_error)
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
void count_launch(unsigned n = 1);

// Check the last launch; map to FB_ERR_CUDA with a message.
int check_launch(const char* what);

constexpr int kNumSMs = 148;

// ---- tensor-core operand format (compile time; fb_operand_format reports it) --
// FB_OPERAND_FP16X2 = 1 (default): an fp32 activation x is scaled by 2^8 and
// split into two fp16 planes, hi = fp16(x 2^8), lo = fp16(x 2^8 - hi): 22
// significant bits, and absolute error <= 2^-32 below the fp16 normal range;
// weights are fp16, scaled per matrix by a power of two (bf16-exact values are
// exact in fp16 there).  Products are exact in fp32; the epilogue undoes both
// scales with one exact multiply (fb_gemm_t.acc_scale).  Two MMAs per K step
// and 4 B per A element.  Operand range: |x| < 255.
// FB_OPERAND_FP16X2 = 0: three bf16 planes hi/mid/lo (24 bits), bf16 weights.
#ifndef FB_OPERAND_FP16X2
#define FB_OPERAND_FP16X2 1
#endif
constexpr int kPlanes = FB_OPERAND_FP16X2 ? 2 : 3;
constexpr float kActScale = FB_OPERAND_FP16X2 ? 256.0f : 1.0f;

// x -> operand planes (raw 16-bit patterns; p[2] unused with 2 planes)
__device__ __forceinline__ void split_operand(float x, uint16_t* p) {
#if FB_OPERAND_FP16X2
  const float y = x * kActScale;
  const __half hi = __float2half_rn(y);
  p[0] = __half_as_ushort(hi);
  p[1] = __half_as_ushort(__float2half_rn(y - __half2float(hi)));
#else
  const __nv_bfloat16 hi = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(hi);
  const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
  p[0] = __bfloat16_as_ushort(hi);
  p[1] = __bfloat16_as_ushort(mid);
  p[2] = __bfloat16_as_ushort(__float2bfloat16_rn(r1 - __bfloat162float(mid)));
#endif
}
constexpr int kWarp = 32;

__device__ __forceinline__ int row_count(int n_max, const int32_t* n_dev) {
  return n_dev ? min(n_max, *n_dev) : n_max;
}

__device__ __forceinline__ int row_at(const int32_t* rows, int i) {
  return rows ? rows[i] : i;
}

// Exact IEEE double ops with no FMA contraction (the reference is numpy).
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }


// ---- programmatic dependent launch (decode-step chain) ---------------------
// Kernels on the per-step chain begin with pdl_entry(): wait until the grid
// before them in the stream has completed and its memory is visible.
// Launched through launch_pdl() (attribute programmaticStreamSerialization),
// each launch is processed while its predecessor still runs and its CTAs
// start as soon as the predecessor's last CTA exits; a kernel launched without
// the attribute (or whose predecessor is not a kernel) runs as before.  No
// kernel triggers its dependents early (griddepcontrol.launch_dependents at
// kernel start was measured slower: early-resident CTAs crowd the overlapped
// streams, 146.3 -> 148.9-150.4 ms), so the wait only hides launch latency.
__device__ __forceinline__ void pdl_entry() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("FB_PDL");
    return e ? atoi(e) != 0 : true;
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

}  // namespace fb

#define FB_CHECK_ARG(cond, msg)                        \
  do {                                                  \
    if (!(cond)) return ::fb::fail(FB_ERR_VALUE, msg); \
  } while (0)
