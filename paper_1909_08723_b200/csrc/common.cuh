// Shared helpers for the fusedbeam_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cmath>
#include <string>

#include "fusedbeam_b200.h"

namespace fb {

// thread-local last-error message (fb_last_error)
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
void count_launch(unsigned n = 1);

// Check the last launch; map to FB_ERR_CUDA with a message.
int check_launch(const char* what);

constexpr int kNumSMs = 148;
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

}  // namespace fb

#define FB_CHECK_ARG(cond, msg)                        \
  do {                                                  \
    if (!(cond)) return ::fb::fail(FB_ERR_VALUE, msg); \
  } while (0)
