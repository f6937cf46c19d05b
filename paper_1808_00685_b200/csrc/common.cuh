// Shared helpers for libcorr2d: error plumbing for the C ABI and small
// device utilities.  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

#include "../../include/corr2d.h"

namespace corr2d {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

// Positive doubles order like their bit patterns: atomicMax on uint64 bits.
__device__ __forceinline__ void atomic_max_abs(unsigned long long* dst, double v) {
  unsigned long long bits = __double_as_longlong(fabs(v));
  atomicMax(dst, bits);
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace corr2d
