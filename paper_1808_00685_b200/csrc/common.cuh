// Shared helpers for libcorr2d: error plumbing for the C ABI and small
// device utilities.  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <stdint.h>
#include <string>

#include "../../include/corr2d.h"

namespace corr2d {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

// Sign flip and |x| bit pattern on the INTEGER pipe.  Written as inline PTX:
// plain C++ bit tricks (xor / and on __double_as_longlong) are turned back into
// DADD -x / DADD |x| by the compiler, which queue on the FP64 pipe behind the
// DMMAs of co-resident CTAs (ncu: ~10 % of contract_f64's samples were
// "math pipe throttle" stalls on those DADDs).
// (ptxas also recognises a 64-bit xor / and of the sign bit as fneg / fabs, so
// the sign bit is flipped by a 32-bit add on the high word.)
__device__ __forceinline__ double neg_bits(double x) {
  int hi = __double2hiint(x), lo = __double2loint(x);
  asm volatile("add.s32 %0, %0, 0x80000000;" : "+r"(hi));
  return __hiloint2double(hi, lo);
}
__device__ __forceinline__ unsigned long long abs_bits(double x) {
  unsigned hi = (unsigned)__double2hiint(x), lo = (unsigned)__double2loint(x);
  asm volatile("shl.b32 %0, %0, 1;" : "+r"(hi));   // drop the sign bit ...
  asm volatile("shr.b32 %0, %0, 1;" : "+r"(hi));   // ... without an and-mask ptxas could fold
  return ((unsigned long long)hi << 32) | lo;
}

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

// ---- CORR2D_PACK_F16F8 (see corr2d.h): per-channel power-of-two scale sc with
// max|x| * sc in [2^7, 2^8); each scaled slot x is stored as fp16(x) * 2^5, the
// e4m3 copy of x and e4m3((x - fp16(x)) * 2^10), so every tensor-core product
// (fp16 hi.hi and the two e4m3 cross terms) lands at scale 2^10 sc_i sc_j.
// Shift s of sc = 2^s from the bit pattern of max|x|; 0 for an all-zero or
// non-finite channel.
__device__ __forceinline__ int f16f8_shift(uint32_t maxbits) {
  if (maxbits == 0u || maxbits >= 0x7f800000u) return 0;
  const int s = 7 - ((int)(maxbits >> 23) - 127);
  return s < -120 ? -120 : (s > 120 ? 120 : s);
}
__device__ __forceinline__ float pow2f(int s) { return __uint_as_float((uint32_t)(127 + s) << 23); }

// Two adjacent scaled slots -> fp16 hi x 2^5 (2 halves), e4m3 hi, e4m3 residual x 2^10.
__device__ __forceinline__ void f16f8_split2(float x0, float x1, uint32_t& h16, uint16_t& h8, uint16_t& l8) {
  const __half2 h = __floats2half2_rn(x0 * 32.f, x1 * 32.f);
  const float2 hf = __half22float2(h);
  const float r0 = x0 - hf.x * 0.03125f, r1 = x1 - hf.y * 0.03125f;
  h16 = *reinterpret_cast<const uint32_t*>(&h);
  h8 = (uint16_t)__nv_cvt_float2_to_fp8x2(make_float2(x0, x1), __NV_SATFINITE, __NV_E4M3);
  l8 = (uint16_t)__nv_cvt_float2_to_fp8x2(make_float2(r0 * 1024.f, r1 * 1024.f), __NV_SATFINITE, __NV_E4M3);
}

}  // namespace corr2d
