// Dependent-chain latency of fp64 DADD / DFMA / DMUL and fp32 FFMA on this GPU
// (clock64 around 1024-deep chains, one warp).  nvcc -arch=sm_100a -o fp64lat fp64lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chains(double x, float xf, long long* out, double* sink) {
  double a = x, b = x * 0.5, c = x * 0.25;
  float f = xf;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) a = fma(a, b, c);
  long long t2 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) a = __dmul_rn(a, b);
  long long t3 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) f = fmaf(f, xf, 1.0f);
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3;
  }
  sink[threadIdx.x] = a + f;
}

int main() {
  long long* d; double* s;
  cudaMalloc(&d, 64); cudaMalloc(&s, 1024 * 8);
  for (int k = 0; k < 3; ++k) chains<<<1, 32>>>(1.0000001, 0.999f, d, s);
  long long h[4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cycles per dependent op: DADD %.1f DFMA %.1f DMUL %.1f FFMA %.1f\n", h[0] / 1024.0, h[1] / 1024.0,
         h[2] / 1024.0, h[3] / 1024.0);
  return 0;
}
