// HBM write-bandwidth variants: the small-K contraction is store-bound, so the
// achievable write-only rate (not the copy rate) is its real ceiling.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__global__ void st_v4(float4* __restrict__ d, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  float4 v = make_float4(1, 2, 3, 4);
  for (; i < n; i += s) d[i] = v;
}
__global__ void st_v4_cs(float4* __restrict__ d, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  float4 v = make_float4(1, 2, 3, 4);
  for (; i < n; i += s) __stcs(d + i, v);
}
// each block writes a contiguous chunk, unrolled x4
__global__ void st_chunk(float4* __restrict__ d, size_t n, size_t per_block) {
  size_t base = blockIdx.x * per_block;
  float4 v = make_float4(1, 2, 3, 4);
  for (size_t i = base + threadIdx.x; i < base + per_block && i < n; i += 4 * blockDim.x) {
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * blockDim.x < n) d[i + u * blockDim.x] = v;
  }
}
// TMA bulk store: smem -> global via cp.async.bulk
__global__ void st_bulk(char* __restrict__ d, size_t bytes, int chunk) {
  extern __shared__ __align__(128) char sm[];
  for (int i = threadIdx.x; i < chunk / 4; i += blockDim.x) ((float*)sm)[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    size_t nchunks = bytes / chunk;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                   :: "l"(d + c * chunk), "r"((unsigned)__cvta_generic_to_shared(sm)), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;\n" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}
__global__ void rd(const float4* __restrict__ s, size_t n, float* out) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  float a = 0;
  for (; i < n; i += st) { float4 v = s[i]; a += v.x + v.y + v.z + v.w; }
  if (a == 1.2345f) out[0] = a;
}

template <class F> float best(F f, int reps = 10) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float m = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b); m = std::min(m, t);
  }
  return m;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t bytes = (size_t)4 << 30;
  char* d; cudaMalloc(&d, bytes);
  float* o; cudaMalloc(&o, 64);
  size_t n4 = bytes / 16;
  auto gbs = [&](float ms) { return bytes / (ms * 1e-3) / 1e9; };
  printf("{");
  for (int bpsm : {2, 4, 8, 16}) for (int thr : {256, 512, 1024}) {
    if (bpsm * thr > 2048) continue;
    float ms = best([&] { st_v4<<<sms * bpsm, thr>>>((float4*)d, n4); });
    printf("\"st_v4_%dx%d\": %.0f, ", bpsm, thr, gbs(ms));
  }
  printf("\"st_v4_cs\": %.0f, ", gbs(best([&] { st_v4_cs<<<sms * 4, 512>>>((float4*)d, n4); })));
  for (int nb : {sms, sms * 4, sms * 16}) {
    size_t per = (n4 + nb - 1) / nb;
    printf("\"st_chunk_%d\": %.0f, ", nb, gbs(best([&] { st_chunk<<<nb, 512>>>((float4*)d, n4, per); })));
  }
  printf("\"memset\": %.0f, ", gbs(best([&] { cudaMemsetAsync(d, 0, bytes); })));
  for (int chunk : {16384, 65536}) {
    cudaFuncSetAttribute(st_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, chunk);
    for (int bpsm : {1, 2}) {
      if (chunk * bpsm > 200000) continue;
      printf("\"st_bulk_%d_%d\": %.0f, ", chunk, bpsm, gbs(best([&] { st_bulk<<<sms * bpsm, 32, chunk>>>(d, bytes, chunk); })));
    }
  }
  printf("\"read\": %.0f", gbs(best([&] { rd<<<sms * 4, 512>>>((const float4*)d, n4, o); })));
  cudaError_t e = cudaDeviceSynchronize();
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
