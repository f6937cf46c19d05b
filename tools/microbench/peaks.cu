// Peak microbenchmarks for the roofline denominators MEASURED_PEAKS.json lacks:
// FP64 DFMA, FP64 DMMA (mma.sync f64 -> DMMA.8x8x4), HBM store-only, HBM copy,
// pinned PCIe H2D/D2H.  Prints one JSON object.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
          "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
            "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += acc[i][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma884_kernel(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = 1e-3 * threadIdx.x, b = 2e-3 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void store_kernel(double4* __restrict__ dst, size_t n4) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  double4 v = make_double4(1.0, 2.0, 3.0, 4.0);
  for (; i < n4; i += stride) dst[i] = v;
}

__global__ void copy_kernel(const double4* __restrict__ src, double4* __restrict__ dst, size_t n4) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n4; i += stride) dst[i] = src[i];
}

template <class F>
float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  std::vector<float> ts;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[0];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  // DFMA
  int iters = 20000;
  int blocks = sms * 8, threads = 256;
  float ms = time_it([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-7); }, 5);
  double dfma_tf = 2.0 * 16 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
  // DMMA m16n8k16
  int iters2 = 2000;
  float ms2 = time_it([&] { dmma_kernel<<<sms * 4, 256>>>(out, iters2); }, 5);
  double dmma_tf = 2.0 * 16 * 8 * 16 * 8.0 * iters2 * (sms * 4 * 256 / 32) / (ms2 * 1e-3) / 1e12;
  float ms3 = time_it([&] { dmma884_kernel<<<sms * 4, 256>>>(out, iters2 * 4); }, 5);
  double dmma884_tf = 2.0 * 8 * 8 * 4 * 8.0 * iters2 * 4 * (sms * 4 * 256 / 32) / (ms3 * 1e-3) / 1e12;
  CK(cudaGetLastError());
  // HBM
  size_t bytes = (size_t)4 << 30;
  double4 *s, *d;
  CK(cudaMalloc(&s, bytes)); CK(cudaMalloc(&d, bytes));
  size_t n4 = bytes / sizeof(double4);
  float mss = time_it([&] { store_kernel<<<sms * 8, 512>>>(d, n4); }, 10);
  float msc = time_it([&] { copy_kernel<<<sms * 8, 512>>>(s, d, n4); }, 10);
  // PCIe
  size_t pb = (size_t)1 << 30;
  void* h; CK(cudaMallocHost(&h, pb));
  float msh2d = time_it([&] { cudaMemcpyAsync(d, h, pb, cudaMemcpyHostToDevice); }, 5);
  float msd2h = time_it([&] { cudaMemcpyAsync(h, d, pb, cudaMemcpyDeviceToHost); }, 5);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"dfma_tflops\": %.2f, \"dmma_m16n8k16_tflops\": %.2f, \"dmma_m8n8k4_tflops\": %.2f, "
         "\"hbm_store_gbs\": %.1f, \"hbm_copy_gbs\": %.1f, \"h2d_pinned_gbs\": %.1f, \"d2h_pinned_gbs\": %.1f, \"clock_khz\": %d}\n",
         sms, dfma_tf, dmma_tf, dmma884_tf, bytes / (mss * 1e-3) / 1e9, 2.0 * bytes / (msc * 1e-3) / 1e9,
         pb / (msh2d * 1e-3) / 1e9, pb / (msd2h * 1e-3) / 1e9, clk);
  return 0;
}
