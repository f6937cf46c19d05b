// Launch and store floors for the small-map steps (cfg1 / cfg2), in the same
// shape bench.py times them: a CUDA graph of K back-to-back launches rotating
// over R independent output buffers whose total exceeds the 126 MB L2.
//   empty      : an empty kernel (the launch floor of one graph node)
//   empty2_pdl : two empty kernels chained by programmatic dependent launch
//                (the small path's two-kernel shape)
//   store16    : a grid-stride kernel writing 16 MB (cfg1's two fp64 planes)
//   store48    : 48 MB (cfg2's planes)
// Prints one JSON object (microseconds per step).
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void empty_kernel(int* p) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (p && threadIdx.x == 1234567) p[0] = 1;
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

__global__ void store_kernel(double2* __restrict__ d, size_t n) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  const double2 v = make_double2(1.0, 2.0);
  for (; i < n; i += s) __stcs(d + i, v);
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

static cudaError_t launch(void (*k)(int*), int grid, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, (int*)nullptr);
}

static cudaError_t launch_store(double2* d, size_t n, int grid, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, store_kernel, d, n);
}

template <class F>
static float time_graph(cudaStream_t st, int K, F body) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int k = 0; k < K; ++k) body(k);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return 1e3f * ms / K;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const int K = 200;
  const float empty = time_graph(st, K, [&](int) { launch(empty_kernel, sms, st, true); });
  const float empty2 = time_graph(st, K, [&](int) {
    launch(empty_kernel, 8, st, true);
    launch(empty_kernel, 136, st, true);
  });
  float store[2];
  const size_t bytes[2] = {16000000, 48000000};
  for (int v = 0; v < 2; ++v) {
    const int R = (int)((4 * 126e6) / bytes[v]) + 1;
    std::vector<double2*> bufs(R);
    for (auto& b : bufs) CK(cudaMalloc(&b, bytes[v]));
    const size_t n = bytes[v] / 16;
    store[v] = time_graph(st, K, [&](int k) { launch_store(bufs[k % R], n, 4 * sms, st); });
    for (auto& b : bufs) cudaFree(b);
  }
  CK(cudaGetLastError());
  printf("{\"sms\": %d, \"graph_steps\": %d, \"empty_kernel_us\": %.3f, \"two_empty_kernels_pdl_us\": %.3f, "
         "\"store_16MB_us\": %.3f, \"store_48MB_us\": %.3f, \"store_16MB_GBs\": %.1f, \"store_48MB_GBs\": %.1f}\n",
         sms, K, empty, empty2, store[0], store[1], 16000000 / (store[0] * 1e3), 48000000 / (store[1] * 1e3));
  return 0;
}
