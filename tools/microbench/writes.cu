// How long do a few CTAs take to write a few KB each to global memory?
// (the small path's K1 operand-row copy-out).  Prints per-config median
// in-kernel time (globaltimer, first lane start -> last lane done) and the
// event-timed kernel duration.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void wr(double* out, int per_warp, unsigned long long* t, int mode) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  double* o = out + (size_t)warp * per_warp;
  if (mode == 0) {
    for (int i = lane; i < per_warp; i += 32) o[i] = (double)i;
  } else if (mode == 1) {
    for (int i = lane; i < per_warp; i += 32) __stcs(o + i, (double)i);
  } else {
    for (int i = 2 * lane; i < per_warp; i += 64) reinterpret_cast<double2*>(o + i)[0] = make_double2(i, i);
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (lane == 0) { t[2 * warp] = t0; t[2 * warp + 1] = t1; }
}

int main() {
  double* out; unsigned long long* t;
  cudaMalloc(&out, 256 << 20); cudaMalloc(&t, 1 << 20);
  double* big; cudaMalloc(&big, 512 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode)
    for (int ctas : {8, 32, 128})
      for (int threads : {32, 128}) {
        const int per_warp = 768 * 2 * 128 / threads / (ctas / 8);   // same total bytes: 8 x 128 lanes x 2 x 768 doubles / 32
        std::vector<float> ev;
        std::vector<double> span;
        for (int rep = 0; rep < 20; ++rep) {
          cudaMemsetAsync(big, rep, 512 << 20);     // evict L2
          cudaEventRecord(a);
          wr<<<ctas, threads>>>(out, per_warp, t, mode);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b); ev.push_back(ms * 1e3f);
          const int nw = ctas * threads / 32;
          std::vector<unsigned long long> h(2 * nw);
          cudaMemcpy(h.data(), t, h.size() * 8, cudaMemcpyDeviceToHost);
          unsigned long long lo = ~0ull, hi = 0;
          for (int w = 0; w < nw; ++w) { lo = std::min(lo, h[2 * w]); hi = std::max(hi, h[2 * w + 1]); }
          span.push_back((double)(hi - lo));
        }
        std::sort(ev.begin(), ev.end()); std::sort(span.begin(), span.end());
        printf("mode %d ctas %3d threads %3d per_warp %6d doubles: kernel %.2f us, in-kernel span %.0f ns\n",
               mode, ctas, threads, per_warp, ev[ev.size() / 2], span[span.size() / 2]);
      }
  return 0;
}
