// fetch.cu -- device -> host transfer of a homo map that moves part of its
// lower triangle as the mirror image only: the host fills it.
//
// A homo map is symmetric / antisymmetric by construction (reference
// fourier.py:106-123: sync = Re(Y^H W Y), async = Im(...), so sync^T = sync and
// async^T = -async), and every homo contraction here writes its off-diagonal
// tiles' mirror as (sync^T, -async^T) exactly.  The planes are the end-to-end
// call's dominant cost (cfg5: 8.6 GB over a ~57 GB/s link against a 2.7 ms
// contraction), so the transfer sends, per row band [r0, r1), only columns
// [split, n), split = fill_pct % of r0, and host threads fill the band's
// columns [0, split) from rows above it (already landed) while later bands
// are in flight.  The diagonal blocks [r0, r1)^2 always travel whole, so
// whatever the kernels wrote inside a diagonal tile is kept bit for bit (band
// a multiple of every contraction's tile edge); the host result equals a
// full-plane copy bit for bit (tests/test_gpu_fetch.py).
//
// Measured (profiles/r2_fetch_probe.txt, r2_fetch_e2e_ab.txt): the host's
// transpose fill and the DMA share the host's memory bandwidth.  On the B200
// boxes' 16-thread hosts the upper-triangle-only transfer (100 %) loses 30 %
// (cfg5: 192 vs 150 ms); a 25-35 % host share is the best split (public-call
// e2e cfg5 154 -> 143-148 ms, cfg3 76.7 -> 75.0 ms), so the Python layer uses
// 30 % (engine.MIRROR_FILL_PCT; CORR2D_FETCH_FILL_PCT=0 = full copy).
#include <cuda_runtime.h>
#include <emmintrin.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <system_error>
#include <thread>
#include <vector>

#include "common.cuh"
#include "../../include/corr2d.h"

using corr2d::fail;

namespace {

constexpr int kCopyStreams = 4;   // one stream ~51 GB/s D2H, four ~56 GB/s (tools/d2h_probe.py)
constexpr int kTileEdge = 256;    // largest contraction tile edge (tcgen05 2-SM pair)
constexpr int kFillCols = 256;    // columns per host fill task
constexpr int kBlk = 32;          // host transpose block

// per-device copy streams, created on first use (a fixed table: pointers handed
// out stay valid while other devices add theirs)
constexpr int kMaxDevices = 64;
std::mutex g_mu;
cudaStream_t g_streams[kMaxDevices][kCopyStreams] = {};

int copy_streams(cudaStream_t** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(CORR2D_ERR_CUDA, "corr2d_fetch_mirrored: no device");
  if (dev < 0 || dev >= kMaxDevices) return fail(CORR2D_ERR_UNSUPPORTED, "corr2d_fetch_mirrored: device index");
  std::lock_guard<std::mutex> lk(g_mu);
  cudaStream_t* s = g_streams[dev];
  if (!s[kCopyStreams - 1])
    for (int k = 0; k < kCopyStreams; ++k)
      if (!s[k] && cudaStreamCreateWithFlags(&s[k], cudaStreamNonBlocking) != cudaSuccess)
        return fail(CORR2D_ERR_CUDA, "corr2d_fetch_mirrored: stream creation failed");
  *out = s;
  return CORR2D_OK;
}

// x[i][j] = sign * x[j][i] for i in [r0, r1), j in [c0, c1)  (all j < r0 <= i),
// in kBlk x kBlk tiles: the source rows are read contiguously into a
// transposed L1 tile, whose rows leave with streaming (non-temporal) 16-byte
// stores when the destination is aligned -- no read-for-ownership of the
// destination lines, which the concurrent PCIe transfer needs the host memory
// bandwidth for.
template <typename T, bool NEG>
void fill_block(T* x, int64_t ld, int r0, int r1, int c0, int c1) {
  alignas(64) T tmp[kBlk][kBlk];
  constexpr int kVec = 16 / sizeof(T);
  const bool aligned = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && (ld % kVec == 0);
  for (int ib = r0; ib < r1; ib += kBlk) {
    const int ie = std::min(ib + kBlk, r1);
    for (int jb = c0; jb < c1; jb += kBlk) {
      const int je = std::min(jb + kBlk, c1);
      for (int j = jb; j < je; ++j) {
        const T* src = x + (int64_t)j * ld + ib;
        for (int i = 0; i < ie - ib; ++i) tmp[i][j - jb] = NEG ? -src[i] : src[i];
      }
      const bool nt = aligned && (jb % kVec == 0) && (je - jb) % kVec == 0;
      for (int i = ib; i < ie; ++i) {
        T* dst = x + (int64_t)i * ld + jb;
        if (nt) {
          for (int j = 0; j < je - jb; j += kVec)
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + j),
                             _mm_load_si128(reinterpret_cast<const __m128i*>(&tmp[i - ib][j])));
        } else {
          for (int j = 0; j < je - jb; ++j) dst[j] = tmp[i - ib][j];
        }
      }
    }
  }
}

template <typename T>
int fetch_impl(const T* ds, const T* da, int64_t ld_dev, int n, T* hs, T* ha, int64_t ld_host, int band,
               int fill_pct, int threads, int64_t* d2h_bytes, cudaStream_t stream) {
  cudaStream_t* cs = nullptr;
  if (int rc = copy_streams(&cs)) return rc;
  const int nb = (n + band - 1) / band;
  // band b sends columns [split(b), n); the host fills [0, split(b)) (64-column
  // multiples of fill_pct % of the band's lower part)
  auto split = [&](int b) { return (int)(((int64_t)b * band * fill_pct / 100) / 64 * 64); };
  std::vector<cudaEvent_t> ev(nb, nullptr);
  cudaEvent_t ready = nullptr;
  auto cleanup = [&] {
    for (auto e : ev) if (e) cudaEventDestroy(e);
    if (ready) cudaEventDestroy(ready);
  };
  if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess) {
    cleanup();
    return fail(CORR2D_ERR_CUDA, "corr2d_fetch_mirrored: event creation failed");
  }
  cudaEventRecord(ready, stream);
  for (int k = 0; k < kCopyStreams; ++k) cudaStreamWaitEvent(cs[k], ready, 0);
  int64_t bytes = 0;
  const size_t es = sizeof(T);
  for (int b = 0; b < nb; ++b) {
    const int r0 = b * band, r1 = std::min(n, r0 + band), c0 = split(b);
    cudaStream_t st = cs[b % kCopyStreams];
    const size_t w = (size_t)(n - c0) * es;
    cudaError_t e1 = cudaMemcpy2DAsync(hs + (int64_t)r0 * ld_host + c0, ld_host * es, ds + (int64_t)r0 * ld_dev + c0,
                                       ld_dev * es, w, r1 - r0, cudaMemcpyDeviceToHost, st);
    cudaError_t e2 = cudaMemcpy2DAsync(ha + (int64_t)r0 * ld_host + c0, ld_host * es, da + (int64_t)r0 * ld_dev + c0,
                                       ld_dev * es, w, r1 - r0, cudaMemcpyDeviceToHost, st);
    if (e1 != cudaSuccess || e2 != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming | cudaEventBlockingSync) != cudaSuccess ||
        cudaEventRecord(ev[b], st) != cudaSuccess) {
      // copies already queued on earlier bands finish on their own streams
      for (int k = 0; k < kCopyStreams; ++k) cudaStreamSynchronize(cs[k]);
      cleanup();
      return fail(CORR2D_ERR_CUDA, std::string("corr2d_fetch_mirrored: ") +
                                        cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    }
    bytes += 2 * (int64_t)w * (r1 - r0);
  }

  // fill tasks, band-major: (band b, columns [c, c + kFillCols) of [0, split(b))).
  // They read rows j < split(b) <= r0 at columns [r0, r1): sent by earlier bands
  // (band(j) < b, whose transfers cover columns >= split(band(j)) <= r0), and
  // write host columns no transfer touches -- so band b's fill waits for bands
  // [0, b) only and overlaps band b's own transfer.
  struct Task { int b, c0, c1; };
  std::vector<Task> tasks;
  for (int b = 1; b < nb; ++b)
    for (int c = 0; c < split(b); c += kFillCols) tasks.push_back({b, c, std::min(c + kFillCols, split(b))});
  std::atomic<size_t> next{0};
  std::atomic<int> err{0};
  // ready_upto: bands [0, ready_upto) have landed; one thread waits at a time
  std::mutex wait_mu;
  std::atomic<int> ready_upto{0};
  auto worker = [&] {
    for (;;) {
      const size_t t = next.fetch_add(1);
      if (t >= tasks.size() || err.load()) return;
      const Task& tk = tasks[t];
      if (ready_upto.load() < tk.b) {
        std::lock_guard<std::mutex> lk(wait_mu);
        while (ready_upto.load() < tk.b) {
          if (cudaEventSynchronize(ev[ready_upto.load()]) != cudaSuccess) { err = 1; return; }
          ready_upto.fetch_add(1);
        }
      }
      const int r0 = tk.b * band, r1 = std::min(n, r0 + band);
      fill_block<T, false>(hs, ld_host, r0, r1, tk.c0, tk.c1);
      fill_block<T, true>(ha, ld_host, r0, r1, tk.c0, tk.c1);
    }
  };
  auto worker_fenced = [&] {
    worker();
    _mm_sfence();   // streaming stores drained before the join publishes them
  };
  const int nt = std::max(1, std::min<int>(threads, (int)tasks.size()));
  std::vector<std::thread> pool;
  for (int k = 1; k < nt; ++k) {
    try {
      pool.emplace_back(worker_fenced);
    } catch (const std::system_error&) {   // fewer threads: the tasks still all run
      break;
    }
  }
  worker_fenced();
  for (auto& th : pool) th.join();
  cudaError_t last = cudaSuccess;
  for (auto e : ev) {
    cudaError_t r = cudaEventSynchronize(e);
    if (r != cudaSuccess) last = r;
  }
  cleanup();
  if (err.load() || last != cudaSuccess)
    return fail(CORR2D_ERR_CUDA, std::string("corr2d_fetch_mirrored: ") + cudaGetErrorString(cudaGetLastError()));
  if (d2h_bytes) *d2h_bytes = bytes;
  return CORR2D_OK;
}

}  // namespace

extern "C" int corr2d_fetch_mirrored(int dtype, const void* d_sync, const void* d_async, int64_t ld_dev, int n,
                                     void* h_sync, void* h_async, int64_t ld_host, int band, int fill_pct,
                                     int threads, int64_t* d2h_bytes, void* stream) {
  if (n < 0 || ld_dev < n || ld_host < n)
    return fail(CORR2D_ERR_DATA, "corr2d_fetch_mirrored: bad shape / leading dimensions");
  if (band <= 0 || band % kTileEdge)
    return fail(CORR2D_ERR_DATA, "corr2d_fetch_mirrored: band must be a positive multiple of 256");
  if (dtype != CORR2D_F64 && dtype != CORR2D_F32) return fail(CORR2D_ERR_DATA, "corr2d_fetch_mirrored: bad dtype");
  if (fill_pct < 0 || fill_pct > 100) return fail(CORR2D_ERR_DATA, "corr2d_fetch_mirrored: fill_pct outside [0, 100]");
  if (n == 0) {
    if (d2h_bytes) *d2h_bytes = 0;
    return CORR2D_OK;
  }
  if (!d_sync || !d_async || !h_sync || !h_async) return fail(CORR2D_ERR_DATA, "corr2d_fetch_mirrored: null plane");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == CORR2D_F64)
    return fetch_impl(static_cast<const double*>(d_sync), static_cast<const double*>(d_async), ld_dev, n,
                      static_cast<double*>(h_sync), static_cast<double*>(h_async), ld_host, band, fill_pct,
                      threads, d2h_bytes, st);
  return fetch_impl(static_cast<const float*>(d_sync), static_cast<const float*>(d_async), ld_dev, n,
                    static_cast<float*>(h_sync), static_cast<float*>(h_async), ld_host, band, fill_pct, threads,
                    d2h_bytes, st);
}
