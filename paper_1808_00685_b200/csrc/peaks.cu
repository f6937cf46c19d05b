// K3 -- cross-peak candidates of a correlation map (reference: analysis.py:136-201,
// SURVEY.md 8f row f4).
//
// A cross-peak candidate is a strict 8-neighbourhood local maximum of |sync| or
// |async| (the map padded with -inf, analysis.py:136-149) above a threshold
// (threshold_fraction * max|.|, :187-194); homo results keep the strict upper
// triangle only (:195-197).  The scan is one HBM pass over both planes: each
// CTA stages a 32 x 32 output tile plus a one-element halo of |sync| and |async|
// in shared memory, tiles entirely below the diagonal of a homo map are skipped,
// and candidates are appended as row-major linear indices through one atomic
// counter (the host sorts them, reproducing np.argwhere's order).
#include "common.cuh"

#include <cmath>

namespace corr2d {

constexpr int kPeakTile = 32;
constexpr int kPeakThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kPeakThreads) peaks_kernel(const T* __restrict__ sync, const T* __restrict__ asyn,
                                                             long long ld, int n1, int n2, int homo, double thr_s,
                                                             double thr_a, long long* __restrict__ out, long long cap,
                                                             unsigned long long* __restrict__ count) {
  constexpr int H = kPeakTile + 2;
  __shared__ double s_abs[H][H + 1];
  __shared__ double a_abs[H][H + 1];
  const int i0 = blockIdx.y * kPeakTile, k0 = blockIdx.x * kPeakTile;
  if (homo && k0 + kPeakTile - 1 <= i0) return;  // every (i, k) here has k <= i
  const double ninf = -INFINITY;
  for (int idx = threadIdx.x; idx < H * H; idx += blockDim.x) {
    const int r = idx / H, c = idx - r * H;
    const int gi = i0 - 1 + r, gk = k0 - 1 + c;
    double vs = ninf, va = ninf;
    if (gi >= 0 && gi < n1 && gk >= 0 && gk < n2) {
      const long long o = (long long)gi * ld + gk;
      vs = fabs((double)sync[o]);
      va = fabs((double)asyn[o]);
    }
    s_abs[r][c] = vs;
    a_abs[r][c] = va;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kPeakTile * kPeakTile; e += blockDim.x) {
    const int r = e / kPeakTile + 1, c = e % kPeakTile + 1;
    const int gi = i0 + r - 1, gk = k0 + c - 1;
    if (gi >= n1 || gk >= n2 || (homo && gk <= gi)) continue;
    auto is_peak = [&](const double (*m)[H + 1], double thr) {
      const double v = m[r][c];
      if (!(v > thr)) return false;
#pragma unroll
      for (int di = -1; di <= 1; ++di)
#pragma unroll
        for (int dk = -1; dk <= 1; ++dk)
          if ((di || dk) && !(v > m[r + di][c + dk])) return false;
      return true;
    };
    if (is_peak(s_abs, thr_s) || is_peak(a_abs, thr_a)) {
      const unsigned long long pos = atomicAdd(count, 1ull);
      if ((long long)pos < cap) out[pos] = (long long)gi * n2 + gk;
    }
  }
}

// Vectorised, persistent variant for 16-byte aligned planes: a tile is 32 rows
// x TW columns (TW = 32 lanes x one 16-byte vector: 128 fp32 / 64 fp64); each
// CTA walks tiles t, t + grid, ... and issues the NEXT tile's 16-byte loads
// into registers before scanning the current one from shared memory, so the
// HBM latency overlaps the scan.  |.| is kept in the planes' own precision.
template <typename T>
struct PeakTileRegs {
  static constexpr int VW = 16 / sizeof(T), TW = 32 * VW, TH = 32;
  static constexpr int NW = kPeakThreads / 32, RI = (TH + 2 + NW - 1) / NW;
  T v[RI][2][VW];
  T h[2];   // halo element of this thread (plane, side, row) = (threadIdx.x), if any
};

template <typename T>
__device__ __forceinline__ void peak_tile_load(PeakTileRegs<T>& R, const T* __restrict__ sync,
                                               const T* __restrict__ asyn, long long ld, int n1, int n2, int i0,
                                               int k0) {
  using P = PeakTileRegs<T>;
  constexpr int VW = P::VW, TW = P::TW, TH = P::TH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const T ninf = -INFINITY;
#pragma unroll
  for (int j = 0; j < P::RI; ++j) {
    const int r = warp + j * P::NW, gi = i0 - 1 + r, gk = k0 + lane * VW;
    const bool row_ok = r < TH + 2 && gi >= 0 && gi < n1;
#pragma unroll
    for (int pl = 0; pl < 2; ++pl) {
      const T* src = pl ? asyn : sync;
      if (row_ok && gk + VW <= n2) {
        if constexpr (sizeof(T) == 4) {
          const float4 q = __ldcs(reinterpret_cast<const float4*>(src + (long long)gi * ld + gk));
          R.v[j][pl][0] = q.x; R.v[j][pl][1] = q.y; R.v[j][pl][2] = q.z; R.v[j][pl][3] = q.w;
        } else {
          const double2 q = __ldcs(reinterpret_cast<const double2*>(src + (long long)gi * ld + gk));
          R.v[j][pl][0] = q.x; R.v[j][pl][1] = q.y;
        }
      } else {
#pragma unroll
        for (int e = 0; e < VW; ++e)
          R.v[j][pl][e] = (row_ok && gk + e < n2) ? src[(long long)gi * ld + gk + e] : ninf;
      }
    }
  }
  // halo columns k0 - 1 and k0 + TW: thread h < 4 (TH + 2) owns (plane, side, row)
  const int hh = threadIdx.x;
  if (hh < 4 * (TH + 2)) {
    const int pl = hh / (2 * (TH + 2)), side = (hh / (TH + 2)) & 1, r = hh % (TH + 2);
    const int gi = i0 - 1 + r, hk = side ? k0 + TW : k0 - 1;
    const T* src = pl ? asyn : sync;
    R.h[0] = (gi >= 0 && gi < n1 && hk >= 0 && hk < n2) ? src[(long long)gi * ld + hk] : ninf;
  }
}

template <typename T>
__global__ void __launch_bounds__(kPeakThreads) peaks_vec_kernel(const T* __restrict__ sync,
                                                                 const T* __restrict__ asyn, long long ld, int n1,
                                                                 int n2, int homo, T thr_s, T thr_a,
                                                                 long long* __restrict__ out, long long cap,
                                                                 unsigned long long* __restrict__ count) {
  using P = PeakTileRegs<T>;
  constexpr int VW = P::VW, TW = P::TW, TH = P::TH;
  constexpr int SW = TW + 2 + 1;               // smem row pitch (halo + pad)
  __shared__ T sm[2][TH + 2][SW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T ninf = -INFINITY;
  const int tcols = (n2 + TW - 1) / TW, trows = (n1 + TH - 1) / TH;
  const long long ntiles = (long long)tcols * trows;
  auto valid = [&](long long t) {               // homo: skip tiles with every k <= i
    const int I = (int)(t / tcols), J = (int)(t % tcols);
    return !(homo && J * TW + TW - 1 <= I * TH);
  };
  long long t = blockIdx.x;
  while (t < ntiles && !valid(t)) t += gridDim.x;
  PeakTileRegs<T> R;
  if (t < ntiles) peak_tile_load(R, sync, asyn, ld, n1, n2, (int)(t / tcols) * TH, (int)(t % tcols) * TW);
  while (t < ntiles) {
    const int i0 = (int)(t / tcols) * TH, k0 = (int)(t % tcols) * TW;
    // registers -> shared memory (|.|, -inf padding kept)
#pragma unroll
    for (int j = 0; j < P::RI; ++j) {
      const int r = warp + j * P::NW;
      if (r < TH + 2) {
#pragma unroll
        for (int pl = 0; pl < 2; ++pl)
#pragma unroll
          for (int e = 0; e < VW; ++e)
            sm[pl][r][1 + lane * VW + e] = R.v[j][pl][e] == ninf ? ninf : fabs(R.v[j][pl][e]);
      }
    }
    if (threadIdx.x < 4 * (TH + 2)) {
      const int hh = threadIdx.x, pl = hh / (2 * (TH + 2)), side = (hh / (TH + 2)) & 1, r = hh % (TH + 2);
      sm[pl][r][side ? TW + 1 : 0] = R.h[0] == ninf ? ninf : fabs(R.h[0]);
    }
    __syncthreads();
    // next tile's loads in flight during the scan
    long long tn = t + gridDim.x;
    while (tn < ntiles && !valid(tn)) tn += gridDim.x;
    if (tn < ntiles) peak_tile_load(R, sync, asyn, ld, n1, n2, (int)(tn / tcols) * TH, (int)(tn % tcols) * TW);
    for (int e = threadIdx.x; e < TH * TW; e += kPeakThreads) {
      const int r = e / TW + 1, c = e % TW + 1;
      const int gi = i0 + r - 1, gk = k0 + c - 1;
      if (gi >= n1 || gk >= n2 || (homo && gk <= gi)) continue;
      bool hit = false;
#pragma unroll
      for (int pl = 0; pl < 2; ++pl) {
        const T v = sm[pl][r][c];
        if (!hit && v > (pl ? thr_a : thr_s)) {   // most elements stop here
          bool ok = true;
#pragma unroll
          for (int di = -1; di <= 1; ++di)
#pragma unroll
            for (int dk = -1; dk <= 1; ++dk)
              if (di || dk) ok = ok && (v > sm[pl][r + di][c + dk]);
          hit = ok;
        }
      }
      if (hit) {
        const unsigned long long pos = atomicAdd(count, 1ull);
        if ((long long)pos < cap) out[pos] = (long long)gi * n2 + gk;
      }
    }
    __syncthreads();
    t = tn;
  }
}

// max |x| over an n1 x n2 plane (leading dimension ld) into *out (IEEE bits,
// reset by the caller's call below)
template <typename T>
__global__ void absmax_kernel(const T* __restrict__ x, long long ld, int n1, int n2,
                              unsigned long long* __restrict__ out) {
  double m = 0.0;
  const long long total = (long long)n1 * n2;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / n2, k = e - i * n2;
    m = fmax(m, fabs((double)x[i * ld + k]));
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomic_max_abs(out, m);
}

}  // namespace corr2d

using namespace corr2d;

extern "C" int corr2d_plane_absmax(int dtype, const void* x, int64_t ld, int n1, int n2, double* out_dev,
                                   void* stream) {
  if (!x || !out_dev || n1 < 1 || n2 < 1 || ld < n2) return fail(CORR2D_ERR_DATA, "corr2d_plane_absmax: bad arguments");
  if (dtype != CORR2D_F64 && dtype != CORR2D_F32) return fail(CORR2D_ERR_DATA, "corr2d_plane_absmax: bad dtype");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(out_dev, 0, sizeof(double), st) != cudaSuccess) return check_launch("absmax reset");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long total = (long long)n1 * n2;
  const long long want = (total + 255) / 256;
  const int grid = (int)(want < 8LL * sms ? want : 8LL * sms);
  auto* o = reinterpret_cast<unsigned long long*>(out_dev);
  if (dtype == CORR2D_F64) absmax_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(x), ld, n1, n2, o);
  else absmax_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(x), ld, n1, n2, o);
  return check_launch("absmax_kernel");
}

extern "C" int corr2d_find_peaks(int dtype, const void* sync, const void* asyn, int64_t ld, int n1, int n2, int homo,
                                 double thr_sync, double thr_async, int64_t* out_idx, int64_t capacity,
                                 unsigned long long* count, void* stream) {
  if (!sync || !asyn || !count || (capacity > 0 && !out_idx) || n1 < 1 || n2 < 1 || ld < n2 || capacity < 0)
    return fail(CORR2D_ERR_DATA, "corr2d_find_peaks: bad arguments");
  if (dtype != CORR2D_F64 && dtype != CORR2D_F32) return fail(CORR2D_ERR_DATA, "corr2d_find_peaks: bad dtype");
  if (homo && n1 != n2) return fail(CORR2D_ERR_DATA, "corr2d_find_peaks: homo needs n1 == n2");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(count, 0, sizeof(unsigned long long), st) != cudaSuccess) return check_launch("peaks reset");
  const dim3 grid((n2 + kPeakTile - 1) / kPeakTile, (n1 + kPeakTile - 1) / kPeakTile);
  if (grid.y > 65535) return fail(CORR2D_ERR_UNSUPPORTED, "corr2d_find_peaks: too many rows");
  auto* o = reinterpret_cast<long long*>(out_idx);
  const int esz = dtype == CORR2D_F64 ? 8 : 4;
  const bool vec = ((reinterpret_cast<uintptr_t>(sync) | reinterpret_cast<uintptr_t>(asyn)) & 15) == 0 &&
                   ((long long)ld * esz) % 16 == 0;
  if (vec) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int TW = 32 * (16 / esz);
    const long long tiles = (long long)((n2 + TW - 1) / TW) * ((n1 + kPeakTile - 1) / kPeakTile);
    // one tile per CTA measured fastest on cfg5 (1.31 ms vs 1.52 ms with 6
    // persistent CTAs / SM prefetching the next tile); the loop stays for grids
    // capped below the tile count (> 2^31 - 1 tiles)
    (void)sms;
    const dim3 g2((unsigned)(tiles < 0x7fffffffLL ? tiles : 0x7fffffffLL));
    if (dtype == CORR2D_F64)
      peaks_vec_kernel<double><<<g2, kPeakThreads, 0, st>>>(static_cast<const double*>(sync),
                                                             static_cast<const double*>(asyn), ld, n1, n2, homo,
                                                             thr_sync, thr_async, o, capacity, count);
    else  // thresholds are float32 values (the planes' dtype, analysis.py:187-194)
      peaks_vec_kernel<float><<<g2, kPeakThreads, 0, st>>>(static_cast<const float*>(sync),
                                                            static_cast<const float*>(asyn), ld, n1, n2, homo,
                                                            (float)thr_sync, (float)thr_async, o, capacity, count);
    return check_launch("peaks_vec_kernel");
  }
  if (dtype == CORR2D_F64)
    peaks_kernel<double><<<grid, kPeakThreads, 0, st>>>(static_cast<const double*>(sync),
                                                         static_cast<const double*>(asyn), ld, n1, n2, homo,
                                                         thr_sync, thr_async, o, capacity, count);
  else
    peaks_kernel<float><<<grid, kPeakThreads, 0, st>>>(static_cast<const float*>(sync),
                                                        static_cast<const float*>(asyn), ld, n1, n2, homo, thr_sync,
                                                        thr_async, o, capacity, count);
  return check_launch("peaks_kernel");
}
