// Small-m path (m <= 32, no resampling, fp64 operands: cfg1 m = 11, cfg2 m = 21).
//
//  * prep_small_kernel -- K1 alone (corr2d_prep): one warp per channel pair.
//  * small_fused_kernel -- the whole correlation in ONE launch
//    (corr2d_correlate_small_f64): K1 with one lane per channel (32-channel
//    blocks, each publishing a ready flag), then the contraction in 16 x 32
//    halves of 32 x 32 warp tiles, each waiting only for its two channel
//    blocks, straight from L2-resident operands into registers (DMMA, no
//    shared-memory staging, no grid or CTA barriers) and from the accumulators
//    to HBM.  At these sizes the step
//    is bound by launch latency and the output write (cfg1: 16 MB of planes,
//    2.5 us at HBM peak), so the two-kernel path's second launch, its two
//    memset nodes and its one-CTA-per-64x64-tile grid (4 warps per SM) were
//    the cost; the status / stat words are self-resetting instead.
//
// Reference path: preprocess.py:123-137, :198-259 (reference, sigma, scaling),
// fourier.py:61-82 (rfft along the perturbation axis), fourier.py:107-123
// (weighted half-spectrum cross sum x Norm, split into sync / async),
// engine_core.py:139-140 (finite check), dataset.py:159-170 (homo symmetry).
#include "prep_params.cuh"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace corr2d {

// One channel pair (c0, c0 + 1) of dataset p, one warp, lane t holding sample t
// of both channels -- no shared-memory staging and no CTA barriers, so K1 is
// one DRAM round trip plus a few hundred dependent instructions.  Statistics in
// the reference's order (sequential sums, the generic kernel's operations: the
// same bits), then a direct complex DFT of z = x_even + i x_odd (lane k -> Z_k,
// the generic radix stage's fma order), the channel split and the fp64 slots
// (s < p.mp; slots m .. mp-1 are zero).  tw: the m twiddles W^q.
__device__ __forceinline__ void small_pair(const PrepParams& p, const double2* tw, int c0, int lane) {
  const int m = p.m;
  if (c0 >= p.n) return;                       // whole warps only
  const bool has1 = c0 + 1 < p.n;
  double y[2] = {0.0, 0.0};
  int bad = 0;
  if (lane < m) {
    const long long o = (long long)lane * p.ld_raw + c0;
    if (p.in_f32) {
      const float* r = static_cast<const float*>(p.raw);
      y[0] = __ldg(r + o);
      if (has1) y[1] = __ldg(r + o + 1);
    } else {
      const double* r = static_cast<const double*>(p.raw);
      y[0] = __ldg(r + o);
      if (has1) y[1] = __ldg(r + o + 1);
    }
    bad = !isfinite(y[0]) + !isfinite(y[1]);
  }
  bad = warp_sum(bad);
  if (lane == 0 && bad) atomicAdd(&p.status[CORR2D_ST_NONFINITE], bad);

  const bool normalise = p.ref_mode != CORR2D_REF_NONE || p.alpha > 0.0;
  if (normalise) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (e == 1 && !has1) break;
      const int c = c0 + e;
      double ref = 0.0;
      if (p.ref_mode == CORR2D_REF_PROVIDED) {
        ref = __ldg(p.ref_in + c);
      } else if (p.ref_mode == CORR2D_REF_MEAN) {
        double sum = 0.0;                      // left to right (numpy's axis-0 order)
        // shuffles issued 8 at a time ahead of the (sequential) adds
        for (int k0 = 0; k0 < m; k0 += 8) {
          double v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = __shfl_sync(0xffffffffu, y[e], (k0 + k) & 31);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (k0 + k < m) sum = __dadd_rn(sum, v[k]);
        }
        ref = __ddiv_rn(sum, (double)m);
      }
      double scale = 1.0;
      if (p.alpha > 0.0) {
        double sigma;
        if (p.sigma_in) {
          sigma = __ldg(p.sigma_in + c);
        } else {
          double ss = 0.0;
          for (int k0 = 0; k0 < m; k0 += 8) {
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __shfl_sync(0xffffffffu, y[e], (k0 + k) & 31);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const double d = __dsub_rn(v[k], ref);
              if (k0 + k < m) ss = __dadd_rn(ss, __dmul_rn(d, d));
            }
          }
          sigma = __dsqrt_rn(__ddiv_rn(ss, (double)(m - 1)));
        }
        if (lane == 0) {
          if (p.sigma_out) p.sigma_out[c] = sigma;
          if (sigma == 0.0) {
            atomicAdd(&p.status[CORR2D_ST_ZEROVAR], 1);
            atomicMax(&p.status[CORR2D_ST_FIRST_ZEROVAR], INT_MAX - c);
          }
        }
        if (sigma == 0.0 && p.substitute) sigma = 1.0;
        scale = (p.alpha == 0.5) ? __dsqrt_rn(sigma) : (p.alpha == 1.0 ? sigma : pow(sigma, p.alpha));
      }
      if (lane == 0 && p.ref_out) p.ref_out[c] = ref;
      if (lane < m) {
        if (p.ref_mode != CORR2D_REF_NONE) y[e] = __dsub_rn(y[e], ref);
        if (p.alpha > 0.0) y[e] = __ddiv_rn(y[e], scale);
      }
    }
  }

  // Z_k = sum_t z_t W^(k t), z_t = y0_t + i y1_t
  double2 Z = make_double2(0.0, 0.0);
  {
    int q = 0;
    const int step = lane < m ? lane : 0;
    for (int t0 = 0; t0 < m; t0 += 4) {
      double2 x[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        x[k] = make_double2(__shfl_sync(0xffffffffu, y[0], (t0 + k) & 31), __shfl_sync(0xffffffffu, y[1], (t0 + k) & 31));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (t0 + k >= m) break;
        const double2 w = tw[q];
        Z.x = fma(x[k].x, w.x, fma(-x[k].y, w.y, Z.x));
        Z.y = fma(x[k].x, w.y, fma(x[k].y, w.x, Z.y));
        q += step;
        if (q >= m) q -= m;
      }
    }
  }
  // the two real spectra at bin w: (Z_w + conj Z_{m-w}) / 2 and (Z_w - conj Z_{m-w}) / (2i)
  const int mirror = lane < m ? (m - lane) % m : 0;
  const double2 Zr = make_double2(__shfl_sync(0xffffffffu, Z.x, mirror), __shfl_sync(0xffffffffu, Z.y, mirror));
  const double2 Y[2] = {make_double2(0.5 * (Z.x + Zr.x), 0.5 * (Z.y - Zr.y)),
                        make_double2(0.5 * (Z.y + Zr.y), -0.5 * (Z.x - Zr.x))};
  // fp64 slots (CORR2D_PACK_F64): s < K -> Re Y(s); K <= s < m -> Im Y(s - K + 1); rest 0
  const int K = m / 2 + 1;
  const bool even = (m % 2) == 0;
  const int s = lane;
  const int w = s < K ? s : (s < m ? s - K + 1 : 0);
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const double yr = __shfl_sync(0xffffffffu, Y[e].x, w), yi = __shfl_sync(0xffffffffu, Y[e].y, w);
    if ((e == 1 && !has1) || s >= p.mp) continue;
    double vphi = 0.0, vpsi = 0.0, vb = 0.0;
    if (s < m) {
      const bool edge = (w == 0 || (even && w == m / 2));
      const double R = yr, I = edge ? 0.0 : yi;
      double nr = p.norm * R, ni = p.norm * I;
      if (!edge) { nr *= 2.0; ni *= 2.0; }
      if (s < K) { vphi = nr; vpsi = ni; vb = R; }
      else { vphi = ni; vpsi = -nr; vb = I; }
    }
    const long long row = (long long)(c0 + e) * p.ld_pack + s;
    if (p.pack_roles & CORR2D_ROLE_A) {
      static_cast<double*>(p.a_phi)[row] = vphi;
      static_cast<double*>(p.a_psi)[row] = vpsi;
    }
    if (p.pack_roles & CORR2D_ROLE_B) static_cast<double*>(p.b)[row] = vb;
  }
}

constexpr int kSmallWarps = 8;

__device__ __forceinline__ void load_twiddles(double2* tw, int m) {
  for (int q = threadIdx.x; q < m; q += blockDim.x) {
    double sv, cv;
    sincospi(-2.0 * (double)q / (double)m, &sv, &cv);
    tw[q] = make_double2(cv, sv);
  }
}

__global__ void __launch_bounds__(32 * kSmallWarps) prep_small_kernel(const PrepParams p) {
  __shared__ double2 tw[32];
  load_twiddles(tw, p.m);
  __syncthreads();
  small_pair(p, tw, 2 * (blockIdx.x * kSmallWarps + (threadIdx.x >> 5)), threadIdx.x & 31);
}

bool small_eligible(const PrepParams& p) {
  if (const char* e = getenv("CORR2D_PREP_SMALL"))
    if (e[0] == '0') return false;
  return p.m <= 32 && p.resample_kind == CORR2D_RESAMPLE_NONE && !p.values_out && !p.half_out &&
         p.pack_kind == CORR2D_PACK_F64 && p.mp <= 32;
}

int launch_prep_small(const PrepParams& p, cudaStream_t st) {
  if (cudaMemsetAsync(p.status, 0, 4 * sizeof(int32_t), st) != cudaSuccess) return check_launch("status reset");
  const int pairs = (p.n + 1) / 2;
  prep_small_kernel<<<(pairs + kSmallWarps - 1) / kSmallWarps, 32 * kSmallWarps, 0, st>>>(p);
  return check_launch("prep_small_kernel");
}

// ---------------------------------------------------------------------------
// Fused small-m correlation: one launch per call.
// ---------------------------------------------------------------------------
constexpr int kFT = 32;          // warp tile edge (output rows and columns)
// one CTA per SM (every CTA resident: the flag waits cannot deadlock), as many
// warps as the register file holds: 16 at <= 128 registers (depth <= 16), 12 above
// Warps per CTA (one CTA per SM): 16 at <= 128 registers (depth <= 16), 12 above.
// (Measured alternatives: 8 / 16 warps at depth 24, a bulk-copy
// staging epilogue, CTA-contiguous unit ranges -- none faster.)
#ifndef CORR2D_SMALL_W12
#define CORR2D_SMALL_W12 16
#endif
#ifndef CORR2D_SMALL_W34
#define CORR2D_SMALL_W34 12
#endif
template <int NCH> __host__ __device__ constexpr int fused_warps() { return NCH <= 2 ? CORR2D_SMALL_W12 : CORR2D_SMALL_W34; }

struct SmallParams {
  PrepParams p1, p2;        // K1 of dataset 1 (roles A, and B when homo) and dataset 2 (role B)
  int homo, n1, n2;
  int nb1;                  // 32-channel blocks of dataset 1 (flags [0, nb1); dataset 2 follows)
  int row0, row1, I0, I1, T;
  long long tile0, tiles;   // this launch's range of the warp-tile enumeration
  const double* a_phi;
  const double* a_psi;
  const double* b;
  long long ld_pack;
  double* phi;
  double* psi;
  long long ld_out;
  int vec;                  // planes 16-B aligned with an even ld_out: 16-byte direct stores
  unsigned long long* stats;
  int* work;                // see kW* below; zero-filled once by the caller
  int* status1;
  int* status2;
  unsigned long long* trace;  // CORR2D_SMALL_TRACE=1: per-CTA globaltimer stamps (start, phase 1 done, first unit, end)
};

// work-buffer words (int32 indices)
constexpr int kWStatus1 = 0;   // [0, 4)  K1 status accumulator, dataset 1
constexpr int kWStatus2 = 4;   // [4, 8)  dataset 2
constexpr int kWDone = 8;      // CTAs finished (the last one publishes and resets)
constexpr int kWEpoch = 9;     // launch epoch: block flags of this launch read epoch + 1
constexpr int kWStats = 10;    // [10, 16) max|sync|, max|async|, non-finite count (3 x uint64)
constexpr int kWK1Done = 16;   // K1 tasks finished (phase-2 warps stop checking flags once all are)
constexpr int kWFlags = 20;    // ready flags: kMaxGroups per 32-channel block
constexpr int kMaxGroups = 5;  // 4-bin groups of K = m / 2 + 1 <= 17

enum FusedMode { kFPlain = 0, kFMirror = 1, kFDiag = 2, kFTransOnly = 3 };

// The warp-tile enumeration of a row shard [I0, I1) of 32-row tiles (the
// enumeration of contract_f64's decode_tile at 32 x 32): homo row tile I0 + d
// owns column tiles [0, I0) (lower tiles outside the shard's square, computed
// as their globally-upper mirror and written through the transpose) and
// [I0 + d, T); every element gets the same bits for any partition.
__device__ __forceinline__ void fused_decode(const SmallParams& p, long long b, int& I, int& J, int& mode) {
  if (!p.homo) {
    I = p.I0 + (int)(b / p.T);
    J = (int)(b % p.T);
    mode = kFPlain;
    return;
  }
  // first guess in fp32 (an fp64 sqrt would queue on the FP64 pipe behind the
  // DMMAs of co-resident CTAs), corrected exactly below
  const long long t2 = 2LL * p.T + 1;
  const long long disc = t2 * t2 - 8LL * b;
  long long d = (long long)((float)t2 - sqrtf((float)(disc > 0 ? disc : 0))) / 2;
  auto S = [&](long long dd) { return dd * (long long)p.T - dd * (dd - 1) / 2; };
  if (d < 0) d = 0;
  while (d > 0 && S(d) > b) --d;
  while (S(d + 1) <= b) ++d;
  I = p.I0 + (int)d;
  const long long o = b - S(d);
  if (o < p.I0) {
    J = I;
    I = (int)o;
    mode = kFTransOnly;
  } else {
    J = I + (int)(o - p.I0);
    mode = (J == I) ? kFDiag : (J < p.I1 ? kFMirror : kFPlain);
  }
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acquire(const int* a) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// Spin (one lane) until a block flag carries this launch's epoch.  The flags
// are set by phase-1 warps that never wait on anything, and every CTA is
// resident (one per SM, grid from the occupancy calculator), so the wait ends;
// if residency were ever violated the kernel traps after 20 s instead of
// hanging the device.
__device__ __forceinline__ int ld_relaxed(const int* a) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

__device__ __forceinline__ void wait_flag(const int* flag, int want) {
  if (ld_acquire(flag) == want) return;
  // relaxed polls with exponential back-off (an acquire load invalidates L1 and
  // a thousand warps polling one L2 line slow down the K1 they are waiting
  // for), then one acquire load
  const unsigned long long t0 = global_ns();
  unsigned ns = 64;
  while (ld_relaxed(flag) != want) {
    __nanosleep(ns);
    ns = ns < 256 ? 2 * ns : 256;
    if (global_ns() - t0 > 20000000000ull) __trap();
  }
  (void)ld_acquire(flag);
}

// The K1 fields one dataset's lanes read, loaded once per block (the kernel
// parameter of the selected dataset would otherwise be re-read through a
// generic pointer on every use).
struct ChanArgs {
  const void* raw;
  long long ld_raw, ld_pack;
  const double* ref_in;
  const double* sigma_in;
  double* ref_out;
  double* sigma_out;
  double* a_phi;
  double* a_psi;
  double* b;
  int* status;
  double alpha, norm;
  int n, m, mp, in_f32, ref_mode, substitute, roles;
};

__device__ __forceinline__ ChanArgs chan_args(const PrepParams& p) {
  ChanArgs a;
  a.raw = p.raw; a.ld_raw = p.ld_raw; a.ld_pack = p.ld_pack; a.ref_in = p.ref_in; a.sigma_in = p.sigma_in;
  a.ref_out = p.ref_out; a.sigma_out = p.sigma_out;
  a.a_phi = static_cast<double*>(p.a_phi); a.a_psi = static_cast<double*>(p.a_psi); a.b = static_cast<double*>(p.b);
  a.status = p.status; a.alpha = p.alpha; a.norm = p.norm; a.n = p.n; a.m = p.m; a.mp = p.mp;
  a.in_f32 = p.in_f32; a.ref_mode = p.ref_mode; a.substitute = p.substitute; a.roles = p.pack_roles;
  return a;
}

// K1 of one spectral channel per lane (channel c): the reference's statistics
// in its order -- sequential sums, the same IEEE operations as the generic /
// small K1 kernels, so reference, sigma and values have the same bits -- then
// a direct real DFT of bins 4g .. 4g + 3 (ceil(K / 4) warps share a block, each
// redoing the cheap statistics), packed straight into the channel's operand
// rows (fp64 slots, zero padded to mp).
// One warp runs this once per launch on an SM, so its cost is latency: the
// samples arrive by cp.async into the warp's shared column block ys[t][lane]
// (all m copies in flight at once), and every step is a short runtime loop --
// straight-line unrolled code here is fetched cold, line by line, and cost
// microseconds of instruction-fetch stalls.
__device__ __forceinline__ void chan_lane(const ChanArgs& p, const double2* tw, double* ys, int c, int lane, int g,
                                          unsigned long long* tr = nullptr) {
  const bool owner = g == 0;                     // group 0 reports status / reference / sigma
  const int m = p.m;
  const bool valid = c < p.n;
  const int cc = valid ? c : p.n - 1;
  {
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(ys + lane));
    if (p.in_f32) {
      const float* r = static_cast<const float*>(p.raw) + cc;
      for (int t = 0; t < m; ++t)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst + 256u * t), "l"(r + (long long)t * p.ld_raw) : "memory");
    } else {
      const double* r = static_cast<const double*>(p.raw) + cc;
      for (int t = 0; t < m; ++t)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + 256u * t), "l"(r + (long long)t * p.ld_raw) : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  }
  // samples -> double in place (f32: the low word of each slot); non-finite count
  int bad = 0;
  for (int t = 0; t < m; ++t) {
    double v = p.in_f32 ? (double)reinterpret_cast<const float*>(ys + 32 * t + lane)[0] : ys[32 * t + lane];
    ys[32 * t + lane] = v;
    bad += !isfinite(v);
  }
  bad = valid ? bad : 0;
  bad = warp_sum(bad);
  if (tr && lane == 0) tr[4] = global_ns();
  if (owner && lane == 0 && bad) atomicAdd(&p.status[CORR2D_ST_NONFINITE], bad);
  if (!valid) return;                            // no warp-collective operation follows
  if (p.ref_mode != CORR2D_REF_NONE || p.alpha > 0.0) {
    double ref = 0.0;
    if (p.ref_mode == CORR2D_REF_PROVIDED) {
      ref = __ldg(p.ref_in + c);
    } else if (p.ref_mode == CORR2D_REF_MEAN) {
      double sum = 0.0;                          // left to right (numpy's axis-0 order)
      for (int t = 0; t < m; ++t) sum = __dadd_rn(sum, ys[32 * t + lane]);
      ref = __ddiv_rn(sum, (double)m);
    }
    double scale = 1.0;
    if (p.alpha > 0.0) {
      double sigma;
      if (p.sigma_in) {
        sigma = __ldg(p.sigma_in + c);
      } else {
        double ss = 0.0;
        for (int t = 0; t < m; ++t) {
          const double d = __dsub_rn(ys[32 * t + lane], ref);
          ss = __dadd_rn(ss, __dmul_rn(d, d));
        }
        sigma = __dsqrt_rn(__ddiv_rn(ss, (double)(m - 1)));
      }
      if (owner && p.sigma_out) p.sigma_out[c] = sigma;
      if (owner && sigma == 0.0) {
        atomicAdd(&p.status[CORR2D_ST_ZEROVAR], 1);
        atomicMax(&p.status[CORR2D_ST_FIRST_ZEROVAR], INT_MAX - c);
      }
      if (sigma == 0.0 && p.substitute) sigma = 1.0;
      scale = (p.alpha == 0.5) ? __dsqrt_rn(sigma) : (p.alpha == 1.0 ? sigma : pow(sigma, p.alpha));
    }
    if (owner && p.ref_out) p.ref_out[c] = ref;
    const bool sub = p.ref_mode != CORR2D_REF_NONE, div = p.alpha > 0.0;
    for (int t = 0; t < m; ++t) {
      double v = ys[32 * t + lane];
      if (sub) v = __dsub_rn(v, ref);
      if (div) v = __ddiv_rn(v, scale);
      ys[32 * t + lane] = v;
    }
  }
  if (tr && lane == 0) tr[5] = global_ns();
  // Y(w) = sum_t y_t W^(w t), w < K; slots: s < K -> Re Y(s), K <= s < m -> Im Y(s - K + 1)
  const int K = m / 2 + 1;
  const bool even = (m % 2) == 0;
  double* aphi = p.a_phi + (long long)c * p.ld_pack;
  double* apsi = p.a_psi + (long long)c * p.ld_pack;
  double* bb = p.b + (long long)c * p.ld_pack;
  const bool roleA = p.roles & CORR2D_ROLE_A, roleB = p.roles & CORR2D_ROLE_B;
  {
    const int w0 = 4 * g;                        // this warp's bins w0 .. w0 + 3
    double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
    int q[4] = {0, 0, 0, 0};
#pragma unroll 2
    for (int t = 0; t < m; ++t) {
      const double yt = ys[32 * t + lane];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 wv = tw[q[k]];
        re[k] = fma(yt, wv.x, re[k]);
        im[k] = fma(yt, wv.y, im[k]);
        q[k] += w0 + k;
        if (q[k] >= m) q[k] -= m;
      }
    }
    for (int k = 0; k < 4; ++k) {
      const int w = w0 + k;
      if (w >= K) break;
      const bool edge = (w == 0 || (even && w == m / 2));
      const double R = re[k], I = edge ? 0.0 : im[k];
      double nr = p.norm * R, ni = p.norm * I;
      if (!edge) { nr *= 2.0; ni *= 2.0; }
      if (roleA) { aphi[w] = nr; apsi[w] = ni; }
      if (roleB) bb[w] = R;
      const int s = K + w - 1;                   // the Im slot of bin w
      if (w >= 1 && s < m) {
        if (roleA) { aphi[s] = ni; apsi[s] = -nr; }
        if (roleB) bb[s] = I;
      }
    }
  }
  for (int s = m; owner && s < p.mp; ++s) {
    if (roleA) { aphi[s] = 0.0; apsi[s] = 0.0; }
    if (roleB) bb[s] = 0.0;
  }
  if (tr && lane == 0) tr[6] = global_ns();
}

__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Operand loads.  L1-cached: a warp reads a channel block only after an
// acquire that saw its K1 flag (or the all-done count), and every acquire
// invalidates the SM's L1 (CCTL.IVALL), so no line of operand data cached
// before it was final survives; neighbouring tiles of a CTA then share rows.
#ifndef CORR2D_SMALL_L1
#define CORR2D_SMALL_L1 1
#endif
__device__ __forceinline__ double2 ld_op(const double* a) {
#if CORR2D_SMALL_L1
  double2 v;
  asm volatile("ld.global.ca.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a));
  return v;
#else
  return __ldcg(reinterpret_cast<const double2*>(a));
#endif
}

__device__ __forceinline__ unsigned long long abits(double x) { return abs_bits(x); }

template <int NCH>
__global__ void __launch_bounds__(32 * fused_warps<NCH>(), 1) small_fused_kernel(const __grid_constant__ SmallParams p) {
  constexpr int kFusedWarps = fused_warps<NCH>();
  constexpr int kK1Warps = 4;                     // warps per CTA that take K1 blocks
  __shared__ double2 tw[32];
  __shared__ double ys[kK1Warps][32 * 32];        // K1 sample columns [t][lane] per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // global warp index, CTA-minor: consecutive work items land on different SMs
  const int gw = warp * (int)gridDim.x + blockIdx.x;
  const int W = gridDim.x * kFusedWarps;

  int* flags = p.work + kWFlags;
  unsigned long long* tr = p.trace ? p.trace + 32 * blockIdx.x : nullptr;
  int unit_no = 0;
  if (tr && threadIdx.x == 0) tr[0] = global_ns();

  // ---- phase 1: K1, one warp per 32-channel block, one lane per channel ----
  for (int q = threadIdx.x; q < p.p1.m; q += blockDim.x) {
    double sv, cv;
    sincospi(-2.0 * (double)q / (double)p.p1.m, &sv, &cv);
    tw[q] = make_double2(cv, sv);
  }
  // programmatic dependent launch: everything above overlapped the previous
  // kernel's tail; from here on memory written by it is visible
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  __syncthreads();
  // this launch's epoch (bumped only by the last CTA of the previous launch)
  const int want = *reinterpret_cast<volatile const int*>(p.work + kWEpoch) + 1;
  const int G = (p.p1.m / 2 + 1 + 3) / 4;         // 4-bin groups per channel block (<= kMaxGroups)
  if (warp < kK1Warps) {
    // K1 tasks (block, bin group) on the first kK1Warps warps of every CTA, CTA-minor
    const int nb2 = p.homo ? 0 : (p.n2 + 31) / 32;
    const int slot = warp * (int)gridDim.x + blockIdx.x;
    for (int task = slot; task < (p.nb1 + nb2) * G; task += kK1Warps * (int)gridDim.x) {
      const int blk = task / G, g = task - blk * G;
      const bool one = blk < p.nb1;                 // one call site: the K1 code is inlined once
      const ChanArgs args = chan_args(one ? p.p1 : p.p2);
      chan_lane(args, tw, ys[warp], 32 * (one ? blk : blk - p.nb1) + lane, lane, g, task == slot ? tr : nullptr);
      __threadfence();                             // this lane's rows, before the flag
      __syncwarp();
      if (tr && task == slot && lane == 0) tr[7] = global_ns();
      if (lane == 0) {
        asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(flags + kMaxGroups * blk + g), "r"(want) : "memory");
        atomicAdd(p.work + kWK1Done, 1);
      }
    }
  }
  if (tr) { __syncthreads(); if (threadIdx.x == 0) tr[1] = global_ns(); }

  // ---- phase 2: 16-row halves of 32 x 32 tiles, operands straight from L2,
  //      each unit waiting only for its two channel blocks ----
  const int lr = lane >> 2, lk = lane & 3;
  const long long ld = p.ld_pack;
  const int fB = p.homo ? 0 : p.nb1;
  unsigned long long mphi = 0, mpsi = 0;
  bool first = true;
  bool all_ready = false;                          // every K1 task of this launch seen finished
  const int k1_tasks = (p.nb1 + (p.homo ? 0 : (p.n2 + 31) / 32)) * G;
  const long long units = 2 * p.tiles;
  // static round robin over every warp of the grid (a shared claim counter
  // measured slower -- thousands of warps serialise on one L2 atomic -- and so
  // did CTA-contiguous unit ranges)
  const long long u_step = W;
  for (long long u = gw; u < units;) {
    int I, J, mode;
    fused_decode(p, p.tile0 + (u >> 1), I, J, mode);
    const int h = (int)(u & 1);
    const int r0 = I * kFT + h * 16;
    if (!all_ready) {
      int done = 0;
      if (lane == 0) done = ld_acquire(p.work + kWK1Done);
      all_ready = __shfl_sync(0xffffffffu, done, 0) == k1_tasks;
      if (!all_ready && lane < G) {
        wait_flag(flags + kMaxGroups * I + lane, want);
        wait_flag(flags + kMaxGroups * (fB + J) + lane, want);
      }
      __syncwarp();
    }
    u += u_step;
    if (r0 >= p.n1) continue;
    if (tr && blockIdx.x == 0 && warp == 0 && lane == 0 && unit_no > 0 && unit_no <= 6) tr[10 + 3 * (unit_no - 1)] = global_ns();
    const bool ut = tr && blockIdx.x == 0 && warp == 0 && lane == 0 && unit_no < 6;
    if (tr) ++unit_no;
    if (ut) tr[8 + 3 * (unit_no - 1)] = global_ns();
    if (tr && first && lane == 0 && warp == 0) tr[2] = global_ns();
    first = false;
    double aphi[4][4], apsi[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int c = 0; c < 4; ++c) aphi[nt][c] = apsi[nt][c] = 0.0;
    const int ra = min(r0 + lr, p.n1 - 1), rb = min(r0 + lr + 8, p.n1 - 1);
    const double* pa = p.a_phi + (long long)ra * ld + 2 * lk;
    const double* pb = p.a_phi + (long long)rb * ld + 2 * lk;
    const double* sa = p.a_psi + (long long)ra * ld + 2 * lk;
    const double* sb = p.a_psi + (long long)rb * ld + 2 * lk;
    const double* bc[4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
      bc[nt] = p.b + (long long)min(J * kFT + nt * 8 + lr, p.n2 - 1) * ld + 2 * lk;
    // depth chunks of 8: lane lk supplies slots 2 lk (first MMA) and 2 lk + 1
    // (second) of A and B alike -- a permutation of the depth, exact
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const double2 a0 = ld_op(pa + 8 * ch);
      const double2 a1 = ld_op(pb + 8 * ch);
      const double2 s0 = ld_op(sa + 8 * ch);
      const double2 s1 = ld_op(sb + 8 * ch);
      double2 bf[4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = ld_op(bc[nt] + 8 * ch);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        dmma(aphi[nt], a0.x, a1.x, bf[nt].x);
        dmma(apsi[nt], s0.x, s1.x, bf[nt].x);
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        dmma(aphi[nt], a0.y, a1.y, bf[nt].y);
        dmma(apsi[nt], s0.y, s1.y, bf[nt].y);
      }
    }
    if (ut) {
      double z = 0.0;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) z += aphi[nt][0] + apsi[nt][3];   // wait for the accumulators
      tr[9 + 3 * (unit_no - 1)] = global_ns() + (z == 12345.678 ? 1 : 0);
    }
    // ---- epilogue: lane holds rows (lr, lr + 8) x columns (2 lk, 2 lk + 1) of each n8 tile
    const bool interior = mode != kFDiag && p.vec && r0 + 16 <= min(p.n1, p.row1) && (J + 1) * kFT <= p.n2 &&
                          (mode == kFPlain || (J * kFT >= p.row0 && (J + 1) * kFT <= p.row1));
    if (interior) {
      // branch-free fast path: full 16 x 32 unit, 16-byte direct stores, 8-byte mirror stores
      const bool direct = mode != kFTransOnly, mirror = mode != kFPlain;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int gi = r0 + lr + 8 * hh, gj = J * kFT + nt * 8 + 2 * lk;
          const double f0 = aphi[nt][2 * hh], f1 = aphi[nt][2 * hh + 1];
          const double s0 = apsi[nt][2 * hh], s1 = apsi[nt][2 * hh + 1];
          mphi = max(mphi, max(abits(f0), abits(f1)));
          mpsi = max(mpsi, max(abits(s0), abits(s1)));
          if (direct) {
            const long long o = (long long)(gi - p.row0) * p.ld_out + gj;
            __stcs(reinterpret_cast<double2*>(p.phi + o), make_double2(f0, f1));
            __stcs(reinterpret_cast<double2*>(p.psi + o), make_double2(s0, s1));
          }
          if (mirror) {
            const long long o = (long long)(gj - p.row0) * p.ld_out + gi;
            __stcs(p.phi + o, f0);
            __stcs(p.psi + o, neg_bits(s0));
            __stcs(p.phi + o + p.ld_out, f1);
            __stcs(p.psi + o + p.ld_out, neg_bits(s1));
          }
        }
      continue;
    }
    const bool direct = mode != kFTransOnly;
    const bool mirror = mode != kFPlain;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int rl = h * 16 + lr + 8 * hh, cl = nt * 8 + 2 * lk;   // tile-local
        const int gi = I * kFT + rl, gj = J * kFT + cl;
        double f0 = aphi[nt][2 * hh], f1 = aphi[nt][2 * hh + 1];
        double s0 = apsi[nt][2 * hh], s1 = apsi[nt][2 * hh + 1];
        bool d0 = direct, d1 = direct, m0 = mirror, m1 = mirror;
        if (mode == kFDiag) {               // upper part incl. the diagonal, mirrored below it
          d0 = rl <= cl; d1 = rl <= cl + 1;
          m0 = rl < cl; m1 = rl < cl + 1;
          if (rl == cl) s0 = 0.0;
          if (rl == cl + 1) s1 = 0.0;
        }
        if (gi >= p.n1) { d0 = d1 = m0 = m1 = false; }
        if (gj >= p.n2) { d0 = m0 = false; }
        if (gj + 1 >= p.n2) { d1 = m1 = false; }
        if (gi >= p.row1) { d0 = d1 = false; }
        if (d0 || m0) { mphi = max(mphi, abits(f0)); mpsi = max(mpsi, abits(s0)); }
        if (d1 || m1) { mphi = max(mphi, abits(f1)); mpsi = max(mpsi, abits(s1)); }
        if (d0 || d1) {
          const long long o = (long long)(gi - p.row0) * p.ld_out + gj;
          if (d0 && d1 && p.vec) {
            __stcs(reinterpret_cast<double2*>(p.phi + o), make_double2(f0, f1));
            __stcs(reinterpret_cast<double2*>(p.psi + o), make_double2(s0, s1));
          } else {
            if (d0) { __stcs(p.phi + o, f0); __stcs(p.psi + o, s0); }
            if (d1) { __stcs(p.phi + o + 1, f1); __stcs(p.psi + o + 1, s1); }
          }
        }
        // mirror: out[j][i] = sync[i][j], -async[i][j] (rows j of the shard only)
        if (m0 && gj >= p.row0 && gj < p.row1) {
          const long long o = (long long)(gj - p.row0) * p.ld_out + gi;
          __stcs(p.phi + o, f0);
          __stcs(p.psi + o, neg_bits(s0));
        }
        if (m1 && gj + 1 >= p.row0 && gj + 1 < p.row1) {
          const long long o = (long long)(gj + 1 - p.row0) * p.ld_out + gi;
          __stcs(p.phi + o, f1);
          __stcs(p.psi + o, neg_bits(s1));
        }
      }
  }
  // ---- max|.| and the finite check (integer pipe, as contract_f64): one set of
  //      atomics per warp into the accumulator words
  constexpr unsigned long long kInf = 0x7ff0000000000000ull;
  int bad = (mphi >= kInf) + (mpsi >= kInf);
  mphi = min(mphi, kInf);
  mpsi = min(mpsi, kInf);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mphi = max(mphi, (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)mphi, o));
    mpsi = max(mpsi, (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)mpsi, o));
  }
  bad = warp_sum(bad);
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(p.work + kWStats);
  if (lane == 0) {
    if (mphi) atomicMax(&acc[0], mphi);
    if (mpsi) atomicMax(&acc[1], mpsi);
    if (bad) atomicAdd(&acc[2], (unsigned long long)bad);
  }
  // ---- the last CTA publishes status / stats and leaves the work words zero
  //      (flags keep their epoch; the epoch moves on)
  __syncthreads();
  if (threadIdx.x == 0) {
    if (tr) tr[3] = global_ns();
    __threadfence();
    if (atomicAdd(p.work + kWDone, 1) == (int)gridDim.x - 1) {
      __threadfence();
      volatile int* wv = p.work;
      for (int k = 0; k < 4; ++k) {
        p.status1[k] = wv[kWStatus1 + k];
        if (p.status2) p.status2[k] = wv[kWStatus2 + k];
        wv[kWStatus1 + k] = 0;
        wv[kWStatus2 + k] = 0;
      }
      volatile unsigned long long* av = acc;
      for (int k = 0; k < 3; ++k) {
        p.stats[k] = av[k];
        av[k] = 0ull;
      }
      wv[kWDone] = 0;
      wv[kWK1Done] = 0;
      wv[kWEpoch] = want;
      __threadfence();
    }
  }
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

static long long fused_tile_count(int n1, int n2, int homo, int row0, int row1) {
  const long long I0 = row0 / kFT, I1 = (row1 + kFT - 1) / kFT, T = (n2 + kFT - 1) / kFT;
  const long long R = I1 - I0;
  return homo ? R * T - R * (R - 1) / 2 : R * T;
}

template <int NCH>
static int launch_fused(const SmallParams& p, cudaStream_t st) {
  // one CTA per SM of the CURRENT device (cached per device: the grid must
  // never exceed what is co-resident, or the flag waits could not complete)
  static int grids[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(CORR2D_ERR_UNSUPPORTED, "small_fused_kernel: device index >= 64");
  int& grid = grids[dev];
  if (grid == 0) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, small_fused_kernel<NCH>, 32 * fused_warps<NCH>(), 0);
    if (per_sm < 1 || sms < 1) return fail(CORR2D_ERR_CUDA, "small_fused_kernel: no resident CTA");
    grid = sms;   // one per SM even if more would fit: one K1 slot set and one arrival per SM
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(32 * fused_warps<NCH>());
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  // programmatic dependent launch: this grid's launch and prologue overlap the
  // previous kernel's tail (griddepcontrol.wait in the kernel orders memory);
  // CORR2D_SMALL_PDL=0 disables
  static const int pdl = [] { const char* e = getenv("CORR2D_SMALL_PDL"); return e && e[0] == '0' ? 0 : 1; }();
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  // the cooperative attribute (guaranteed co-residency) costs ~7 us per launch in
  // a graph (cfg1: 22 vs 15 us per step); with one CTA per SM from the occupancy
  // calculator every CTA is resident once the stream reaches the kernel, and the
  // barrier traps rather than hangs if that is ever violated.  CORR2D_SMALL_COOP=1
  // restores the attribute.
  static const int coop = [] { const char* e = getenv("CORR2D_SMALL_COOP"); return e && e[0] == '1' ? 1 : 0; }();
  cfg.numAttrs = 1 + coop;
  static unsigned long long* trace = nullptr;
  const char* te = getenv("CORR2D_SMALL_TRACE");   // read per launch (experiments toggle it)
  const bool want_trace = te && te[0] == '1';
  SmallParams q = p;
  if (want_trace) {
    if (!trace) cudaMalloc(&trace, 32 * sizeof(unsigned long long) * grid);
    cudaMemsetAsync(trace, 0, 32 * sizeof(unsigned long long) * grid, st);
    q.trace = trace;
  }
  cudaLaunchKernelEx(&cfg, small_fused_kernel<NCH>, q);
  if (want_trace) {
    std::vector<unsigned long long> h(32 * (size_t)grid);
    cudaMemcpyAsync(h.data(), trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < grid; ++b) t0 = std::min(t0, h[32 * b]);
    double mx[8] = {0}, avg[8] = {0};
    int cnt[8] = {0};
    for (int b = 0; b < grid; ++b)
      for (int k = 0; k < 8; ++k) {
        if (!h[32 * b + k]) continue;
        const double v = (double)(h[32 * b + k] - t0);
        mx[k] = std::max(mx[k], v);
        avg[k] += v;
        ++cnt[k];
      }
    const char* names[8] = {"start", "phase1", "first-unit", "end", "k1-loaded", "k1-stats", "k1-packed", "k1-fenced"};
    fprintf(stderr, "small_fused trace (ns, max/avg):");
    for (int k = 0; k < 8; ++k) fprintf(stderr, " %s %.0f/%.0f", names[k], mx[k], cnt[k] ? avg[k] / cnt[k] : 0.0);
    fprintf(stderr, "\nwarp 0 of CTA 0, per unit (ns: flags-ok, mma-done, stored):");
    for (int u = 0; u < 6; ++u)
      if (h[8 + 3 * u]) fprintf(stderr, " [%.0f %.0f %.0f]", (double)(h[8 + 3 * u] - t0), (double)(h[9 + 3 * u] - t0),
                                (double)(h[10 + 3 * u] - t0));
    fprintf(stderr, "\n");
  }
  return check_launch("small_fused_kernel");
}

}  // namespace corr2d

using namespace corr2d;

extern "C" int corr2d_small_depth(int m) { return (m >= 2 && m <= 32) ? (m + 7) / 8 * 8 : -1; }

extern "C" int64_t corr2d_small_tile_count(int n1, int n2, int homo, int row0, int row1) {
  if (n1 < 1 || n2 < 1 || row0 < 0 || row1 > n1 || row0 >= row1 || (homo && n1 != n2)) return -1;
  return fused_tile_count(n1, n2, homo, row0, row1);
}

extern "C" int corr2d_correlate_small_f64(
    int in_dtype, const void* raw1, int64_t ld_raw1, const void* raw2, int64_t ld_raw2,
    int m, int n1, int n2,
    int ref_mode1, const double* ref_in1, const double* sigma_in1,
    int ref_mode2, const double* ref_in2, const double* sigma_in2,
    double alpha, int substitute_zero_var, double norm_const,
    double* a_phi, double* a_psi, double* b, int64_t ld_pack,
    double* ref_out1, double* sigma_out1, double* ref_out2, double* sigma_out2,
    int row0, int row1, int64_t tile0, int64_t tile1,
    double* phi, double* psi, int64_t ld_out,
    int32_t* status1, int32_t* status2, unsigned long long* stats, int32_t* work, void* stream) {
  const bool homo = raw2 == nullptr;
  if (!raw1 || !a_phi || !a_psi || !b || !phi || !psi || !status1 || !stats || !work || (!homo && !status2))
    return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: null pointer");
  if (in_dtype != CORR2D_F64 && in_dtype != CORR2D_F32) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad dtype");
  const int mp = corr2d_small_depth(m);
  if (mp < 0) return fail(CORR2D_ERR_UNSUPPORTED, "corr2d_correlate_small_f64: needs 2 <= m <= 32");
  if (n1 < 1 || n2 < 1) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad sizes");
  if (homo && n1 != n2) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: homo needs n1 == n2");
  if (ld_raw1 < n1 || (!homo && ld_raw2 < n2)) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: ld_raw < n");
  if (ld_pack < mp || ld_pack % 2 || (reinterpret_cast<uintptr_t>(a_phi) | reinterpret_cast<uintptr_t>(a_psi) |
                                      reinterpret_cast<uintptr_t>(b)) & 15)
    return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: ld_pack must be even and >= the packed depth, operands 16-B aligned");
  if (ld_out < n2) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: ld_out < n2");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(CORR2D_ERR_DATA, "scaling exponent must lie in [0, 1]");
  if (row0 < 0 || row1 > n1 || row0 >= row1 || row0 % kFT || (row1 != n1 && row1 % kFT))
    return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: row shard bounds must be multiples of 32 (or n1)");
  for (int r : {ref_mode1, ref_mode2})
    if (r < CORR2D_REF_MEAN || r > CORR2D_REF_NONE) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad ref_mode");
  if ((ref_mode1 == CORR2D_REF_PROVIDED && !ref_in1) || (!homo && ref_mode2 == CORR2D_REF_PROVIDED && !ref_in2))
    return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: provided reference missing");

  SmallParams p{};
  auto prep = [&](PrepParams& q, const void* raw, int64_t ld_raw, int n, int ref_mode, const double* ref_in,
                  const double* sigma_in, int roles, double* ref_out, double* sigma_out, int* acc) {
    q.raw = raw; q.in_f32 = in_dtype == CORR2D_F32; q.ld_raw = ld_raw; q.m_in = m; q.n = n;
    q.resample_kind = CORR2D_RESAMPLE_NONE; q.m = m;
    q.ref_mode = ref_mode; q.ref_in = ref_in; q.sigma_in = sigma_in; q.alpha = alpha;
    q.substitute = substitute_zero_var; q.norm = norm_const;
    q.pack_kind = CORR2D_PACK_F64; q.pack_roles = roles;
    q.a_phi = a_phi; q.a_psi = a_psi; q.b = b; q.ld_pack = ld_pack; q.mp = mp;
    q.ref_out = ref_out; q.sigma_out = sigma_out; q.status = acc; q.do_fft = 1;
  };
  prep(p.p1, raw1, ld_raw1, n1, ref_mode1, ref_in1, sigma_in1,
       CORR2D_ROLE_A | (homo ? CORR2D_ROLE_B : 0), ref_out1, sigma_out1, work);
  if (!homo) prep(p.p2, raw2, ld_raw2, n2, ref_mode2, ref_in2, sigma_in2, CORR2D_ROLE_B, ref_out2, sigma_out2, work + 4);
  p.homo = homo; p.n1 = n1; p.n2 = n2; p.nb1 = (n1 + 31) / 32;
  p.row0 = row0; p.row1 = row1; p.I0 = row0 / kFT; p.I1 = (row1 + kFT - 1) / kFT; p.T = (n2 + kFT - 1) / kFT;
  const long long tiles = fused_tile_count(n1, n2, homo, row0, row1);
  if (tile1 < 0 || tile1 > tiles) tile1 = tiles;
  if (tile0 < 0 || tile0 > tile1) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad tile range");
  p.tile0 = tile0; p.tiles = tile1 - tile0;
  p.a_phi = a_phi; p.a_psi = a_psi; p.b = b; p.ld_pack = ld_pack;
  p.phi = phi; p.psi = psi; p.ld_out = ld_out;
  p.vec = (ld_out % 2 == 0) && ((reinterpret_cast<uintptr_t>(phi) | reinterpret_cast<uintptr_t>(psi)) & 15) == 0;
  p.stats = stats; p.work = work; p.status1 = status1; p.status2 = homo ? nullptr : status2;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (mp / 8) {
    case 1: return launch_fused<1>(p, st);
    case 2: return launch_fused<2>(p, st);
    case 3: return launch_fused<3>(p, st);
    default: return launch_fused<4>(p, st);
  }
}
