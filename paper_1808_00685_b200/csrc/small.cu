// Small-m path (m <= 32, no resampling, fp64 operands: cfg1 m = 11, cfg2 m = 21).
//
//  * prep_small_kernel -- K1 alone (corr2d_prep): one warp per channel pair.
//  * small_block_kernel -- the whole correlation in ONE launch
//    (corr2d_correlate_small_f64): every CTA owns one 64 x 64 output block,
//    recomputes K1 for the 128 channels that block needs (one lane per
//    channel: statistics, a folded direct real DFT, the three-product Gauss
//    operand slots) into SHARED memory, contracts them on the FP64 tensor pipe
//    and stores both planes (plus the mirror of homo blocks) from registers.
//    No CTA ever waits for another: no ready flags, no grid barrier, no
//    co-residency assumption (any grid size, any SM partition).  At these sizes
//    the step is bound by launch latency, one DRAM round trip and the output
//    write (cfg1: 16 MB of planes, 2.5 us at HBM peak); the status / stat
//    words are self-resetting (the last CTA to finish publishes them).
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
// Fused small-m correlation: one launch per call, independent CTAs.
// ---------------------------------------------------------------------------
constexpr int kSB = 64;                 // output block edge (rows and columns)
constexpr int kSThreads = 128;          // 4 warps: one lane per K1 channel, 32 x 32 warp tiles
constexpr int kSMaxM = 32;

struct SmallParams {
  const void* raw1;
  const void* raw2;
  long long ld1, ld2;
  int in_f32;
  int m, n1, n2, homo;
  int ref_mode1, ref_mode2;
  const double* ref_in1;
  const double* ref_in2;
  const double* sigma_in1;
  const double* sigma_in2;
  double alpha;
  int substitute;
  double norm;
  double* ref_out1;
  double* sigma_out1;
  double* ref_out2;
  double* sigma_out2;
  int kg, ks;               // Gauss slots per segment; shared-memory row stride (doubles, = 4 mod 16)
  int T1, T2;               // 64-blocks along rows / columns
  double* phi;
  double* psi;
  long long ld_out;
  int vec;                  // planes 16-B aligned with an even ld_out: 16-byte direct stores
  int* status1;
  int* status2;
  unsigned long long* stats;
  int* work;                // kW* words, zero-filled once by the caller
};

// work-buffer words (int32 indices); every launch leaves them zero
constexpr int kWStatus1 = 0;   // [0, 4)  K1 status accumulator, dataset 1
constexpr int kWStatus2 = 4;   // [4, 8)  dataset 2
constexpr int kWDone = 8;      // CTAs finished (the last one publishes and resets)
constexpr int kWStats = 10;    // [10, 16) max|sync|, max|async|, non-finite count (3 x uint64)
constexpr int kWWords = 16;

__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Block b of the enumeration -> (row block I, column block J).  homo: the upper
// triangle J >= I, row by row (row I owns T - I blocks).
__device__ __forceinline__ void small_decode(const SmallParams& p, long long b, int& I, int& J) {
  if (!p.homo) {
    I = (int)(b / p.T2);
    J = (int)(b - (long long)I * p.T2);
    return;
  }
  const long long T = p.T1;
  const long long t2 = 2 * T + 1;
  const long long disc = t2 * t2 - 8 * b;
  long long d = (long long)((float)t2 - sqrtf((float)(disc > 0 ? disc : 0))) / 2;   // fp32 guess, exact fix-up
  auto S = [&](long long dd) { return dd * T - dd * (dd - 1) / 2; };
  if (d < 0) d = 0;
  while (d > 0 && S(d) > b) --d;
  while (S(d + 1) <= b) ++d;
  I = (int)d;
  J = I + (int)(b - S(d));
}

// K1 of one channel in one lane: the reference's statistics in its order
// (sequential sums, the IEEE operations of the other K1 kernels: bitwise-equal
// reference / sigma / values), a direct real DFT folded over t <-> m - t, then
// the CORR2D_PACK_F64_GAUSS slots of role A (row operand, x Norm x weight)
// and / or role B (column operand) into shared-memory rows.
// ys: this lane's samples at ys[t * kSThreads]; tw: cos / sin of 2 pi q / m.
__device__ __forceinline__ void tiny_k1(const SmallParams& p, int set, int c, bool valid, bool owner,
                                        double* ys, const double2* tw, double* rowA, double* rowB) {
  const int m = p.m;
  const int ref_mode = set ? p.ref_mode2 : p.ref_mode1;
  const double* ref_in = set ? p.ref_in2 : p.ref_in1;
  const double* sigma_in = set ? p.sigma_in2 : p.sigma_in1;
  int* status = p.work + (set ? kWStatus2 : kWStatus1);
  double ref = 0.0, scale = 1.0;
  int bad = 0;
  for (int t = 0; t < m; ++t) bad += !isfinite(ys[t * kSThreads]);
  if (owner && valid && bad) atomicAdd(&status[CORR2D_ST_NONFINITE], bad);
  if (ref_mode == CORR2D_REF_PROVIDED) {
    ref = valid ? __ldg(ref_in + c) : 0.0;
  } else if (ref_mode == CORR2D_REF_MEAN) {
    double sum = 0.0;                                  // left to right (numpy's axis-0 order)
    for (int t = 0; t < m; ++t) sum = __dadd_rn(sum, ys[t * kSThreads]);
    ref = __ddiv_rn(sum, (double)m);
  }
  if (p.alpha > 0.0) {
    double sigma;
    if (sigma_in) {
      sigma = valid ? __ldg(sigma_in + c) : 1.0;
    } else {
      double ss = 0.0;
      for (int t = 0; t < m; ++t) {
        const double d = __dsub_rn(ys[t * kSThreads], ref);
        ss = __dadd_rn(ss, __dmul_rn(d, d));
      }
      sigma = __dsqrt_rn(__ddiv_rn(ss, (double)(m - 1)));
    }
    if (owner && valid) {
      double* so = set ? p.sigma_out2 : p.sigma_out1;
      if (so) so[c] = sigma;
      if (sigma == 0.0) {
        atomicAdd(&status[CORR2D_ST_ZEROVAR], 1);
        atomicMax(&status[CORR2D_ST_FIRST_ZEROVAR], INT_MAX - c);
      }
    }
    if (sigma == 0.0 && p.substitute) sigma = 1.0;
    scale = (p.alpha == 0.5) ? __dsqrt_rn(sigma) : (p.alpha == 1.0 ? sigma : pow(sigma, p.alpha));
  }
  if (owner && valid) {
    double* ro = set ? p.ref_out2 : p.ref_out1;
    if (ro && ref_mode != CORR2D_REF_NONE) ro[c] = ref;
  }
  // dynamic values y_t, in place in the lane's shared-memory column; then the
  // folded pairs u_t = y_t + y_{m-t} (at t) and v_t = y_t - y_{m-t} (at m - t)
  const bool sub = ref_mode != CORR2D_REF_NONE, div = p.alpha > 0.0;
  for (int t = 0; t < m; ++t) {
    double v = ys[t * kSThreads];
    if (sub) v = __dsub_rn(v, ref);
    if (div) v = __ddiv_rn(v, scale);
    ys[t * kSThreads] = valid ? v : 0.0;
  }
  const int F = (m - 1) / 2;
  const bool even = (m % 2) == 0;
  for (int t = 1; t <= F; ++t) {
    const double a = ys[t * kSThreads], b = ys[(m - t) * kSThreads];
    ys[t * kSThreads] = a + b;
    ys[(m - t) * kSThreads] = a - b;
  }
  const double y0 = ys[0], yh = even ? ys[(m / 2) * kSThreads] : 0.0;
  const int kg = p.kg;
  const int H = m / 2;                                 // last bin (Nyquist when m is even)
  for (int w = 0; w <= H; ++w) {
    double re = y0, im = 0.0;
    int q = 0;
    for (int t = 1; t <= F; ++t) {
      q += w;
      if (q >= m) q -= m;
      const double2 cs = tw[q];
      re = fma(ys[t * kSThreads], cs.x, re);
      im = fma(-ys[(m - t) * kSThreads], cs.y, im);
    }
    if (even) re = (w & 1) ? re - yh : re + yh;
    // the Gauss slots of bin w (corr2d.h CORR2D_PACK_F64_GAUSS)
    double va, vb;
    if (w < H || !even) {                              // DC / interior: segments 0 and 1 at slot w
      gauss_values(0, w, m, p.norm, re, im, va, vb);
      if (rowA) rowA[w] = va;
      if (rowB) rowB[w] = vb;
      gauss_values(1, w, m, p.norm, re, im, va, vb);
      if (rowA) rowA[kg + w] = va;
      if (rowB) rowB[kg + w] = vb;
    }
    if (w >= 1) {                                      // interior at w - 1; Nyquist at slot F
      gauss_values(2, w, m, p.norm, re, im, va, vb);
      if (rowA) rowA[2 * kg + w - 1] = va;
      if (rowB) rowB[2 * kg + w - 1] = vb;
    }
  }
  // zero pads: segments 0 / 1 past slot F (interior F bins + DC); segment 2 past its bins
  const int used2 = even ? F + 1 : F;
  for (int j = F + 1; j < kg; ++j) {
    if (rowA) { rowA[j] = 0.0; rowA[kg + j] = 0.0; }
    if (rowB) { rowB[j] = 0.0; rowB[kg + j] = 0.0; }
  }
  for (int j = used2; j < kg; ++j) {
    if (rowA) rowA[2 * kg + j] = 0.0;
    if (rowB) rowB[2 * kg + j] = 0.0;
  }
}

// One Gauss segment of the depth (kg slots) into one accumulator set.
__device__ __forceinline__ void small_mma_seg(double (&acc)[2][4][4], const double* As, const double* Bs, int ks,
                                              int k0, int kg, int wm, int wn, int lr, int lk) {
  for (int kk = 0; kk < kg; kk += 4) {
    double ap[2][2], bf[4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r = wm * 32 + mt * 16 + lr;
      ap[mt][0] = As[r * ks + k0 + kk + lk];
      ap[mt][1] = As[(r + 8) * ks + k0 + kk + lk];
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[nt] = Bs[(wn * 32 + nt * 8 + lr) * ks + k0 + kk + lk];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], ap[mt][0], ap[mt][1], bf[nt]);
  }
}

__global__ void __launch_bounds__(kSThreads) small_block_kernel(const __grid_constant__ SmallParams p) {
  extern __shared__ __align__(16) double sm[];
  const int m = p.m, ks = p.ks;
  double2* tw = reinterpret_cast<double2*>(sm);                 // [32]
  double* ys = sm + 2 * kSMaxM;                                  // [m][kSThreads]
  double* As = ys + (size_t)m * kSThreads;                       // [64][ks]
  double* Bs = As + (size_t)kSB * ks;                            // [64][ks]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int q = tid; q < m; q += kSThreads) {
    double sv, cv;
    sincospi(2.0 * (double)q / (double)m, &sv, &cv);
    tw[q] = make_double2(cv, sv);
  }
  int I, J;
  small_decode(p, blockIdx.x, I, J);
  const bool diag = p.homo && I == J;
  // programmatic dependent launch: everything above overlapped the previous
  // kernel's tail; from here on memory written by it is visible
  asm volatile("griddepcontrol.wait;\n" ::: "memory");

  // ---- K1 for the block's channels: lanes 0..63 the 64 row channels (role A;
  //      homo diagonal blocks also role B), lanes 64..127 the 64 column
  //      channels (role B; idle on diagonal blocks) ----
  const bool col_lane = tid >= kSB;
  const int set = (col_lane && !p.homo) ? 1 : 0;
  const int c = col_lane ? J * kSB + tid - kSB : I * kSB + tid;
  const int n = set ? p.n2 : (col_lane ? p.n2 : p.n1);
  const bool active = !(diag && col_lane);
  const bool valid = c < n;
  if (active) {
    const void* raw = set ? p.raw2 : p.raw1;
    const long long ld = set ? p.ld2 : p.ld1;
    const int cc = valid ? c : n - 1;
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(ys + tid));
    if (p.in_f32) {
      const float* r = static_cast<const float*>(raw) + cc;
      for (int t = 0; t < m; ++t)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst + 8u * kSThreads * t), "l"(r + (long long)t * ld) : "memory");
    } else {
      const double* r = static_cast<const double*>(raw) + cc;
      for (int t = 0; t < m; ++t)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + 8u * kSThreads * t), "l"(r + (long long)t * ld) : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    if (p.in_f32)
      for (int t = 0; t < m; ++t) ys[t * kSThreads + tid] = (double)reinterpret_cast<const float*>(ys + t * kSThreads + tid)[0];
  }
  __syncthreads();                                  // twiddles
  if (active) {
    // the channel's statistics / status are reported by one block only: the
    // diagonal block (homo), column block 0 (dataset 1) or row block 0 (dataset 2)
    const bool owner = p.homo ? diag : (col_lane ? I == 0 : J == 0);
    double* rowA = col_lane ? nullptr : As + (size_t)tid * ks;
    double* rowB = col_lane ? Bs + (size_t)(tid - kSB) * ks : (diag ? Bs + (size_t)tid * ks : nullptr);
    tiny_k1(p, set, c, valid, owner, ys + tid, tw, rowA, rowB);
  }
  __syncthreads();

  // ---- contraction (Gauss): P1 -> sync, copy to async; -P3 -> sync, P2 -> async ----
  const int wm = warp >> 1, wn = warp & 1, lr = lane >> 2, lk = lane & 3;
  double aphi[2][4][4], apsi[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int q = 0; q < 4; ++q) aphi[a][b][q] = 0.0;
  const int kg = p.kg;
  small_mma_seg(aphi, As, Bs, ks, 0, kg, wm, wn, lr, lk);
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int q = 0; q < 4; ++q) apsi[a][b][q] = aphi[a][b][q];
  small_mma_seg(aphi, As, Bs, ks, 2 * kg, kg, wm, wn, lr, lk);
  small_mma_seg(apsi, As, Bs, ks, kg, kg, wm, wn, lr, lk);

  // ---- epilogue from registers: lane holds rows (lr, lr + 8) x columns
  //      (2 lk, 2 lk + 1) of each m16n8 tile ----
  unsigned long long mphi = 0, mpsi = 0;
  const int i0 = I * kSB + wm * 32, j0 = J * kSB + wn * 32;
  const bool mirror = p.homo && !diag;
  const bool full = p.vec && i0 + 32 <= p.n1 && j0 + 32 <= p.n2 && !diag;
  if (full) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gi = i0 + mt * 16 + lr + 8 * h, gj = j0 + nt * 8 + 2 * lk;
          const double f0 = aphi[mt][nt][2 * h], f1 = aphi[mt][nt][2 * h + 1];
          const double s0 = apsi[mt][nt][2 * h], s1 = apsi[mt][nt][2 * h + 1];
          mphi = max(mphi, max(abs_bits(f0), abs_bits(f1)));
          mpsi = max(mpsi, max(abs_bits(s0), abs_bits(s1)));
          const long long o = (long long)gi * p.ld_out + gj;
          __stcs(reinterpret_cast<double2*>(p.phi + o), make_double2(f0, f1));
          __stcs(reinterpret_cast<double2*>(p.psi + o), make_double2(s0, s1));
          if (mirror) {
            const long long om = (long long)gj * p.ld_out + gi;
            __stcs(p.phi + om, f0);
            __stcs(p.psi + om, neg_bits(s0));
            __stcs(p.phi + om + p.ld_out, f1);
            __stcs(p.psi + om + p.ld_out, neg_bits(s1));
          }
        }
  } else {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int gi = i0 + mt * 16 + lr + 8 * h, gj = j0 + nt * 8 + 2 * lk + e;
            double f = aphi[mt][nt][2 * h + e], s = apsi[mt][nt][2 * h + e];
            if (gi >= p.n1 || gj >= p.n2) continue;
            bool direct = true, mir = mirror;
            if (diag) {                      // upper part incl. the diagonal, mirrored below it
              direct = gi <= gj;
              mir = gi < gj;
              if (gi == gj) s = 0.0;
            }
            if (!direct) continue;
            mphi = max(mphi, abs_bits(f));
            mpsi = max(mpsi, abs_bits(s));
            __stcs(p.phi + (long long)gi * p.ld_out + gj, f);
            __stcs(p.psi + (long long)gi * p.ld_out + gj, s);
            if (mir) {
              __stcs(p.phi + (long long)gj * p.ld_out + gi, f);
              __stcs(p.psi + (long long)gj * p.ld_out + gi, neg_bits(s));
            }
          }
  }
  // ---- max|.| and the finite check (integer pipe), one set of atomics per CTA ----
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
  __shared__ unsigned long long red[3][4];
  if (lane == 0) {
    red[0][warp] = mphi;
    red[1][warp] = mpsi;
    red[2][warp] = (unsigned long long)bad;
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(p.work + kWStats);
    unsigned long long a0 = 0, a1 = 0, a2 = 0;
    for (int w = 0; w < kSThreads / 32; ++w) {
      a0 = max(a0, red[0][w]);
      a1 = max(a1, red[1][w]);
      a2 += red[2][w];
    }
    if (a0) atomicMax(&acc[0], a0);
    if (a1) atomicMax(&acc[1], a1);
    if (a2) atomicAdd(&acc[2], a2);
    // the last CTA to finish publishes status / stats and leaves the words zero
    // (an arrival counter, never a wait)
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
      __threadfence();
    }
  }
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

static long long small_blocks(int n1, int n2, int homo) {
  const long long T1 = (n1 + kSB - 1) / kSB, T2 = (n2 + kSB - 1) / kSB;
  return homo ? T1 * (T1 + 1) / 2 : T1 * T2;
}

}  // namespace corr2d

using namespace corr2d;

extern "C" int64_t corr2d_small_block_count(int n1, int n2, int homo) {
  if (n1 < 1 || n2 < 1 || (homo && n1 != n2)) return -1;
  return small_blocks(n1, n2, homo);
}

extern "C" int corr2d_correlate_small_f64(
    int in_dtype, const void* raw1, int64_t ld_raw1, const void* raw2, int64_t ld_raw2,
    int m, int n1, int n2,
    int ref_mode1, const double* ref_in1, const double* sigma_in1,
    int ref_mode2, const double* ref_in2, const double* sigma_in2,
    double alpha, int substitute_zero_var, double norm_const,
    double* ref_out1, double* sigma_out1, double* ref_out2, double* sigma_out2,
    double* phi, double* psi, int64_t ld_out,
    int32_t* status1, int32_t* status2, unsigned long long* stats, int32_t* work, void* stream) {
  const bool homo = raw2 == nullptr;
  if (!raw1 || !phi || !psi || !status1 || !stats || !work || (!homo && !status2))
    return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: null pointer");
  if (in_dtype != CORR2D_F64 && in_dtype != CORR2D_F32) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad dtype");
  if (m < 2 || m > kSMaxM) return fail(CORR2D_ERR_UNSUPPORTED, "corr2d_correlate_small_f64: needs 2 <= m <= 32");
  if (n1 < 1 || n2 < 1) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad sizes");
  if (homo && n1 != n2) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: homo needs n1 == n2");
  if (ld_raw1 < n1 || (!homo && ld_raw2 < n2)) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: ld_raw < n");
  if (ld_out < n2) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: ld_out < n2");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(CORR2D_ERR_DATA, "scaling exponent must lie in [0, 1]");
  for (int r : {ref_mode1, ref_mode2})
    if (r < CORR2D_REF_MEAN || r > CORR2D_REF_NONE) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad ref_mode");
  if ((ref_mode1 == CORR2D_REF_PROVIDED && !ref_in1) || (!homo && ref_mode2 == CORR2D_REF_PROVIDED && !ref_in2))
    return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: provided reference missing");

  SmallParams p{};
  p.raw1 = raw1; p.raw2 = raw2; p.ld1 = ld_raw1; p.ld2 = ld_raw2; p.in_f32 = in_dtype == CORR2D_F32;
  p.m = m; p.n1 = n1; p.n2 = n2; p.homo = homo;
  p.ref_mode1 = ref_mode1; p.ref_mode2 = ref_mode2; p.ref_in1 = ref_in1; p.ref_in2 = ref_in2;
  p.sigma_in1 = sigma_in1; p.sigma_in2 = sigma_in2; p.alpha = alpha; p.substitute = substitute_zero_var;
  p.norm = norm_const;
  p.ref_out1 = ref_out1; p.sigma_out1 = sigma_out1; p.ref_out2 = ref_out2; p.sigma_out2 = sigma_out2;
  p.kg = gauss_kg(m);
  p.ks = (3 * p.kg + 11) / 16 * 16 + 4;
  p.T1 = (n1 + kSB - 1) / kSB; p.T2 = (n2 + kSB - 1) / kSB;
  p.phi = phi; p.psi = psi; p.ld_out = ld_out;
  p.vec = (ld_out % 2 == 0) && ((reinterpret_cast<uintptr_t>(phi) | reinterpret_cast<uintptr_t>(psi)) & 15) == 0;
  p.status1 = status1; p.status2 = homo ? nullptr : status2; p.stats = stats; p.work = work;
  const long long blocks = small_blocks(n1, n2, homo);
  if (blocks > 0x7fffffffLL) return fail(CORR2D_ERR_UNSUPPORTED, "corr2d_correlate_small_f64: too many blocks");
  const size_t smem = (2 * kSMaxM + (size_t)m * kSThreads + 2 * (size_t)kSB * p.ks) * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(small_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((2 * kSMaxM + (size_t)kSMaxM * kSThreads + 2 * (size_t)kSB * 52) * sizeof(double)));
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kSThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  // programmatic dependent launch: this grid's launch and prologue overlap the
  // previous kernel's tail (griddepcontrol.wait orders memory).  No CTA waits
  // for another, so the grid needs no co-residency.
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, small_block_kernel, p);
  return check_launch("small_block_kernel");
}
