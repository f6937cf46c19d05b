// The whole small-m correlation (corr2d_correlate_small_f64): fp64,
// 2 <= m <= 32, no resampling -- the cfg1 (m = 11) and cfg2 (m = 21) shapes,
// where a step is bound by launch latency, one DRAM round trip and the output
// write (cfg1: 16 MB of planes, 2.5 us at HBM peak).  Two kernels, chained by
// programmatic dependent launch (the second grid launches while the first
// runs and waits at griddepcontrol.wait for its completion -- a kernel
// boundary, never a wait of one CTA on another):
//
// small_prep_kernel   -- K1 once per channel, one lane per channel: the
//   reference's statistics in its order (sequential sums: bitwise-equal
//   reference / sigma / values), the real DFT of each warp's 32 channels as an
//   FP64 tensor-core product Y[bins x channels] = W[bins x t] . y[t x channels]
//   (W: cos / -sin rows from a per-m host table), then the
//   CORR2D_PACK_F64_GAUSS operand rows (three real products per bin).
// small_contract_kernel -- one CTA per 64 x 64 output block (homo: the upper
//   triangle, mirrored): operand rows from L2 into shared memory, the Gauss
//   contraction on the FP64 tensor pipe with two independent accumulator
//   chains, both planes staged in shared memory and written as coalesced rows
//   plus the mirror (sync^T, -async^T), diagonal blocks symmetrised, with the
//   max|.| / finite reduction fused.  Status / stat words are self-resetting:
//   the last CTA to finish (an arrival counter, never a wait) publishes and
//   re-zeroes them.
//
// Reference path: preprocess.py:123-137, :198-259 (reference, sigma, scaling),
// fourier.py:61-82 (rfft along the perturbation axis), fourier.py:107-123
// (weighted half-spectrum cross sum x Norm, split into sync / async),
// engine_core.py:139-140 (finite check), dataset.py:159-170 (homo symmetry).
#include "prep_params.cuh"

#include <algorithm>
#include <climits>
#include <cmath>
#include <mutex>
#include <vector>

namespace corr2d {

constexpr int kSB = 64;          // output block edge (rows and columns)
#ifndef CORR2D_SMALL_MINB
#define CORR2D_SMALL_MINB 2      // contraction CTAs per SM (register budget)
#endif
constexpr int kSThreads = 128;   // 4 warps: one lane per K1 channel, 32 x 32 warp tiles
constexpr int kSMaxM = 32;
constexpr int kCS = kSB + 1;     // epilogue staging stride
constexpr int kYS = 132;         // sample rows [t][channel]: stride = 4 mod 16 doubles (conflict-free B fragments)

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
  const double* W;          // DFT rows: [3 x 16][mpad] (cos bins 0..15 | -sin bins 0..15 | cos bins 16..31)
  int mpad;                 // m rounded up to 4 (the DMMA k-step); samples past m are 0
  int yrows;                // rows of the sample / spectrum region: max(mpad, 2 (m / 2 + 1))
  int kg, ks;               // Gauss slots per segment; operand row stride (doubles, = 4 mod 16)
  int T1, T2;               // 64-blocks along rows / columns
  int nb1;                  // 128-channel K1 blocks of dataset 1 (dataset 2's follow)
  double* opsA;             // Gauss operand rows, role A (row operand), n1 x ld_ops
  double* opsB;             // role B (column operand), n2 x ld_ops (homo: n1)
  long long ld_ops;
  double* phi;
  double* psi;
  long long ld_out;
  int vec;                  // planes 16-B aligned with an even ld_out: 16-byte stores
  int* status1;
  int* status2;
  unsigned long long* stats;
  int* work;                // kW* words, zero-filled once by the caller
  unsigned long long* trace;  // profiling builds: per-CTA globaltimer stamps (NULL otherwise)
};

// work-buffer words (int32 indices); every launch leaves them zero
constexpr int kWStatus1 = 0;   // [0, 4)  K1 status accumulator, dataset 1
constexpr int kWStatus2 = 4;   // [4, 8)  dataset 2
// (K1 accumulates into them; the contraction grid's CTA 0 publishes them to
// status1 / status2 and re-zeroes them -- after K1 completed, before the next
// call's K1 starts: both grids order memory with griddepcontrol.wait)

// profiling builds (-DCORR2D_PROFILING, CORR2D_SMALL_TRACE=1): thread 0 of
// every CTA records %globaltimer at phase boundaries (K1 CTAs at slots
// [8 b, 8 b + 8), contraction CTAs at [8 (kTraceK1 + b), ...)); release
// builds compile the stamps away
constexpr int kTraceK1 = 1024;
#ifdef CORR2D_PROFILING
#define SMALL_STAMP(base, k)                                                                   \
  do {                                                                                         \
    if (p.trace && threadIdx.x == 0) {                                                         \
      unsigned long long t_;                                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
      p.trace[8 * ((base) + blockIdx.x) + (k)] = t_;                                           \
    }                                                                                          \
  } while (0)
#else
#define SMALL_STAMP(base, k) do { } while (0)
#endif

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

// Statistics and dynamic values of one channel (one lane), in place in its
// shared-memory column ys[t * kYS]: the IEEE operations of the other K1
// kernels in the reference's order.  The owner lane reports status /
// reference / sigma.
__device__ __forceinline__ void lane_stats(const SmallParams& p, int set, int c, bool valid, bool owner,
                                           double* ys) {
  const int m = p.m;
  const int ref_mode = set ? p.ref_mode2 : p.ref_mode1;
  int* status = p.work + (set ? kWStatus2 : kWStatus1);
  double ref = 0.0, scale = 1.0;
  int bad = 0;
  double sum = 0.0;                                    // left to right (numpy's axis-0 order)
#pragma unroll 4
  for (int t = 0; t < m; ++t) {
    const double v = ys[t * kYS];
    bad += !isfinite(v);
    sum = __dadd_rn(sum, v);
  }
  if (owner && valid && bad) atomicAdd(&status[CORR2D_ST_NONFINITE], bad);
  if (ref_mode == CORR2D_REF_PROVIDED) {
    ref = valid ? __ldg((set ? p.ref_in2 : p.ref_in1) + c) : 0.0;
  } else if (ref_mode == CORR2D_REF_MEAN) {
    ref = __ddiv_rn(sum, (double)m);
  }
  if (p.alpha > 0.0) {
    const double* sigma_in = set ? p.sigma_in2 : p.sigma_in1;
    double sigma;
    if (sigma_in) {
      sigma = valid ? __ldg(sigma_in + c) : 1.0;
    } else {
      double ss = 0.0;
      for (int t = 0; t < m; ++t) {
        const double d = __dsub_rn(ys[t * kYS], ref);
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
  if (owner && valid && ref_mode != CORR2D_REF_NONE) {
    double* ro = set ? p.ref_out2 : p.ref_out1;
    if (ro) ro[c] = ref;
  }
  const bool sub = ref_mode != CORR2D_REF_NONE, div = p.alpha > 0.0;
  if (!div) {
#pragma unroll 4
    for (int t = 0; t < m; ++t) {
      const double v = ys[t * kYS];
      ys[t * kYS] = valid ? (sub ? __dsub_rn(v, ref) : v) : 0.0;
    }
    return;
  }
  for (int t = 0; t < m; ++t) {
    double v = ys[t * kYS];
    if (sub) v = __dsub_rn(v, ref);
    v = __ddiv_rn(v, scale);
    ys[t * kYS] = valid ? v : 0.0;
  }
}

// The Gauss slots of bin w (spectrum R + i I) of one channel into its operand
// row(s) (corr2d.h CORR2D_PACK_F64_GAUSS).
__device__ __forceinline__ void put_bin(int w, int m, int kg, double norm, double R, double I, double* rowA,
                                        double* rowB) {
  const int H = m / 2, Iint = gauss_interior(m);
  if (w > H) return;
  double va, vb;
  if (w <= Iint) {                                     // DC / interior: segments 0 and 1 at slot w
#pragma unroll
    for (int seg = 0; seg < 2; ++seg) {
      gauss_values(seg, w, m, norm, R, I, va, vb);
      if (rowA) rowA[seg * kg + w] = va;
      if (rowB) rowB[seg * kg + w] = vb;
    }
  }
  if (w >= 1) {                                        // interior at w - 1, Nyquist at slot Iint
    gauss_values(2, w, m, norm, R, I, va, vb);
    if (rowA) rowA[2 * kg + w - 1] = va;
    if (rowB) rowB[2 * kg + w - 1] = vb;
  }
}

// One Gauss segment of the depth (kg slots) into one accumulator set.
__device__ __forceinline__ void small_mma_seg(double (&acc)[2][4][4], const double* As, const double* Bs, int ks,
                                              int k0, int kg, int wm, int wn, int lr, int lk) {
#pragma unroll 1
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

// Two Gauss segments into two accumulator sets, interleaved per k-step: 16
// independent DMMAs per warp and k-step.
__device__ __forceinline__ void small_mma_seg2(double (&acc0)[2][4][4], double (&acc1)[2][4][4], const double* As,
                                               const double* Bs, int ks, int k0, int k1, int kg, int wm, int wn,
                                               int lr, int lk) {
#pragma unroll 1
  for (int kk = 0; kk < kg; kk += 4) {
    double a0[2][2], a1[2][2], b0[4], b1[4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r = wm * 32 + mt * 16 + lr;
      a0[mt][0] = As[r * ks + k0 + kk + lk];
      a0[mt][1] = As[(r + 8) * ks + k0 + kk + lk];
      a1[mt][0] = As[r * ks + k1 + kk + lk];
      a1[mt][1] = As[(r + 8) * ks + k1 + kk + lk];
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      b0[nt] = Bs[(wn * 32 + nt * 8 + lr) * ks + k0 + kk + lk];
      b1[nt] = Bs[(wn * 32 + nt * 8 + lr) * ks + k1 + kk + lk];
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        dmma(acc0[mt][nt], a0[mt][0], a0[mt][1], b0[nt]);
        dmma(acc1[mt][nt], a1[mt][0], a1[mt][1], b1[nt]);
      }
  }
}

// ---- K1: one lane per channel, 128 channels per CTA, each channel once ----
__global__ void __launch_bounds__(kSThreads) small_prep_kernel(const __grid_constant__ SmallParams p) {
  extern __shared__ __align__(16) double sm[];
  const int m = p.m, mpad = p.mpad;
  double* ys = sm;                                   // [yrows][kYS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  const int set = (int)blockIdx.x >= p.nb1 ? 1 : 0;
  const int c = ((int)blockIdx.x - (set ? p.nb1 : 0)) * kSThreads + tid;
  const int n = set ? p.n2 : p.n1;
  const bool valid = c < n;
  // the contraction grid may launch now: it waits for this grid's completion
  // (griddepcontrol.wait) before it reads the operand rows
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  SMALL_STAMP(0, 0);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");   // inputs written by earlier kernels are visible
  SMALL_STAMP(0, 1);
  // this call's stats words start at zero (the contraction grid reduces into
  // them only after this grid completed)
  if (blockIdx.x == 0 && tid < 3) p.stats[tid] = 0ull;
  // the DFT rows and the slot table into shared memory, in flight together
  // with the samples (one DRAM round trip; the loops below then never touch
  // global memory for them)
  double* tab = ys + (size_t)p.yrows * kYS;
  {
    const int ntab = 48 * mpad + 5 * 3 * p.kg;       // even: 16-byte pieces
    for (int i = tid; 2 * i < ntab; i += kSThreads)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n"
                   ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(tab + 2 * i))), "l"(p.W + 2 * i) : "memory");
  }
  {
    const void* raw = set ? p.raw2 : p.raw1;
    const long long ld = set ? p.ld2 : p.ld1;
    const int cc = valid ? c : n - 1;
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(ys + tid));
    if (p.in_f32) {
      const float* r = static_cast<const float*>(raw) + cc;
      for (int t = 0; t < m; ++t)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst + 8u * kYS * t), "l"(r + (long long)t * ld) : "memory");
    } else {
      const double* r = static_cast<const double*>(raw) + cc;
      for (int t = 0; t < m; ++t)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + 8u * kYS * t), "l"(r + (long long)t * ld) : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    if (p.in_f32)
      for (int t = 0; t < m; ++t) ys[t * kYS + tid] = (double)reinterpret_cast<const float*>(ys + t * kYS + tid)[0];
    for (int t = m; t < mpad; ++t) ys[t * kYS + tid] = 0.0;
    SMALL_STAMP(0, 2);
    lane_stats(p, set, c, valid, true, ys + tid);
  }
  __syncthreads();                                   // every thread's table pieces have landed
  SMALL_STAMP(0, 3);
  // DFT of this warp's 32 channels on the FP64 tensor pipe: Y[16 bins x 8
  // channels] tiles = W rows . y, k over t
  const int nt3 = m / 2 >= 16 ? 3 : 2;               // bins 16.. only for m = 32
  double acc[3][4][4];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[a][b][q] = 0.0;
  double* yw = ys + warp * 32;
  for (int kk = 0; kk < mpad; kk += 4) {
    double bf[4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[nt] = yw[(kk + lk) * kYS + nt * 8 + lr];
#pragma unroll
    for (int tl = 0; tl < 3; ++tl) {
      if (tl == 2 && nt3 < 3) break;
      const double a0 = tab[(tl * 16 + lr) * mpad + kk + lk];
      const double a1 = tab[(tl * 16 + lr + 8) * mpad + kk + lk];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma(acc[tl][nt], a0, a1, bf[nt]);
    }
  }
  SMALL_STAMP(0, 4);
  // the spectra back into the warp's own sample columns (bin w: Re in row 2 w,
  // Im in row 2 w + 1), then each lane writes its channel's operand row(s)
  __syncwarp();                                      // the warp's DMMAs have read its columns
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = nt * 8 + 2 * lk + e, w = lr + 8 * h;
        if (w > m / 2) continue;                       // rows past 2 H + 1 are not part of the region
        yw[(2 * w) * kYS + col] = acc[0][nt][2 * h + e];
        yw[(2 * w + 1) * kYS + col] = acc[1][nt][2 * h + e];
        if (nt3 == 3 && h == 0 && lr == 0) {
          yw[32 * kYS + col] = acc[2][nt][e];          // bin 16 (m = 32: Nyquist, real)
          yw[33 * kYS + col] = 0.0;
        }
      }
  __syncwarp();
  // every slot once (pads are 0), from the per-slot table after W: bin w and
  // small exact coefficients -- A = Norm (pa R + qa I), B = pb R + qb I
  // (gauss_values' operands: a + b, a, -b | a at Nyquist; c, d - c, c + d).
  // The rows are staged per warp in shared memory in their global layout
  // (ld_ops = 3 kg: the warp's 32 rows are one contiguous run), then leave as
  // coalesced 16-byte stores.
  const int ns = 3 * p.kg;
  // the warp's 32 rows staged in their global layout (ld_ops = ns: ONE
  // contiguous run), then one bulk copy per role
  double* stA = tab + 48 * mpad + 5 * ns + (size_t)warp * 32 * ns;   // [32][ns] per warp
  double* stB = stA + (size_t)kSThreads * ns;
  const bool wantA = !set, wantB = set || p.homo;
  {
    // pads are zero: the warp zeroes its run with consecutive 16-B stores
    double2* zA = reinterpret_cast<double2*>(stA);
    double2* zB = reinterpret_cast<double2*>(stB);
    for (int i = lane; i < 16 * ns; i += 32) zA[i] = zB[i] = make_double2(0.0, 0.0);
    __syncwarp();
    // every bin's three Gauss slots from registers.  Lane l takes the bins in
    // the rotated order w = (it + l) mod (H + 1), so the 32 lanes' rows (pitch
    // ns) are written at different slots: few bank conflicts
    const int kg = p.kg, H = m / 2, Iint = gauss_interior(m);
    const double nrm = p.norm;
    double* a = stA + lane * ns;
    double* b = stB + lane * ns;
    int w = lane % (H + 1);
    // a runtime loop: straight-line code is fetched cold, line by line, on
    // every step of a stream that evicts L2 (the bench's rotation does)
#pragma unroll 1
    for (int it = 0; it <= H; ++it, w = (w == H) ? 0 : w + 1) {
      const double R = ys[(2 * w) * kYS + tid];
      const double I = (w == 0 || 2 * w == m) ? 0.0 : ys[(2 * w + 1) * kYS + tid];
      const double k = (w == 0 || 2 * w == m) ? 1.0 : 2.0;
      const double ra = nrm * (k * R), ia = nrm * (k * I);    // a, b (x 2 exact)
      if (w <= Iint) {                               // DC / interior: segments 0 and 1 at slot w
        a[w] = ra + ia;      b[w] = R;               // a + b, c
        a[kg + w] = ra;      b[kg + w] = -I - R;     // a, d - c
      }
      if (w >= 1) {
        if (w <= Iint) { a[2 * kg + w - 1] = -ia; b[2 * kg + w - 1] = R - I; }   // -b, c + d
        else { a[2 * kg + Iint] = ra; b[2 * kg + Iint] = R; }                     // Nyquist: a, c
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic-proxy writes -> bulk copy
  __syncwarp();
  SMALL_STAMP(0, 7);
  {
    const int cw = c - lane;                         // the warp's first channel
    const int nrow = min(32, n - cw);
    if (nrow > 0 && lane == 0) {
      const unsigned bytes = (unsigned)(nrow * ns) * 8u;
      if (wantA)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                     ::"l"(p.opsA + (long long)cw * p.ld_ops),
                       "r"(static_cast<unsigned>(__cvta_generic_to_shared(stA))), "r"(bytes) : "memory");
      if (wantB)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                     ::"l"(p.opsB + (long long)cw * p.ld_ops),
                       "r"(static_cast<unsigned>(__cvta_generic_to_shared(stB))), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;\n" ::: "memory");
    }
  }
  SMALL_STAMP(0, 5);
}

__device__ __noinline__ void small_publish(const SmallParams& p, unsigned long long mphi, unsigned long long mpsi,
                                           int lane, int warp, int tid);

// ---- contraction: one CTA per 64 x 64 output block ----
__global__ void __launch_bounds__(kSThreads, CORR2D_SMALL_MINB) small_contract_kernel(const __grid_constant__ SmallParams p) {
  extern __shared__ __align__(16) double sm[];
  const int ks = p.ks, kg = p.kg;
  double* As = sm;                                   // [64][ks]
  double* Bs = As + (size_t)kSB * ks;                // [64][ks]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  int I, J;
  small_decode(p, blockIdx.x, I, J);
  const bool diag = p.homo && I == J;
  __shared__ __align__(8) unsigned long long bar;
  const unsigned bar_s = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
  const int rows_a = min(kSB, p.n1 - I * kSB), rows_b = min(kSB, p.n2 - J * kSB);
  const unsigned row_bytes = 3u * kg * 8u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_s) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  SMALL_STAMP(kTraceK1, 0);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");   // K1 complete, its operand rows visible
  SMALL_STAMP(kTraceK1, 1);
  // K1's status accumulators are final now: CTA 0 publishes them and leaves
  // the words zero for the next call (whose K1 starts after this grid ends)
  if (blockIdx.x == 0 && tid < 4) {
    p.status1[tid] = p.work[kWStatus1 + tid];
    p.work[kWStatus1 + tid] = 0;
    if (p.status2) p.status2[tid] = p.work[kWStatus2 + tid];
    p.work[kWStatus2 + tid] = 0;
  }
  // one bulk copy per operand row (thread t: A row t or B row t - 64), all
  // completing on one mbarrier; rows past the map are zero-filled
  if (tid == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                 ::"r"(bar_s), "r"((unsigned)(rows_a + rows_b) * row_bytes) : "memory");
  __syncthreads();                                   // expect_tx before any complete_tx
  {
    const bool is_b = tid >= kSB;
    const int r = is_b ? tid - kSB : tid;
    double* dst = (is_b ? Bs : As) + r * ks;
    if (r < (is_b ? rows_b : rows_a)) {
      const double* src = (is_b ? p.opsB : p.opsA) + (long long)((is_b ? J : I) * kSB + r) * p.ld_ops;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))), "l"(src), "r"(row_bytes), "r"(bar_s)
                   : "memory");
    } else {
      for (int s = 0; s < 3 * kg; ++s) dst[s] = 0.0;
    }
  }
  {
    unsigned done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(bar_s) : "memory");
  }
  __syncthreads();                                   // zero-filled rows visible
  SMALL_STAMP(kTraceK1, 2);
  // Gauss: P1 (segment 0) and -P3 (segment 2) as two independent chains, then
  // sync = P1 - P3 and async = P1 + P2 (segment 1)
  const int wm = warp >> 1, wn = warp & 1;
  double aphi[2][4][4], apsi[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int q = 0; q < 4; ++q) aphi[a][b][q] = apsi[a][b][q] = 0.0;
  small_mma_seg2(apsi, aphi, As, Bs, ks, 0, 2 * kg, kg, wm, wn, lr, lk);
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int q = 0; q < 4; ++q) aphi[a][b][q] += apsi[a][b][q];
  small_mma_seg(apsi, As, Bs, ks, kg, kg, wm, wn, lr, lk);
  __syncthreads();                                   // operands consumed: the staging overlays them
  SMALL_STAMP(kTraceK1, 3);

  const int i0 = I * kSB, j0 = J * kSB;
  // ---- 5. stage both planes, then coalesced row stores (+ mirror), with
  //      max|.| / the finite check folded into the stores' smem reads ----
  double* Cphi = sm;                                 // [64][kCS]
  double* Cpsi = sm + kSB * kCS;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = wm * 32 + mt * 16 + lr + 8 * h, cl = wn * 32 + nt * 8 + 2 * lk;
        Cphi[r * kCS + cl] = aphi[mt][nt][2 * h];
        Cphi[r * kCS + cl + 1] = aphi[mt][nt][2 * h + 1];
        Cpsi[r * kCS + cl] = apsi[mt][nt][2 * h];
        Cpsi[r * kCS + cl + 1] = apsi[mt][nt][2 * h + 1];
      }
  __syncthreads();
  unsigned long long mphi = 0, mpsi = 0;
  const bool rows_full = i0 + kSB <= p.n1, cols_full = j0 + kSB <= p.n2;
  if (!diag && rows_full && cols_full && p.vec) {
    // whole off-diagonal block: a thread owns one column pair of rows
    // r0, r0 + 4, ... (and of the mirror block) -- pointer steps only
    const int cp = (tid & 31) * 2, r0 = tid >> 5;
    const long long step = 4 * p.ld_out;
    const double* cph = Cphi + r0 * kCS + cp;
    const double* cps = Cpsi + r0 * kCS + cp;
    double* dph = p.phi + (long long)(i0 + r0) * p.ld_out + j0 + cp;
    double* dps = p.psi + (dph - p.phi);
#pragma unroll 4
    for (int k = 0; k < kSB / 4; ++k) {
      const double f0 = cph[0], f1 = cph[1], s0 = cps[0], s1 = cps[1];
      mphi = max(mphi, max(abs_bits(f0), abs_bits(f1)));
      mpsi = max(mpsi, max(abs_bits(s0), abs_bits(s1)));
      __stcs(reinterpret_cast<double2*>(dph), make_double2(f0, f1));
      __stcs(reinterpret_cast<double2*>(dps), make_double2(s0, s1));
      cph += 4 * kCS; cps += 4 * kCS; dph += step; dps += step;
    }
    if (p.homo) {     // mirror rows j0 + r (C column r), columns i0 + cp, +1 (C rows)
      const double* mph = Cphi + cp * kCS + r0;
      const double* mps = Cpsi + cp * kCS + r0;
      double* eph = p.phi + (long long)(j0 + r0) * p.ld_out + i0 + cp;
      double* eps = p.psi + (eph - p.phi);
#pragma unroll 4
      for (int k = 0; k < kSB / 4; ++k) {
        __stcs(reinterpret_cast<double2*>(eph), make_double2(mph[0], mph[kCS]));
        __stcs(reinterpret_cast<double2*>(eps), make_double2(neg_bits(mps[0]), neg_bits(mps[kCS])));
        mph += 4; mps += 4; eph += step; eps += step;
      }
    }
  } else {
  // direct block: rows i0.., a thread stores column pairs (32 pairs per row)
  for (int idx = tid; idx < kSB * (kSB / 2); idx += kSThreads) {
    const int r = idx >> 5, cp = (idx & 31) * 2;
    const int gi = i0 + r, gj = j0 + cp;
    if (gi >= p.n1 || gj >= p.n2) continue;
    double f0, f1, s0, s1;
    if (diag) {          // upper triangle incl. the diagonal; below it the mirror of the upper
      f0 = r <= cp ? Cphi[r * kCS + cp] : Cphi[cp * kCS + r];
      f1 = r <= cp + 1 ? Cphi[r * kCS + cp + 1] : Cphi[(cp + 1) * kCS + r];
      s0 = r < cp ? Cpsi[r * kCS + cp] : (r == cp ? 0.0 : neg_bits(Cpsi[cp * kCS + r]));
      s1 = r < cp + 1 ? Cpsi[r * kCS + cp + 1] : (r == cp + 1 ? 0.0 : neg_bits(Cpsi[(cp + 1) * kCS + r]));
    } else {
      f0 = Cphi[r * kCS + cp]; f1 = Cphi[r * kCS + cp + 1];
      s0 = Cpsi[r * kCS + cp]; s1 = Cpsi[r * kCS + cp + 1];
    }
    mphi = max(mphi, abs_bits(f0));
    mpsi = max(mpsi, abs_bits(s0));
    const long long o = (long long)gi * p.ld_out + gj;
    if (gj + 1 < p.n2) {
      mphi = max(mphi, abs_bits(f1));
      mpsi = max(mpsi, abs_bits(s1));
      if (p.vec) {
        __stcs(reinterpret_cast<double2*>(p.phi + o), make_double2(f0, f1));
        __stcs(reinterpret_cast<double2*>(p.psi + o), make_double2(s0, s1));
        continue;
      }
      __stcs(p.phi + o + 1, f1);
      __stcs(p.psi + o + 1, s1);
    }
    __stcs(p.phi + o, f0);
    __stcs(p.psi + o, s0);
  }
  // mirror block of a homo block above the diagonal: rows j0.., columns i0..
  if (p.homo && !diag) {
    for (int idx = tid; idx < kSB * (kSB / 2); idx += kSThreads) {
      const int r = idx >> 5, cp = (idx & 31) * 2;        // mirror row r (= C column), columns cp, cp + 1 (= C rows)
      const int gi = j0 + r, gj = i0 + cp;
      if ((!cols_full && gi >= p.n2) || gj >= p.n1) continue;
      const double f0 = Cphi[cp * kCS + r], f1 = Cphi[(cp + 1) * kCS + r];
      const double s0 = neg_bits(Cpsi[cp * kCS + r]), s1 = neg_bits(Cpsi[(cp + 1) * kCS + r]);
      const long long o = (long long)gi * p.ld_out + gj;
      if (p.vec && (rows_full || gj + 1 < p.n1)) {
        __stcs(reinterpret_cast<double2*>(p.phi + o), make_double2(f0, f1));
        __stcs(reinterpret_cast<double2*>(p.psi + o), make_double2(s0, s1));
      } else {
        __stcs(p.phi + o, f0);
        __stcs(p.psi + o, s0);
        if (gj + 1 < p.n1) {
          __stcs(p.phi + o + 1, f1);
          __stcs(p.psi + o + 1, s1);
        }
      }
    }
  }
  }  // general blocks
  SMALL_STAMP(kTraceK1, 4);
  // ---- 6. one set of fire-and-forget reductions per CTA (no fence, no wait) ----
  small_publish(p, mphi, mpsi, lane, warp, tid);
  SMALL_STAMP(kTraceK1, 5);
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// One set of atomics per CTA into the work words; the last CTA to arrive (an
// arrival counter, never a wait) publishes status / stats and re-zeroes them.
__device__ __noinline__ void small_publish(const SmallParams& p, unsigned long long mphi, unsigned long long mpsi,
                                           int lane, int warp, int tid) {
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
    // fire-and-forget reductions straight into the caller's stats words
    // (zeroed by this call's K1 grid, which completed before this grid began)
    unsigned long long a0 = 0, a1 = 0, a2 = 0;
    for (int w = 0; w < kSThreads / 32; ++w) {
      a0 = max(a0, red[0][w]);
      a1 = max(a1, red[1][w]);
      a2 += red[2][w];
    }
    if (a0) atomicMax(&p.stats[0], a0);
    if (a1) atomicMax(&p.stats[1], a1);
    if (a2) atomicAdd(&p.stats[2], a2);
  }
}

static long long small_blocks(int n1, int n2, int homo) {
  const long long T1 = (n1 + kSB - 1) / kSB, T2 = (n2 + kSB - 1) / kSB;
  return homo ? T1 * (T1 + 1) / 2 : T1 * T2;
}

// Per-(device, m) DFT row table W in device memory, built once on the host in
// double precision: row 16 k + r, column t < m holds cos(2 pi w t / m) for
// k = 0 (bins w = r), -sin(2 pi w t / m) for k = 1 (w = r), cos for k = 2
// (w = 16 + r); bins past m / 2 and columns past m are zero.
static const double* dft_table(int m, int mpad, cudaStream_t st, int* rc) {
  constexpr int kDev = 64;
  static double* tab[kDev][kSMaxM + 1] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kDev) {
    *rc = fail(CORR2D_ERR_UNSUPPORTED, "corr2d_correlate_small_f64: device index >= 64");
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (tab[dev][m]) return tab[dev][m];
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs != cudaStreamCaptureStatusNone) {
    *rc = fail(CORR2D_ERR_UNSUPPORTED,
               "corr2d_correlate_small_f64: the first call for this m on this device must not be graph-captured");
    return nullptr;
  }
  const int kg = gauss_kg(m), ns = 3 * kg;
  std::vector<double> h((size_t)48 * mpad + 5 * (size_t)ns, 0.0);
  const double two_pi = 6.283185307179586476925286766559;
  for (int k = 0; k < 3; ++k)
    for (int r = 0; r < 16; ++r) {
      const int w = (k == 2 ? 16 : 0) + r;
      if (w > m / 2) continue;
      for (int t = 0; t < m; ++t) {
        const int q = (w * t) % m;
        const double ang = two_pi * (double)q / (double)m;
        // exact zeros of sin at 0 and pi (DC / Nyquist rows are real)
        const double sn = (q == 0 || 2 * q == m) ? 0.0 : std::sin(ang);
        h[(size_t)(16 * k + r) * mpad + t] = k == 1 ? -sn : std::cos(ang);
      }
    }
  // per-slot table of the CORR2D_PACK_F64_GAUSS rows (corr2d.h; gauss_values):
  // bin w, then A = Norm (pa R + qa I) and B = pb R + qb I, with a = k R,
  // b = k I (k = 2, or 1 at DC / Nyquist where I = 0), c = R, d = -I
  double* slot = h.data() + (size_t)48 * mpad;
  for (int s = 0; s < ns; ++s, slot += 5) {
    const int seg = s / kg, j = s - seg * kg, w = gauss_bin(seg, j, m);
    slot[0] = w;
    if (w < 0) continue;
    const bool edge = w == 0 || (m % 2 == 0 && w == m / 2);
    const double kk = edge ? 1.0 : 2.0, ki = edge ? 0.0 : 1.0;
    double pa, qa, pb, qb;
    if (seg == 0) { pa = kk; qa = kk * ki; pb = 1.0; qb = 0.0; }          // a + b, c
    else if (seg == 1) { pa = kk; qa = 0.0; pb = -1.0; qb = -ki; }        // a, d - c
    else if (edge) { pa = kk; qa = 0.0; pb = 1.0; qb = 0.0; }             // Nyquist: a, c
    else { pa = 0.0; qa = -kk; pb = 1.0; qb = -1.0; }                     // -b, c + d
    slot[1] = pa; slot[2] = qa; slot[3] = pb; slot[4] = qb;
  }
  double* d = nullptr;
  if (cudaMalloc(&d, h.size() * sizeof(double)) != cudaSuccess ||
      cudaMemcpy(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
    *rc = check_launch("small DFT table");
    return nullptr;
  }
  tab[dev][m] = d;
  return d;
}

}  // namespace corr2d

using namespace corr2d;

extern "C" int64_t corr2d_small_block_count(int n1, int n2, int homo) {
  if (n1 < 1 || n2 < 1 || (homo && n1 != n2)) return -1;
  return small_blocks(n1, n2, homo);
}

extern "C" int corr2d_small_ops_depth(int m) { return (m >= 2 && m <= kSMaxM) ? 3 * gauss_kg(m) : -1; }

extern "C" int corr2d_correlate_small_f64(
    int in_dtype, const void* raw1, int64_t ld_raw1, const void* raw2, int64_t ld_raw2,
    int m, int n1, int n2,
    int ref_mode1, const double* ref_in1, const double* sigma_in1,
    int ref_mode2, const double* ref_in2, const double* sigma_in2,
    double alpha, int substitute_zero_var, double norm_const,
    double* ops_a, double* ops_b, int64_t ld_ops,
    double* ref_out1, double* sigma_out1, double* ref_out2, double* sigma_out2,
    double* phi, double* psi, int64_t ld_out,
    int32_t* status1, int32_t* status2, unsigned long long* stats, int32_t* work, void* stream) {
  const bool homo = raw2 == nullptr;
  if (!raw1 || !ops_a || !ops_b || !phi || !psi || !status1 || !stats || !work || (!homo && !status2))
    return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: null pointer");
  if (in_dtype != CORR2D_F64 && in_dtype != CORR2D_F32) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad dtype");
  if (m < 2 || m > kSMaxM) return fail(CORR2D_ERR_UNSUPPORTED, "corr2d_correlate_small_f64: needs 2 <= m <= 32");
  if (n1 < 1 || n2 < 1) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad sizes");
  if (homo && n1 != n2) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: homo needs n1 == n2");
  if (ld_raw1 < n1 || (!homo && ld_raw2 < n2)) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: ld_raw < n");
  if (ld_out < n2) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: ld_out < n2");
  if (ld_ops != corr2d_small_ops_depth(m) ||
      ((reinterpret_cast<uintptr_t>(ops_a) | reinterpret_cast<uintptr_t>(ops_b)) & 15))
    return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: operand rows must be 16-B aligned with "
                                 "ld_ops == corr2d_small_ops_depth(m)");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(CORR2D_ERR_DATA, "scaling exponent must lie in [0, 1]");
  for (int r : {ref_mode1, ref_mode2})
    if (r < CORR2D_REF_MEAN || r > CORR2D_REF_NONE) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad ref_mode");
  if ((ref_mode1 == CORR2D_REF_PROVIDED && !ref_in1) || (!homo && ref_mode2 == CORR2D_REF_PROVIDED && !ref_in2))
    return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: provided reference missing");
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  SmallParams p{};
  p.raw1 = raw1; p.raw2 = raw2; p.ld1 = ld_raw1; p.ld2 = ld_raw2; p.in_f32 = in_dtype == CORR2D_F32;
  p.m = m; p.n1 = n1; p.n2 = n2; p.homo = homo;
  p.ref_mode1 = ref_mode1; p.ref_mode2 = ref_mode2; p.ref_in1 = ref_in1; p.ref_in2 = ref_in2;
  p.sigma_in1 = sigma_in1; p.sigma_in2 = sigma_in2; p.alpha = alpha; p.substitute = substitute_zero_var;
  p.norm = norm_const;
  p.ref_out1 = ref_out1; p.sigma_out1 = sigma_out1; p.ref_out2 = ref_out2; p.sigma_out2 = sigma_out2;
  p.mpad = (m + 3) / 4 * 4;
  p.yrows = p.mpad > 2 * (m / 2 + 1) ? p.mpad : 2 * (m / 2 + 1);
  int rc = CORR2D_OK;
  p.W = dft_table(m, p.mpad, st, &rc);
  if (!p.W) return rc;
  p.kg = gauss_kg(m);
  p.ks = (3 * p.kg + 11) / 16 * 16 + 4;
  p.T1 = (n1 + kSB - 1) / kSB; p.T2 = (n2 + kSB - 1) / kSB;
  p.nb1 = (n1 + kSThreads - 1) / kSThreads;
  p.opsA = ops_a; p.opsB = ops_b; p.ld_ops = ld_ops;
  p.phi = phi; p.psi = psi; p.ld_out = ld_out;
  p.vec = (ld_out % 2 == 0) && ((reinterpret_cast<uintptr_t>(phi) | reinterpret_cast<uintptr_t>(psi)) & 15) == 0;
  p.status1 = status1; p.status2 = homo ? nullptr : status2; p.stats = stats; p.work = work;
#ifdef CORR2D_PROFILING
  if (const char* e = getenv("CORR2D_SMALL_TRACE"))
    if (e[0] == '1') {
      static unsigned long long* tbuf = nullptr;
      const size_t words = 8 * (size_t)(kTraceK1 + 65536);
      if (!tbuf) cudaMalloc(&tbuf, words * 8);
      cudaMemsetAsync(tbuf, 0, words * 8, st);
      p.trace = tbuf;
    }
#endif
  const long long blocks = small_blocks(n1, n2, homo);
  if (blocks > 0x7fffffffLL) return fail(CORR2D_ERR_UNSUPPORTED, "corr2d_correlate_small_f64: too many blocks");
  const int prep_blocks = p.nb1 + (homo ? 0 : (n2 + kSThreads - 1) / kSThreads);
  const size_t prep_smem = ((size_t)p.yrows * kYS + 48 * (size_t)p.mpad + 15 * (size_t)p.kg +
                            2 * (size_t)kSThreads * 3 * p.kg) * sizeof(double);
  const size_t ops = 2 * (size_t)kSB * p.ks * sizeof(double);
  const size_t stage = 2 * (size_t)kSB * kCS * sizeof(double);
  const size_t smem = ops > stage ? ops : stage;
  static bool attr_set = false;
  if (!attr_set) {
    const size_t worst_ops = 2 * (size_t)kSB * 52 * sizeof(double);
    cudaFuncSetAttribute(small_contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(worst_ops > stage ? worst_ops : stage));
    cudaFuncSetAttribute(small_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(((size_t)(kSMaxM + 2) * kYS + 48 * kSMaxM + 15 * 16 + 2 * kSThreads * 48) *
                               sizeof(double)));   // m = 32: kg = 16
    attr_set = true;
  }
  // programmatic dependent launch for both grids: each launches while its
  // predecessor drains and orders memory with griddepcontrol.wait -- a kernel
  // boundary, so no grid needs co-residency
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kSThreads);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)prep_blocks);
  cfg.dynamicSmemBytes = prep_smem;
  cudaLaunchKernelEx(&cfg, small_prep_kernel, p);
  if (int e = check_launch("small_prep_kernel")) return e;
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchKernelEx(&cfg, small_contract_kernel, p);
  int code = check_launch("small_contract_kernel");
#ifdef CORR2D_PROFILING
  if (p.trace) {       // per-phase timeline (ns after the first K1 stamp): min / median / max over CTAs
    std::vector<unsigned long long> h(8 * (size_t)(kTraceK1 + blocks));
    cudaMemcpyAsync(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < prep_blocks; ++b) t0 = std::min(t0, h[8 * b]);
    auto row = [&](const char* name, int base, int nb, int k) {
      std::vector<double> v;
      for (int b = 0; b < nb; ++b)
        if (h[8 * (base + b) + k]) v.push_back((double)(h[8 * (base + b) + k] - t0));
      if (v.empty()) return;
      std::sort(v.begin(), v.end());
      fprintf(stderr, "  %-22s min %8.0f  med %8.0f  max %8.0f ns\n", name, v.front(), v[v.size() / 2], v.back());
    };
    fprintf(stderr, "small path trace (m %d, %d x %d, %s):\n", m, n1, n2, homo ? "homo" : "hetero");
    const char* k1n[8] = {"K1 start", "K1 after wait", "K1 samples in", "K1 stats done", "K1 dft done",
                          "K1 rows written", "", "K1 slots staged"};
    const char* k2n[6] = {"K2 start", "K2 after wait", "K2 operands in", "K2 mma done", "K2 stores issued", "K2 end"};
    for (int k : {0, 1, 2, 3, 4, 7, 5}) row(k1n[k], 0, prep_blocks, k);
    for (int k = 0; k < 6; ++k) row(k2n[k], kTraceK1, (int)blocks, k);
  }
#endif
  return code;
}
