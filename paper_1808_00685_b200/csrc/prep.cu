// K1 -- fused preprocessing + perturbation-axis DFT + operand packing.
//
// Reference path restated here (files under /root/reference/pkg/src/corrtwo/):
//   resample_equidistant / resample_to_axis / _interp_linear  preprocess.py:147-195
//   mean_reference / ReferenceSpec.resolve / dynamic_spectra  preprocess.py:56-64,123-137
//   stddev_spectrum                                           preprocess.py:198-211
//   apply_scaling (sigma**alpha, zero-variance policy)        preprocess.py:214-259
//   dft_channels (scipy.fft.rfft along axis 0)                fourier.py:61-82
//   half_spectrum_weights, weighted1 = half1.T * w, x Norm    fourier.py:50-58,107,121
//
// Every step is local to one spectral channel (a column of the m x n matrix),
// so one CTA owns a tile of C consecutive channels: the raw m_in x C block is
// read once with coalesced row segments, everything else happens in shared
// memory, and the packed operand rows are written once.  The elementwise
// arithmetic uses explicit round-to-nearest intrinsics (no FMA contraction) and
// the reference's summation order (sequential over the perturbation axis, as
// numpy's axis-0 reduction), so values / reference / sigma reproduce the
// reference bit-for-bit; the FFT is a mixed-radix Stockham transform.
#include "prep_params.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

namespace corr2d {

constexpr int kPrepThreads = 256;
constexpr int kSeqStatsMax = 128;  // longest axis summed strictly left to right


__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }   // a * (-i)

__device__ __forceinline__ void store_pack(const PrepParams&, void* base, long long idx, double v) {
  static_cast<double*>(base)[idx] = v;   // CORR2D_PACK_F64 (bf16 packing is vectorised below)
}

// In-register forward DFTs of length 2, 4, 8 (natural order in and out).
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  const double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 t0 = cadd(x0, x2), t1 = csub(x0, x2), t2 = cadd(x1, x3), t3 = mul_mi(csub(x1, x3));
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}
template <int R> __device__ __forceinline__ void dft_r(double2 (&x)[R]);
template <> __device__ __forceinline__ void dft_r<2>(double2 (&x)[2]) { dft2(x[0], x[1]); }
template <> __device__ __forceinline__ void dft_r<4>(double2 (&x)[4]) { dft4(x[0], x[1], x[2], x[3]); }
template <> __device__ __forceinline__ void dft_r<8>(double2 (&x)[8]) {
  constexpr double h = 0.70710678118654752440;  // sqrt(1/2)
  dft4(x[0], x[2], x[4], x[6]);                   // evens E0..E3 in x0,x2,x4,x6
  dft4(x[1], x[3], x[5], x[7]);                   // odds  O0..O3 in x1,x3,x5,x7
  const double2 o1 = make_double2(h * (x[3].x + x[3].y), h * (x[3].y - x[3].x));     // W8^1 O1
  const double2 o2 = mul_mi(x[5]);                                                  // W8^2 O2
  const double2 o3 = make_double2(h * (x[7].y - x[7].x), -h * (x[7].x + x[7].y));    // W8^3 O3
  const double2 e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6], o0 = x[1];
  x[0] = cadd(e0, o0); x[4] = csub(e0, o0);
  x[1] = cadd(e1, o1); x[5] = csub(e1, o1);
  x[2] = cadd(e2, o2); x[6] = csub(e2, o2);
  x[3] = cadd(e3, o3); x[7] = csub(e3, o3);
}

// One Stockham stage of radix R over CH interleaved columns (pairs of channels).
//   output (j, u) = sum_t in[j + t m/R] W_m^{t k span} W_R^{t u},  k = j mod Ns
// NORM (first stage only): the loaded values are (v - ref) / scale of their
// channel -- the same two IEEE operations as the separate normalisation pass,
// so the results are identical; cst = [C refs | C scales].
template <int R, bool NORM = false>
__device__ __forceinline__ void stage_r(const double2* __restrict__ in, double2* __restrict__ out,
                                        const double2* __restrict__ tw, int m, int Ns, int CH, int CPc,
                                        const double* __restrict__ cst = nullptr, int C = 0, bool sub = false,
                                        bool scaled = false) {
  const int stride = m / R, span = m / (Ns * R);
  const int chs = 31 - __clz(CH);  // CH is a power of two
  for (int idx = threadIdx.x; idx < stride * CH; idx += blockDim.x) {
    const int pc = idx & (CH - 1), j = idx >> chs, k = j % Ns;
    double2 x[R];
#pragma unroll
    for (int t = 0; t < R; ++t) x[t] = in[(j + t * stride) * CPc + pc];
    if (NORM) {
      const double r0 = cst[2 * pc], r1 = cst[2 * pc + 1], s0 = cst[C + 2 * pc], s1 = cst[C + 2 * pc + 1];
#pragma unroll
      for (int t = 0; t < R; ++t) {
        if (sub) { x[t].x = __dsub_rn(x[t].x, r0); x[t].y = __dsub_rn(x[t].y, r1); }
        if (scaled) { x[t].x = __ddiv_rn(x[t].x, s0); x[t].y = __ddiv_rn(x[t].y, s1); }
      }
    }
    if (k) {
#pragma unroll
      for (int t = 1; t < R; ++t) x[t] = cmul(x[t], tw[t * k * span]);
    }
    dft_r<R>(x);
    const int base = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int u = 0; u < R; ++u) out[(base + u * Ns) * CPc + pc] = x[u];
  }
}

// Any other radix (3, 5, 7, 11, ... and large primes): one output per item.
__device__ __forceinline__ void stage_generic(const double2* __restrict__ in, double2* __restrict__ out,
                                              const double2* __restrict__ tw, int m, int r, int Ns, int CH, int CPc) {
  const int stride = m / r, span = m / (Ns * r);
  for (int idx = threadIdx.x; idx < m * CH; idx += blockDim.x) {
    const int pc = idx % CH, rest = idx / CH;
    const int u = rest % r, j = rest / r, k = j % Ns;
    const int e = span * (k + u * Ns);
    double2 acc = make_double2(0.0, 0.0);
    int q = 0;
    for (int t = 0; t < r; ++t) {
      const double2 x = in[(j + t * stride) * CPc + pc], w = tw[q];
      acc.x = fma(x.x, w.x, fma(-x.y, w.y, acc.x));
      acc.y = fma(x.x, w.y, fma(x.y, w.x, acc.y));
      q += e;
      if (q >= m) q -= m;
    }
    out[((j / Ns) * Ns * r + k + u * Ns) * CPc + pc] = acc;
  }
}

// Spectrum of channel c at bin w from the paired transform Z = FFT(x_even + i x_odd).
__device__ __forceinline__ double2 channel_bin(const double2* X, int w, int c, int m, int CPc) {
  const double2 z = X[w * CPc + (c >> 1)];
  const double2 zr = X[((m - w) % m) * CPc + (c >> 1)];
  if ((c & 1) == 0) return make_double2(0.5 * (z.x + zr.x), 0.5 * (z.y - zr.y));   // (Z + conj Zr)/2
  return make_double2(0.5 * (z.y + zr.y), -0.5 * (z.x - zr.x));                     // (Z - conj Zr)/(2i)
}

__global__ void __launch_bounds__(kPrepThreads) prep_kernel(const PrepParams p) {
  extern __shared__ __align__(16) double smem[];
  const int C = p.C, CH = C / 2, CPc = CH + 1, RS = 2 * CPc;   // RS: real-view row stride
  const int m = p.m, m_in = p.m_in;
  const int c0 = blockIdx.x * C;
  const int nc = min(C, p.n - c0);
  const int tid = threadIdx.x;
  long long tr_t = (p.trace && tid == 0) ? clock64() : 0;
  auto mark = [&](int ph) {
    if (p.trace && tid == 0) {
      const long long now = clock64();
      atomicAdd(reinterpret_cast<unsigned long long*>(p.trace + ph), (unsigned long long)(now - tr_t));
      tr_t = now;
    }
  };

  // bufA / bufB: m x CPc complex; the real view of bufA holds channel c of row k
  // at [k * RS + c], so channels (2p, 2p+1) ARE the complex column p.
  double2* bufA = reinterpret_cast<double2*>(smem);
  double2* bufB = bufA + (size_t)m * CPc;
  double2* tw = bufB + (size_t)m * CPc;
  double* raw_s = reinterpret_cast<double*>(tw + m);
  const bool resample = (p.resample_kind != CORR2D_RESAMPLE_NONE);
  double* cstat = raw_s + (resample ? (size_t)m_in * (C + 1) : 0);  // [C] ref, [C] scale
  double* rv = reinterpret_cast<double*>(bufA);

  if (p.do_fft) {  // twiddles W[q] = exp(-2 pi i q / m)
    for (int q = tid; q < m; q += blockDim.x) {
      double s, c;
      sincospi(-2.0 * (double)q / (double)m, &s, &c);
      tw[q] = make_double2(c, s);
    }
  }

  // 1. load the raw m_in x C block (row segments of C channels), count non-finite
  //    All element copies are issued as cp.async (no register round trip), so
  //    the whole block is in flight at once; then one conversion pass.
  int bad = 0;
  const int total_in = m_in * C;
  const int esz = p.in_f32 ? 4 : 8;
  const int csh = 31 - __clz(C);  // C is a power of two
  uint8_t* landing = reinterpret_cast<uint8_t*>(cstat + 2 * C);
  // full, 16-B aligned blocks: 16-byte vector loads straight into registers,
  // converted and written to the FFT buffer (or the resampling input) at once
  const bool vec = (C % 4 == 0) && nc == C && ((reinterpret_cast<uintptr_t>(p.raw) & 15) == 0) &&
                   (((long long)p.ld_raw * esz) % 16 == 0) && (((long long)c0 * esz) % 16 == 0);
  if (vec) {
    const int V = 16 / esz, vsh = p.in_f32 ? 2 : 1;   // channels per vector
    const int vpr_sh = csh - vsh;                     // log2(vectors per row)
    const int total_v = total_in >> vsh;
    constexpr int U = 4;
    for (int base = tid; base < total_v; base += U * blockDim.x) {
      float4 f[U];
      double2 d[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * blockDim.x;
        if (idx < total_v) {
          const int r = idx >> vpr_sh, g = idx & ((1 << vpr_sh) - 1);
          const long long off = (long long)r * p.ld_raw + c0 + g * V;
          if (p.in_f32) f[u] = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(p.raw) + off));
          else d[u] = __ldg(reinterpret_cast<const double2*>(static_cast<const double*>(p.raw) + off));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * blockDim.x;
        if (idx >= total_v) continue;
        const int r = idx >> vpr_sh, c = (idx & ((1 << vpr_sh) - 1)) * V;
        double v[4];
        if (p.in_f32) { v[0] = f[u].x; v[1] = f[u].y; v[2] = f[u].z; v[3] = f[u].w; }
        else { v[0] = d[u].x; v[1] = d[u].y; v[2] = v[3] = 0.0; }
        double* dst = resample ? raw_s + r * (C + 1) + c : rv + r * RS + c;
        for (int e = 0; e < V; ++e) {
          bad += !isfinite(v[e]);
          dst[e] = v[e];
        }
      }
    }
  }
  for (int idx = tid; idx < (vec ? 0 : total_in); idx += blockDim.x) {
    const int r = idx >> csh, c = idx & (C - 1);
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(landing + (size_t)idx * esz));
    if (c < nc) {
      const char* src = static_cast<const char*>(p.raw) + ((long long)r * p.ld_raw + c0 + c) * esz;
      if (esz == 4) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src) : "memory");
      else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
    }
  }
  mark(0);
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  mark(1);
  for (int idx = tid; idx < (vec ? 0 : total_in); idx += blockDim.x) {
    const int r = idx >> csh, c = idx & (C - 1);
    double v = 0.0;
    if (c < nc) v = p.in_f32 ? (double)reinterpret_cast<const float*>(landing)[idx]
                             : reinterpret_cast<const double*>(landing)[idx];
    bad += !isfinite(v);
    if (resample) raw_s[r * (C + 1) + c] = v;
    else rv[r * RS + c] = v;
  }
  bad = warp_sum(bad);
  if ((tid & 31) == 0 && bad) atomicAdd(&p.status[CORR2D_ST_NONFINITE], bad);
  __syncthreads();
  mark(2);

  // 2. resample onto the equidistant axis
  if (resample) {
    for (int idx = tid; idx < m * C; idx += blockDim.x) {
      const int k = idx >> csh, c = idx & (C - 1);
      double v;
      if (p.resample_kind == CORR2D_RESAMPLE_LINEAR) {
        // values[idx] + frac * (values[idx + 1] - values[idx])   (preprocess.py:152)
        const int i = __ldg(p.lin_idx + k);
        const double f = __ldg(p.lin_frac + k);
        const double v0 = raw_s[i * (C + 1) + c], v1 = raw_s[(i + 1) * (C + 1) + c];
        v = __dadd_rn(v0, __dmul_rn(f, __dsub_rn(v1, v0)));
      } else {
        const double* row = p.rs_mat + (size_t)k * m_in;
        double acc = 0.0;
        for (int j = 0; j < m_in; ++j) acc = fma(__ldg(row + j), raw_s[j * (C + 1) + c], acc);
        v = acc;
      }
      rv[k * RS + c] = v;
    }
    __syncthreads();
  }

  // 3. per-channel reference / sigma / scale.  For m <= kSeqStatsMax one thread
  //    per channel sums left to right over the perturbation axis (numpy's
  //    axis-0 order: values / reference / sigma match the reference bit for
  //    bit); longer axes use one warp per channel (strided partial sums + a
  //    fixed xor tree: deterministic, within a few ulp of numpy).
  // the normalisation is folded into the first FFT stage when nothing else
  // needs the normalised values (m even: the first stage is radix 8/4/2)
  const bool normalise = p.ref_mode != CORR2D_REF_NONE || p.alpha > 0.0;
  const bool fuse_norm = normalise && p.do_fft && !p.values_out && (m % 2 == 0);
  if (normalise) {
    const bool wide = m > kSeqStatsMax;
    const int lanes = wide ? 32 : 1;
    const int lane = wide ? (tid & 31) : 0;
    const int worker = wide ? (tid >> 5) : tid;
    const int nworkers = wide ? (int)(blockDim.x >> 5) : (int)blockDim.x;
    auto reduce = [&](double s) {
      if (wide) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
      }
      return s;
    };
    for (int c = worker; c < nc; c += nworkers) {
      const double* col = rv + c;
      double ref;
      if (p.ref_mode == CORR2D_REF_PROVIDED) {
        ref = __ldg(p.ref_in + c0 + c);
      } else if (p.ref_mode == CORR2D_REF_NONE) {
        ref = 0.0;
      } else {
        double s = 0.0;
#pragma unroll 8
        for (int k = lane; k < m; k += lanes) s = __dadd_rn(s, col[k * RS]);
        ref = __ddiv_rn(reduce(s), (double)m);
      }
      double scale = 1.0;
      if (p.alpha > 0.0) {
        double sigma;
        if (p.sigma_in) {
          sigma = __ldg(p.sigma_in + c0 + c);
        } else {
          double ss = 0.0;
#pragma unroll 8
          for (int k = lane; k < m; k += lanes) {
            const double d = __dsub_rn(col[k * RS], ref);
            ss = __dadd_rn(ss, __dmul_rn(d, d));
          }
          sigma = __dsqrt_rn(__ddiv_rn(reduce(ss), (double)(m - 1)));
        }
        if (lane != 0) continue;
        if (p.sigma_out) p.sigma_out[c0 + c] = sigma;  // before substitution
        if (sigma == 0.0) {
          atomicAdd(&p.status[CORR2D_ST_ZEROVAR], 1);
          atomicMax(&p.status[CORR2D_ST_FIRST_ZEROVAR], INT_MAX - (c0 + c));
          if (p.substitute) sigma = 1.0;
        }
        // numpy's power fast paths: x**0.5 -> sqrt, x**1 -> x
        scale = (p.alpha == 0.5) ? __dsqrt_rn(sigma) : (p.alpha == 1.0 ? sigma : pow(sigma, p.alpha));
      }
      if (lane != 0) continue;
      if (p.ref_out) p.ref_out[c0 + c] = ref;
      cstat[c] = ref;
      cstat[C + c] = scale;
    }
    if (fuse_norm && tid >= nc && tid < C) {  // padding channels of a tail block stay 0
      cstat[tid] = 0.0;
      cstat[C + tid] = 1.0;
    }
    __syncthreads();
    mark(3);
    const bool scaled = p.alpha > 0.0;
    for (int idx = tid; idx < (fuse_norm ? 0 : m * C); idx += blockDim.x) {
      const int k = idx >> csh, c = idx & (C - 1);
      double v = rv[k * RS + c];
      if (c < nc) {
        if (p.ref_mode != CORR2D_REF_NONE) v = __dsub_rn(v, cstat[c]);
        if (scaled) v = __ddiv_rn(v, cstat[C + c]);
      }
      rv[k * RS + c] = v;
    }
    __syncthreads();
    mark(4);
  }

  if (p.values_out) {
    for (int idx = tid; idx < m * C; idx += blockDim.x) {
      const int k = idx >> csh, c = idx & (C - 1);
      if (c < nc) p.values_out[(long long)k * p.ld_values + c0 + c] = rv[k * RS + c];
    }
  }
  // 5c. time-domain packing for the Hilbert route (no DFT): slot s < m holds
  //     the dynamic value y(t_s) -- A_phi = Norm * y, B = y; zero padded to mp
  if (p.pack_kind == CORR2D_PACK_F64_TIME) {
    const int mp = p.mp;
    for (int idx = tid; idx < nc * mp; idx += blockDim.x) {
      const int c = idx / mp, s = idx - c * mp;
      const double v = s < m ? rv[s * RS + c] : 0.0;
      const long long row = (long long)(c0 + c) * p.ld_pack + s;
      if (p.pack_roles & CORR2D_ROLE_A) static_cast<double*>(p.a_phi)[row] = p.norm * v;
      if (p.pack_roles & CORR2D_ROLE_B) static_cast<double*>(p.b)[row] = v;
    }
    return;
  }
  if (!p.do_fft) return;

  // 4. DFT along the perturbation axis: two real channels per complex
  //    transform, mixed-radix Stockham autosort (radix 8/4/2 in registers).
  double2* in = bufA;
  double2* out = bufB;
  int Ns = 1;
  for (int f = 0; f < p.nfactors; ++f) {
    const int r = p.factors[f];
    if (f == 0 && fuse_norm) {
      const bool sub = p.ref_mode != CORR2D_REF_NONE, scaled = p.alpha > 0.0;
      if (r == 8) stage_r<8, true>(in, out, tw, m, Ns, CH, CPc, cstat, C, sub, scaled);
      else if (r == 4) stage_r<4, true>(in, out, tw, m, Ns, CH, CPc, cstat, C, sub, scaled);
      else stage_r<2, true>(in, out, tw, m, Ns, CH, CPc, cstat, C, sub, scaled);
    } else if (r == 8) stage_r<8>(in, out, tw, m, Ns, CH, CPc);
    else if (r == 4) stage_r<4>(in, out, tw, m, Ns, CH, CPc);
    else if (r == 2) stage_r<2>(in, out, tw, m, Ns, CH, CPc);
    else stage_generic(in, out, tw, m, r, Ns, CH, CPc);
    __syncthreads();
    double2* t = in; in = out; out = t;
    Ns *= r;
  }
  mark(5);
  const double2* X = in;
  const int K = m / 2 + 1;
  const bool even = (m % 2) == 0;

  if (p.half_out) {
    for (int idx = tid; idx < K * C; idx += blockDim.x) {
      const int w = idx >> csh, c = idx & (C - 1);
      if (c >= nc) continue;
      double2 v = channel_bin(X, w, c, m, CPc);
      if (w == 0 || (even && w == m / 2)) v.y = 0.0;  // rfft: exactly real there
      reinterpret_cast<double2*>(p.half_out)[(long long)w * p.n + c0 + c] = v;
    }
  }

  // 5a. fp64 slot layout: s < K -> Re Y(s); K <= s < m -> Im Y(s - K + 1); rest 0.
  if (p.pack_kind == CORR2D_PACK_F64) {
    const int mp = p.mp;
    const bool p2 = (mp & (mp - 1)) == 0;
    const int msh = 31 - __clz(mp);
    for (int idx = tid; idx < nc * mp; idx += blockDim.x) {
      const int c = p2 ? idx >> msh : idx / mp, s = idx - c * mp;
      double vphi = 0.0, vpsi = 0.0, vb = 0.0;
      if (s < m) {
        int w;
        bool re;
        if (s < K) { w = s; re = true; } else { w = s - K + 1; re = false; }
        const double2 y = channel_bin(X, w, c, m, CPc);
        const bool edge = (w == 0 || (even && w == m / 2));
        const double R = y.x;
        const double I = edge ? 0.0 : y.y;
        double nr = p.norm * R, ni = p.norm * I;
        if (!edge) { nr *= 2.0; ni *= 2.0; }
        if (re) { vphi = nr; vpsi = ni; vb = R; }
        else    { vphi = ni; vpsi = -nr; vb = I; }
      }
      const long long row = (long long)(c0 + c) * p.ld_pack + s;
      if (p.pack_roles & CORR2D_ROLE_A) {
        store_pack(p, p.a_phi, row, vphi);
        store_pack(p, p.a_psi, row, vpsi);
      }
      if (p.pack_roles & CORR2D_ROLE_B) store_pack(p, p.b, row, vb);
    }
  }
  // 5a'. fp64 Gauss layout (corr2d.h CORR2D_PACK_F64_GAUSS): A = [a+b | a | -b],
  //      B = [c | d-c | c+d] over three segments of kg slots
  if (p.pack_kind == CORR2D_PACK_F64_GAUSS) {
    const int mp = p.mp, kg = mp / 3;
    for (int idx = tid; idx < nc * mp; idx += blockDim.x) {
      const int c = idx / mp, s = idx - c * mp;
      const int seg = s / kg, j = s - seg * kg;
      const int w = gauss_bin(seg, j, m);
      double va = 0.0, vb = 0.0;
      if (w >= 0) {
        const double2 y = channel_bin(X, w, c, m, CPc);
        gauss_values(seg, w, m, p.norm, y.x, y.y, va, vb);
      }
      const long long row = (long long)(c0 + c) * p.ld_pack + s;
      if (p.pack_roles & CORR2D_ROLE_A) store_pack(p, p.a_phi, row, va);
      if (p.pack_roles & CORR2D_ROLE_B) store_pack(p, p.b, row, vb);
    }
  }
  // 5b. bf16 layout (see corr2d.h): [Re' | Im' | -Im'] thirds of hp slots each,
  //     Re'[s] = R_s (s < h), Im'[0] = R_{m/2} (even m) or 0, Im'[s] = I_s,
  //     every slot scaled by sqrt(Norm * weight) so A and B share one format;
  //     the negated copy feeds the conj() half of the 2-SM N=256 MMA.
  if (p.pack_kind == CORR2D_PACK_BF16X2) {
    // one item = 4 consecutive slots q..q+3 of one channel: each bin is read
    // once and written as 8-byte (4 x bf16) vectors into the 3 thirds x 2 planes
    const int hp = p.mp / 3;
    const int h = even ? m / 2 : (m + 1) / 2;
    const double sn1 = sqrt(p.norm), sn2 = sqrt(2.0 * p.norm);
    const int q4n = hp / 4;
    const bool p2 = (q4n & (q4n - 1)) == 0;
    const int qsh = 31 - __clz(q4n);
    for (int idx = tid; idx < nc * q4n; idx += blockDim.x) {
      const int c = p2 ? idx >> qsh : idx / q4n, q0 = (idx - c * q4n) * 4;
      // [third][plane] x 4 slots
      __align__(8) __nv_bfloat16 v[3][2][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u;
        double vr = 0.0, vi = 0.0;
        if (q < h) {
          const double2 y = channel_bin(X, q, c, m, CPc);
          vr = y.x * (q == 0 ? sn1 : sn2);
          vi = (q == 0) ? (even ? channel_bin(X, m / 2, c, m, CPc).x * sn1 : 0.0) : y.y * sn2;
        }
        const __nv_bfloat16 rh = __double2bfloat16(vr), ih = __double2bfloat16(vi);
        const __nv_bfloat16 rl = __double2bfloat16(vr - (double)__bfloat162float(rh));
        const __nv_bfloat16 il = __double2bfloat16(vi - (double)__bfloat162float(ih));
        v[0][0][u] = rh; v[0][1][u] = rl;
        v[1][0][u] = ih; v[1][1][u] = il;
        v[2][0][u] = __hneg(ih); v[2][1][u] = __hneg(il);
      }
      // row layout: third t, 32-slot block k -> [hi 32 | lo 32] at t*2hp + 64k
      const long long o = (long long)(c0 + c) * p.ld_pack + (q0 >> 5) * 64 + (q0 & 31);
      // after the 2*mp packed values: fp32 (hi + lo) of Re'[0] and Im'[0], the
      // contraction epilogue's Nyquist x DC correction operands
      const float2 dcn = make_float2(__bfloat162float(v[0][0][0]) + __bfloat162float(v[0][1][0]),
                                     __bfloat162float(v[1][0][0]) + __bfloat162float(v[1][1][0]));
      auto put = [&](void* base) {
        __nv_bfloat16* b = static_cast<__nv_bfloat16*>(base);
#pragma unroll
        for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
          for (int pl = 0; pl < 2; ++pl)
            *reinterpret_cast<uint2*>(b + o + t3 * 2 * hp + pl * 32) = *reinterpret_cast<const uint2*>(v[t3][pl]);
        if (q0 == 0) *reinterpret_cast<float2*>(b + (long long)(c0 + c) * p.ld_pack + 6 * hp) = dcn;
      };
      if (p.pack_roles & CORR2D_ROLE_A) put(p.a_phi);
      if (p.pack_roles & CORR2D_ROLE_B) put(p.b);
    }
  }
  // 5c. fp16 + e4m3 layout (CORR2D_PACK_F16F8, see corr2d.h): same thirds and
  //     32-slot blocks of 128 B, [fp16 hi x 2^5 | e4m3 hi | e4m3 residual x 2^10]
  //     of the channel scaled by its power-of-two sc; pass 1 finds max|slot|.
  if (p.pack_kind == CORR2D_PACK_F16F8) {
    __shared__ unsigned chmax[64];
    const int hp = p.mp / 3;
    const int h = even ? m / 2 : (m + 1) / 2;
    const double sn1 = sqrt(p.norm), sn2 = sqrt(2.0 * p.norm);
    auto slot = [&](int c, int q, float& vr, float& vi) {
      vr = 0.f;
      vi = 0.f;
      if (q < h) {
        const double2 y = channel_bin(X, q, c, m, CPc);
        vr = (float)(y.x * (q == 0 ? sn1 : sn2));
        vi = (float)((q == 0) ? (even ? channel_bin(X, m / 2, c, m, CPc).x * sn1 : 0.0) : y.y * sn2);
      }
    };
    for (int c = tid; c < nc; c += blockDim.x) chmax[c] = 0u;
    __syncthreads();
    for (int idx = tid; idx < nc * h; idx += blockDim.x) {
      const int c = idx / h, q = idx - c * h;
      float vr, vi;
      slot(c, q, vr, vi);
      atomicMax(&chmax[c], max(__float_as_uint(vr) & 0x7fffffffu, __float_as_uint(vi) & 0x7fffffffu));
    }
    __syncthreads();
    const int q4n = hp / 4;
    for (int idx = tid; idx < nc * q4n; idx += blockDim.x) {
      const int c = idx / q4n, q0 = (idx - c * q4n) * 4;
      const int sh = f16f8_shift(chmax[c]);
      const float sc = pow2f(sh);
      float vr[4], vi[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) slot(c, q0 + u, vr[u], vi[u]);
      uint32_t rh[2], ih[2];
      uint16_t rh8[2], rl8[2], ih8[2], il8[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        f16f8_split2(vr[2 * u] * sc, vr[2 * u + 1] * sc, rh[u], rh8[u], rl8[u]);
        f16f8_split2(vi[2 * u] * sc, vi[2 * u + 1] * sc, ih[u], ih8[u], il8[u]);
      }
      // byte offsets inside a third: block q0/32 at 128 B, slot i = q0 % 32 at
      // 2i (fp16), 64 + i (e4m3 hi), 96 + i (e4m3 residual)
      const long long row = (long long)(c0 + c) * p.ld_pack * 2;
      const int o = (q0 >> 5) * 128 + (q0 & 31);
      auto put = [&](void* base) {
        uint8_t* b = static_cast<uint8_t*>(base) + row;
        const uint32_t thr[3] = {0u, (uint32_t)(4 * hp), (uint32_t)(8 * hp)};
#pragma unroll
        for (int t3 = 0; t3 < 3; ++t3) {
          const uint32_t n16 = t3 == 2 ? 0x80008000u : 0u, n8 = t3 == 2 ? 0x80808080u : 0u;
          const uint32_t* h16 = t3 == 0 ? rh : ih;
          const uint16_t* h8 = t3 == 0 ? rh8 : ih8;
          const uint16_t* l8 = t3 == 0 ? rl8 : il8;
          *reinterpret_cast<uint2*>(b + thr[t3] + o + (q0 & 31)) = make_uint2(h16[0] ^ n16, h16[1] ^ n16);
          *reinterpret_cast<uint32_t*>(b + thr[t3] + o + 64) = ((uint32_t)h8[0] | ((uint32_t)h8[1] << 16)) ^ n8;
          *reinterpret_cast<uint32_t*>(b + thr[t3] + o + 96) = ((uint32_t)l8[0] | ((uint32_t)l8[1] << 16)) ^ n8;
        }
        if (q0 == 0)
          *reinterpret_cast<float4*>(b + 12 * hp) = make_float4(vr[0], vi[0], pow2f(-sh - 5), 0.f);
      };
      if (p.pack_roles & CORR2D_ROLE_A) put(p.a_phi);
      if (p.pack_roles & CORR2D_ROLE_B) put(p.b);
    }
  }
  __syncthreads();
  mark(6);
}

// ---------------------------------------------------------------------------
// K1 fast path: one warp per channel pair, the whole length-m transform in
// registers.  m = 32 R (R = 2, 4, 8, 16), no resampling, CORR2D_PACK_BF16X2 or
// CORR2D_PACK_F64 (m <= 128).  A CTA of 8 warps takes 16 channels: the raw
// m x 16 block is staged in shared memory channel-major (conflict-free column
// reads), each warp pulls its two channels into registers as z = x_even + i x_odd
// (lane l holds samples l + 32 t), takes the per-channel statistics in the same
// summation order as the generic kernel (so reference / sigma / values are the
// same bits), and runs the four-step FFT m = R x 32: a length-R DFT in registers,
// twiddles W_m^(l k1), a length-32 DIF butterfly network across lanes (shuffles;
// lane l ends with X[k1 + R bitrev5(l)]).  The two real spectra are split with
// one xor-31 shuffle, packed into a shared-memory row image and written with
// 16-byte stores.  Numerically a different FFT than the generic kernel's
// Stockham passes (both ~1e-16 relative).
// ---------------------------------------------------------------------------
constexpr int kFastThreads = 256;
constexpr int kFastCh = 16;

// complex helpers for the single-precision transform of the bf16 packing path
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }
template <typename C2> __device__ __forceinline__ C2 cmake(double a, double b);
template <> __device__ __forceinline__ double2 cmake<double2>(double a, double b) { return make_double2(a, b); }
template <> __device__ __forceinline__ float2 cmake<float2>(double a, double b) { return make_float2((float)a, (float)b); }

template <typename C2> __device__ __forceinline__ void gdft2(C2& a, C2& b) {
  const C2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}
template <typename C2> __device__ __forceinline__ void gdft4(C2& x0, C2& x1, C2& x2, C2& x3) {
  const C2 t0 = cadd(x0, x2), t1 = csub(x0, x2), t2 = cadd(x1, x3), t3 = mul_mi(csub(x1, x3));
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}
// length-R DFT in registers, natural order in and out (R = 2, 4, 8, 16);
// tw = W_m^q table of the compute type
template <int R, typename C2> __device__ __forceinline__ void gdft(C2 (&x)[R], const C2* __restrict__ tw, int m) {
  if constexpr (R == 2) {
    gdft2(x[0], x[1]);
  } else if constexpr (R == 4) {
    gdft4(x[0], x[1], x[2], x[3]);
  } else if constexpr (R == 8) {
    // 8 = 2 x 4: evens / odds by radix 4, then W8 twiddles and a radix-2 combine
    gdft4(x[0], x[2], x[4], x[6]);
    gdft4(x[1], x[3], x[5], x[7]);
    const int step = m / 8;
    const C2 o0 = x[1], o1 = cmul(x[3], tw[step]), o2 = cmul(x[5], tw[2 * step]), o3 = cmul(x[7], tw[3 * step]);
    const C2 e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6];
    x[0] = cadd(e0, o0); x[4] = csub(e0, o0);
    x[1] = cadd(e1, o1); x[5] = csub(e1, o1);
    x[2] = cadd(e2, o2); x[6] = csub(e2, o2);
    x[3] = cadd(e3, o3); x[7] = csub(e3, o3);
  } else {
    // 16 = 4 x 4: y[t1][u] = DFT4_t2 x[t1 + 4 t2]; y *= W16^(t1 u); X[u + 4 v] = DFT4_t1 y
    C2 y[4][4];
#pragma unroll
    for (int t1 = 0; t1 < 4; ++t1) {
#pragma unroll
      for (int t2 = 0; t2 < 4; ++t2) y[t1][t2] = x[t1 + 4 * t2];
      gdft4(y[t1][0], y[t1][1], y[t1][2], y[t1][3]);
    }
    const int step = m / 16;
#pragma unroll
    for (int t1 = 1; t1 < 4; ++t1)
#pragma unroll
      for (int u = 1; u < 4; ++u) y[t1][u] = cmul(y[t1][u], tw[t1 * u * step]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      C2 a = y[0][u], b = y[1][u], c = y[2][u], d = y[3][u];
      gdft4(a, b, c, d);
      x[u] = a; x[u + 4] = b; x[u + 8] = c; x[u + 12] = d;
    }
  }
}

__device__ __forceinline__ double2 shfl_c(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
__device__ __forceinline__ double2 shfl_xor_c(double2 v, int mask) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, mask), __shfl_xor_sync(0xffffffffu, v.y, mask));
}
__device__ __forceinline__ float2 shfl_c(float2 v, int src) {
  return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
__device__ __forceinline__ float2 shfl_xor_c(float2 v, int mask) {
  return make_float2(__shfl_xor_sync(0xffffffffu, v.x, mask), __shfl_xor_sync(0xffffffffu, v.y, mask));
}

// BF: CORR2D_PACK_BF16X2 -- the transform runs in fp32 (the spectra are then
// split into bf16 hi + lo, ~16 bits, far below fp32's rounding), else fp64.
// --- TMA / mbarrier helpers of the persistent fast kernel
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }
__device__ __forceinline__ void fast_mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fast_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "FAST_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra FAST_DONE;\n\t"
      "bra FAST_WAIT;\n\t"
      "FAST_DONE:\n\t}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// raw rows [r0, M) x channels [c0, c0 + 16) of block `blk` into `dst` (row-major,
// 16 * sizeof(TIN) bytes per row, SWIZZLE_64B for fp32 / SWIZZLE_128B for fp64)
template <int M, typename TIN>
__device__ __forceinline__ void fast_issue(const CUtensorMap* map, uint8_t* dst, uint64_t* bar, int blk) {
  constexpr int BOX = M < 256 ? M : 256;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"((uint32_t)(M * kFastCh * sizeof(TIN))) : "memory");
#pragma unroll
  for (int r0 = 0; r0 < M; r0 += BOX)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
        ::"r"(smem_u32(dst + (size_t)r0 * kFastCh * sizeof(TIN))), "l"(reinterpret_cast<uint64_t>(map)),
          "r"(blk * kFastCh), "r"(r0), "r"(smem_u32(bar)) : "memory");
}

// BF: tensor-core packing (CORR2D_PACK_BF16X2 / F16F8) -- the transform runs in
// fp32 (the spectra are then split into ~16-bit operands, far below fp32's
// rounding), else fp64.
// p.fast_tma: persistent CTAs; each loops over 16-channel blocks, the raw block
// of the block after next is fetched by TMA into the buffer this block has just
// finished with, so DRAM reads overlap the statistics / FFT / packing of the
// blocks in flight.  Otherwise one block per CTA, loaded through registers.
template <int R, typename TIN, bool BF>
__global__ void __launch_bounds__(kFastThreads, 2) prep_fast_kernel(const PrepParams p,
                                                                    const __grid_constant__ CUtensorMap rawmap,
                                                                    const __grid_constant__ CUtensorMap outA,
                                                                    const __grid_constant__ CUtensorMap outB) {
  constexpr int M = 32 * R;
  constexpr int SZ = (int)sizeof(TIN);
  using C2 = typename std::conditional<BF, float2, double2>::type;
  using CT = typename std::conditional<BF, float, double>::type;
  extern __shared__ __align__(1024) double smem[];
  C2* tw = reinterpret_cast<C2*>(smem);                               // M
  uint8_t* bufs = reinterpret_cast<uint8_t*>(smem) + M * sizeof(double2);
  bufs += (1024u - (smem_u32(bufs) & 1023u)) & 1023u;                 // TMA swizzle alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(bufs + 2 * (size_t)p.fast_buf);
  const bool tma = p.fast_tma != 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nblk = (p.n + kFastCh - 1) / kFastCh;
  long long tr_t = (p.trace && tid == 0) ? clock64() : 0;
  auto mark = [&](int ph) {
    if (p.trace && tid == 0) {
      const long long now = clock64();
      atomicAdd(reinterpret_cast<unsigned long long*>(p.trace + ph), (unsigned long long)(now - tr_t));
      tr_t = now;
    }
  };

  if (tma && tid == 0) {
    fast_mbar_init(&bars[0]);
    fast_mbar_init(&bars[1]);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&rawmap)) : "memory");
    for (int s = 0; s < 2; ++s) {
      const int b = blockIdx.x + s * gridDim.x;
      if (b < nblk) fast_issue<M, TIN>(&rawmap, bufs + s * (size_t)p.fast_buf, &bars[s], b);
    }
  }
  for (int q = tid; q < M; q += kFastThreads) {
    double sv, cv;
    sincospi(-2.0 * (double)q / (double)M, &sv, &cv);
    tw[q] = cmake<C2>(cv, sv);
  }
  __syncthreads();

  int it = 0;
  int pend_blk = -1;   // fast_store: raw load deferred until the row-image store has read its buffer
  for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
  uint8_t* work = bufs + (tma ? (it & 1) * (size_t)p.fast_buf : 0);   // raw block, later row images
  TIN* raw_s = reinterpret_cast<TIN*>(work);                           // [16][M + 1] (register path)
  const int c0 = blk * kFastCh;
  const int nc = min(kFastCh, p.n - c0);
  // sample r of channel c of the staged block (TMA: swizzled row-major rows)
  auto raw_at = [&](int c, int r) -> double {
    if (!tma) return (double)raw_s[c * (M + 1) + r];
    const int byte = r * kFastCh * SZ + ((((c * SZ) >> 4) ^ (SZ == 4 ? ((r >> 1) & 3) : (r & 7))) << 4) + ((c * SZ) & 15);
    return (double)*reinterpret_cast<const TIN*>(work + byte);
  };

  int bad = 0;
  if (!tma) {
  // raw block, channel-major in shared memory; full aligned blocks use 16-byte
  // loads, all of a thread's loads issued before the first store
  const TIN* raw = static_cast<const TIN*>(p.raw);
  constexpr int V = 16 / (int)sizeof(TIN), G = kFastCh / V;      // channels per vector, vectors per row
  const bool vec = nc == kFastCh && ((reinterpret_cast<uintptr_t>(raw) & 15) == 0) &&
                   ((p.ld_raw * (long long)sizeof(TIN)) % 16 == 0);
  if (vec) {
    constexpr int PER = M * G / kFastThreads;                     // vectors per thread
    uint4 buf[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = tid + u * kFastThreads, r = idx / G, g = idx % G;
      buf[u] = __ldcs(reinterpret_cast<const uint4*>(raw + (long long)r * p.ld_raw + c0 + g * V));
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = tid + u * kFastThreads, r = idx / G, g = idx % G;
      const TIN* v = reinterpret_cast<const TIN*>(&buf[u]);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        bad += !isfinite(v[e]);
        raw_s[(g * V + e) * (M + 1) + r] = v[e];
      }
    }
  } else {
    for (int idx = tid; idx < M * kFastCh; idx += kFastThreads) {
      const int r = idx >> 4, c = idx & 15;
      TIN v = (TIN)0;
      if (c < nc) {
        v = raw[(long long)r * p.ld_raw + c0 + c];
        bad += !isfinite(v);
      }
      raw_s[c * (M + 1) + r] = v;
    }
  }
  __syncthreads();
  } else {
    fast_mbar_wait(&bars[it & 1], (uint32_t)(it >> 1) & 1u);
  }
  mark(0);

  // this warp's channel pair, samples l + 32 t
  double xv[2][R];
  if (tma) {
    // the pair (2w, 2w+1) shares one 16-byte chunk: one 8 / 16-byte load per row
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const int r = lane + 32 * t, c = 2 * warp;
      const int byte = r * kFastCh * SZ + ((((c * SZ) >> 4) ^ (SZ == 4 ? ((r >> 1) & 3) : (r & 7))) << 4) + ((c * SZ) & 15);
      if constexpr (SZ == 4) {
        const float2 v = *reinterpret_cast<const float2*>(work + byte);
        xv[0][t] = v.x;
        xv[1][t] = v.y;
      } else {
        const double2 v = *reinterpret_cast<const double2*>(work + byte);
        xv[0][t] = v.x;
        xv[1][t] = v.y;
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e)
      if (2 * warp + e < nc)
#pragma unroll
        for (int t = 0; t < R; ++t) bad += !isfinite(xv[e][t]);
  } else {
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int t = 0; t < R; ++t) xv[e][t] = (double)raw_s[(2 * warp + e) * (M + 1) + lane + 32 * t];
  }
  bad = warp_sum(bad);
  if (lane == 0 && bad) atomicAdd(&p.status[CORR2D_ST_NONFINITE], bad);

  // per-channel statistics (generic kernel's summation orders), normalisation
  const bool normalise = p.ref_mode != CORR2D_REF_NONE || p.alpha > 0.0;
  if (normalise) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = 2 * warp + e;
      if (c >= nc) continue;   // padding channels stay 0 (warp-uniform branch)
      double ref = 0.0;
      if (p.ref_mode == CORR2D_REF_PROVIDED) {
        ref = c < nc ? __ldg(p.ref_in + c0 + c) : 0.0;
      } else if (p.ref_mode == CORR2D_REF_MEAN) {
        double sum = 0.0;
        if (M <= kSeqStatsMax) {        // numpy's axis-0 order, left to right
          if (lane == 0) {   // 16 loads in flight ahead of the dependent adds
#pragma unroll
            for (int k0 = 0; k0 < M; k0 += 16) {
              double cv[16];
#pragma unroll
              for (int u = 0; u < 16; ++u) cv[u] = raw_at(c, k0 + u);
#pragma unroll
              for (int u = 0; u < 16; ++u) sum = __dadd_rn(sum, cv[u]);
            }
          }
          sum = __shfl_sync(0xffffffffu, sum, 0);
        } else {                        // lane partials over k = lane + 32 t, xor tree
#pragma unroll
          for (int t = 0; t < R; ++t) sum = __dadd_rn(sum, xv[e][t]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sum = __dadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, o));
        }
        ref = __dmul_rn(sum, 1.0 / (double)M);   // M = 32 R is a power of two: the same bits as sum / M
      }
      double scale = 1.0;
      if (p.alpha > 0.0) {
        double sigma;
        if (p.sigma_in) {
          sigma = c < nc ? __ldg(p.sigma_in + c0 + c) : 1.0;
        } else {
          double ss = 0.0;
          if (M <= kSeqStatsMax) {
            if (lane == 0) {
#pragma unroll
              for (int k0 = 0; k0 < M; k0 += 16) {
                double dv[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                  const double d = __dsub_rn(raw_at(c, k0 + u), ref);
                  dv[u] = __dmul_rn(d, d);
                }
#pragma unroll
                for (int u = 0; u < 16; ++u) ss = __dadd_rn(ss, dv[u]);
              }
            }
            ss = __shfl_sync(0xffffffffu, ss, 0);
          } else {
#pragma unroll
            for (int t = 0; t < R; ++t) {
              const double d = __dsub_rn(xv[e][t], ref);
              ss = __dadd_rn(ss, __dmul_rn(d, d));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
          }
          sigma = __dsqrt_rn(__ddiv_rn(ss, (double)(M - 1)));
        }
        if (lane == 0 && c < nc) {
          if (p.sigma_out) p.sigma_out[c0 + c] = sigma;
          if (sigma == 0.0) {
            atomicAdd(&p.status[CORR2D_ST_ZEROVAR], 1);
            atomicMax(&p.status[CORR2D_ST_FIRST_ZEROVAR], INT_MAX - (c0 + c));
          }
        }
        if (sigma == 0.0 && p.substitute) sigma = 1.0;
        scale = (p.alpha == 0.5) ? __dsqrt_rn(sigma) : (p.alpha == 1.0 ? sigma : pow(sigma, p.alpha));
      }
      if (lane == 0 && c < nc && p.ref_out) p.ref_out[c0 + c] = ref;
      const bool sub = p.ref_mode != CORR2D_REF_NONE, scaled = p.alpha > 0.0;
#pragma unroll
      for (int t = 0; t < R; ++t) {
        if (sub) xv[e][t] = __dsub_rn(xv[e][t], ref);
        if (scaled) xv[e][t] = __ddiv_rn(xv[e][t], scale);
      }
    }
  }

  mark(1);
  // four-step FFT of z = x_even + i x_odd (compute type CT)
  // fp32 transform: each channel of the pair is first brought to max|x| in
  // [1, 2) by an exact power of two 2^pe, so the partner's rounding error in
  // the paired transform is ~2^-24 of the channel's OWN scale, not of the
  // larger partner's; the packing below folds 2^-pe back in
  int pe[2] = {0, 0};
  if constexpr (BF) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double mx = 0.0;
#pragma unroll
      for (int t = 0; t < R; ++t) mx = fmax(mx, fabs(xv[e][t]));
      mx = warp_max(mx);
      if (mx > 0.0 && mx <= 1.7976931348623157e308) pe[e] = min(100, max(-100, -ilogb(mx)));
      const double f = __longlong_as_double((long long)(1023 + pe[e]) << 52);
#pragma unroll
      for (int t = 0; t < R; ++t) xv[e][t] *= f;
    }
  }
  C2 z[R];
#pragma unroll
  for (int t = 0; t < R; ++t) z[t] = cmake<C2>(xv[0][t], xv[1][t]);
  gdft<R, C2>(z, tw, M);
  {
    // W_m^(lane k1) by recurrence from W_m^lane: one shared-memory load instead
    // of R - 1 strided (bank-conflicting) table reads
    const C2 w1 = tw[lane];
    C2 wk = w1;
#pragma unroll
    for (int k1 = 1; k1 < R; ++k1) {
      z[k1] = cmul(z[k1], wk);
      if (k1 + 1 < R) wk = cmul(wk, w1);
    }
  }
#pragma unroll
  for (int h = 16; h > 0; h >>= 1) {   // length-32 DIF across lanes
    const C2 w = tw[(lane & (h - 1)) * (M / (2 * h))];
    const bool upper = (lane & h) != 0;
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) {
      const C2 o = shfl_xor_c(z[k1], h);
      z[k1] = upper ? cmul(csub(o, z[k1]), w) : cadd(z[k1], o);
    }
  }
  // lane holds Z[k1 + R k2], k2 = bitrev5(lane), k1 = 0..R-1 (R consecutive
  // bins); the two real spectra at bin q need Z[m - q]: lane ^ 31, register
  // R - k1 (k1 > 0), or lane bitrev5(-k2 mod 32), register 0 (k1 = 0)
  const int k2 = (int)(__brev((unsigned)lane) >> 27);
  const int src0 = (int)(__brev((unsigned)((32 - k2) & 31)) >> 27);
  auto split = [&](int k1, C2& ye, C2& yo) {
    const C2 zr = k1 == 0 ? shfl_c(z[0], src0) : shfl_xor_c(z[R - k1], 31);
    // (a + b) / 2 rounds the same in the transform's own precision (halving is
    // exact), so the fp32 path needs no fp64 round trip
    ye = cmake<C2>((CT)0.5 * (z[k1].x + zr.x), (CT)0.5 * (z[k1].y - zr.y));
    yo = cmake<C2>((CT)0.5 * (z[k1].y + zr.y), (CT)-0.5 * (z[k1].x - zr.x));
  };
  mark(2);
  __syncthreads();  // raw block consumed: the area now holds the packed row images
  if (pend_blk >= 0 && tid == 0) {
    // the previous block's row-image store has had the statistics / FFT of this
    // block to read its buffer; then the block after this one lands there
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    fast_issue<M, TIN>(&rawmap, bufs + ((it + 1) & 1) * (size_t)p.fast_buf, &bars[(it + 1) & 1], pend_blk);
  }
  pend_blk = -1;

  const int H = M / 2;
  if constexpr (BF) {
   if (p.pack_kind == CORR2D_PACK_F16F8) {
    // CORR2D_PACK_F16F8 row image: thirds [Re' | Im' | -Im'] of hp = H slots,
    // 32-slot blocks of 128 B [fp16 hi x 2^5 | e4m3 hi | e4m3 residual x 2^10]
    // of the channel scaled by its power-of-two sc (warp max first), then
    // float4 (Re'[0], Im'[0], 2^-(s+5), 0) at 12 hp; 16-byte chunks swizzled
    // as in the bf16 image.
    const int hp = H;
    const int img = 6 * hp * 2 + 128;
    // 16-byte chunks XOR-swizzled by the 128-byte line index of the whole block
    // buffer (the TMA SWIZZLE_128B pattern of the copy-out)
    auto aswz = [](int x) { return x ^ (((x >> 7) & 7) << 4); };
    const float sn1 = (float)sqrt(p.norm), sn2 = (float)sqrt(2.0 * p.norm);
    C2 ye[R], yo[R];
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) split(k1, ye[k1], yo[k1]);
    const float nyq0 = __shfl_sync(0xffffffffu, (float)ye[0].x, 1);
    const float nyq1 = __shfl_sync(0xffffffffu, (float)yo[0].x, 1);
    const int q0 = R * k2;
    auto slot = [&](int e, int k1, float& vr, float& vi) {
      const C2 y = e ? yo[k1] : ye[k1];
      const int q = q0 + k1;
      vr = (float)y.x * (q == 0 ? sn1 : sn2);
      vi = q == 0 ? (e ? nyq1 : nyq0) * sn1 : (float)y.y * sn2;
    };
    uint32_t mb[2] = {0u, 0u};
    if (q0 < H) {
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int k1 = 0; k1 < R; ++k1) {
          float vr, vi;
          slot(e, k1, vr, vi);
          mb[e] = max(mb[e], max(__float_as_uint(vr) & 0x7fffffffu, __float_as_uint(vi) & 0x7fffffffu));
        }
    }
    // total shift of channel e: 2^pe (pre-scale) x 2^sh (format scale of the
    // pre-scaled slots), clamped like f16f8_shift
    int sh[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const uint32_t mx = __reduce_max_sync(0xffffffffu, mb[e]);
      sh[e] = (mx == 0u || mx >= 0x7f800000u) ? 0 : min(120, max(-120, f16f8_shift(mx) + pe[e]));
    }
    if (q0 < H) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int rbo = (2 * warp + e) * img;
        const float sc = pow2f(sh[e] - pe[e]);
        __align__(16) uint32_t re_h[R / 2], im_h[R / 2];
        __align__(16) uint16_t re_h8[R / 2], re_l8[R / 2], im_h8[R / 2], im_l8[R / 2];
#pragma unroll
        for (int k1 = 0; k1 < R; k1 += 2) {
          float vr0, vi0, vr1, vi1;
          slot(e, k1, vr0, vi0);
          slot(e, k1 + 1, vr1, vi1);
          f16f8_split2(vr0 * sc, vr1 * sc, re_h[k1 / 2], re_h8[k1 / 2], re_l8[k1 / 2]);
          f16f8_split2(vi0 * sc, vi1 * sc, im_h[k1 / 2], im_h8[k1 / 2], im_l8[k1 / 2]);
        }
        const int blk = (q0 >> 5) * 128, i0 = q0 & 31;
        // NB bytes from v (contiguous, NB | 16-byte chunk), optionally negated
        auto put = [&](int off, const void* v, int nb, uint32_t neg) {
          const uint32_t* w = static_cast<const uint32_t*>(v);
          if (nb >= 16) {
            for (int j = 0; j < nb / 16; ++j)
              *reinterpret_cast<uint4*>(work + aswz(rbo + off + 16 * j)) =
                  make_uint4(w[4 * j] ^ neg, w[4 * j + 1] ^ neg, w[4 * j + 2] ^ neg, w[4 * j + 3] ^ neg);
          } else if (nb == 8) {
            *reinterpret_cast<uint2*>(work + aswz(rbo + off)) = make_uint2(w[0] ^ neg, w[1] ^ neg);
          } else if (nb == 4) {
            *reinterpret_cast<uint32_t*>(work + aswz(rbo + off)) = w[0] ^ neg;
          } else {
            *reinterpret_cast<uint16_t*>(work + aswz(rbo + off)) =
                (uint16_t)(*static_cast<const uint16_t*>(v) ^ (uint16_t)neg);
          }
        };
#pragma unroll
        for (int t3 = 0; t3 < 3; ++t3) {
          const int tb = t3 * 4 * hp + blk;
          const uint32_t n16 = t3 == 2 ? 0x80008000u : 0u, n8 = t3 == 2 ? 0x80808080u : 0u;
          put(tb + 2 * i0, t3 == 0 ? re_h : im_h, 2 * R, n16);
          put(tb + 64 + i0, t3 == 0 ? re_h8 : im_h8, R, n8);
          put(tb + 96 + i0, t3 == 0 ? re_l8 : im_l8, R, n8);
        }
        if (q0 == 0) {
          float vr, vi;
          slot(e, 0, vr, vi);
          const float un = pow2f(-pe[e]);
          *reinterpret_cast<float4*>(work + aswz(rbo + 12 * hp)) =
              make_float4(vr * un, vi * un, pow2f(-sh[e] - 5), 0.f);
        }
      }
    }
    __syncwarp();
    const int vec = (6 * hp * 2 + 16) / 16;
    if (!p.fast_store)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = 2 * warp + e;
      if (c >= nc) continue;
      const uint8_t* src = work + (size_t)c * img;
      for (int role = 0; role < 2; ++role) {
        if (!(p.pack_roles & (role ? CORR2D_ROLE_B : CORR2D_ROLE_A))) continue;
        uint8_t* base = static_cast<uint8_t*>(role ? p.b : p.a_phi);
        uint4* dst = reinterpret_cast<uint4*>(base + (long long)(c0 + c) * p.ld_pack * 2);
        for (int i = lane; i < vec; i += 32) dst[i] = *reinterpret_cast<const uint4*>(work + aswz(c * img + 16 * i));
      }
    }
   } else {
    // row image: thirds [Re' | Im' | -Im'] of hp = H slots, 32-slot blocks
    // [hi 32 | lo 32], then float2 (hi + lo of Re'[0], Im'[0]) at 6 hp.  A
    // lane's R consecutive bins land as 2R contiguous bytes per (third, plane);
    // 16-byte chunks are XOR-swizzled within each 128-byte line by the line
    // index (bank spread), undone by the copy-out.
    const int hp = H;
    const int img = 6 * hp * 2 + 128;
    // 16-byte chunks XOR-swizzled by the 128-byte line index of the whole block
    // buffer (the TMA SWIZZLE_128B pattern of the copy-out)
    auto aswz = [](int x) { return x ^ (((x >> 7) & 7) << 4); };
    const float sn1 = (float)sqrt(p.norm), sn2 = (float)sqrt(2.0 * p.norm);
    C2 ye[R], yo[R];
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) split(k1, ye[k1], yo[k1]);
    const float nyq0 = __shfl_sync(0xffffffffu, (float)ye[0].x, 1);   // bin m/2: register 0 of lane 1
    const float nyq1 = __shfl_sync(0xffffffffu, (float)yo[0].x, 1);
    const int q0 = R * k2;
    if (q0 < H) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int rbo = (2 * warp + e) * img;
        __align__(16) __nv_bfloat16 re_h[R], re_l[R], im_h[R], im_l[R], ng_h[R], ng_l[R];
        // two adjacent bins per conversion instruction (F2FP pack)
#pragma unroll
        for (int k1 = 0; k1 < R; k1 += 2) {
          float vr[2], vi[2];
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            const C2 y = e ? yo[k1 + d] : ye[k1 + d];
            const int q = q0 + k1 + d;
            const float un = pow2f(-pe[e]);   // undo the pre-scale (exact)
            vr[d] = (float)y.x * (q == 0 ? sn1 : sn2) * un;
            vi[d] = (q == 0 ? (e ? nyq1 : nyq0) * sn1 : (float)y.y * sn2) * un;
          }
          const __nv_bfloat162 rh = __floats2bfloat162_rn(vr[0], vr[1]);
          const __nv_bfloat162 ih = __floats2bfloat162_rn(vi[0], vi[1]);
          const float2 rhf = __bfloat1622float2(rh), ihf = __bfloat1622float2(ih);
          const __nv_bfloat162 rl = __floats2bfloat162_rn(vr[0] - rhf.x, vr[1] - rhf.y);
          const __nv_bfloat162 il = __floats2bfloat162_rn(vi[0] - ihf.x, vi[1] - ihf.y);
          *reinterpret_cast<__nv_bfloat162*>(&re_h[k1]) = rh;
          *reinterpret_cast<__nv_bfloat162*>(&re_l[k1]) = rl;
          *reinterpret_cast<__nv_bfloat162*>(&im_h[k1]) = ih;
          *reinterpret_cast<__nv_bfloat162*>(&im_l[k1]) = il;
          *reinterpret_cast<__nv_bfloat162*>(&ng_h[k1]) = __hneg2(ih);
          *reinterpret_cast<__nv_bfloat162*>(&ng_l[k1]) = __hneg2(il);
        }
        const int o = ((q0 >> 5) * 64 + (q0 & 31)) * 2;    // byte offset of bin q0 in a third
        auto put = [&](int off, const __nv_bfloat16 (&v)[R]) {
          if constexpr (2 * R >= 16) {
#pragma unroll
            for (int j = 0; j < 2 * R / 16; ++j)
              *reinterpret_cast<uint4*>(work + aswz(rbo + off + 16 * j)) = reinterpret_cast<const uint4*>(v)[j];
          } else if constexpr (2 * R == 8) {
            *reinterpret_cast<uint2*>(work + aswz(rbo + off)) = *reinterpret_cast<const uint2*>(v);
          } else {
            *reinterpret_cast<uint32_t*>(work + aswz(rbo + off)) = *reinterpret_cast<const uint32_t*>(v);
          }
        };
        put(o, re_h); put(o + 64, re_l);
        put(4 * hp + o, im_h); put(4 * hp + o + 64, im_l);
        put(8 * hp + o, ng_h); put(8 * hp + o + 64, ng_l);
        if (q0 == 0)
          *reinterpret_cast<float2*>(work + aswz(rbo + 12 * hp)) =
              make_float2(__bfloat162float(re_h[0]) + __bfloat162float(re_l[0]),
                          __bfloat162float(im_h[0]) + __bfloat162float(im_l[0]));
      }
    }
    __syncwarp();
    const int vec = (6 * hp * 2 + 8 + 15) / 16;      // 16-byte chunks incl. the float2 pad
    if (!p.fast_store)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = 2 * warp + e;
      if (c >= nc) continue;
      const uint8_t* src = work + (size_t)c * img;
      for (int role = 0; role < 2; ++role) {
        if (!(p.pack_roles & (role ? CORR2D_ROLE_B : CORR2D_ROLE_A))) continue;
        __nv_bfloat16* base = static_cast<__nv_bfloat16*>(role ? p.b : p.a_phi);
        uint4* dst = reinterpret_cast<uint4*>(base + (long long)(c0 + c) * p.ld_pack);
        for (int i = lane; i < vec; i += 32) dst[i] = *reinterpret_cast<const uint4*>(work + aswz(c * img + 16 * i));
      }
    }
   }
  } else {
    // CORR2D_PACK_F64 (M <= 128): slot s < K -> Re Y(s), K <= s < m -> Im Y(s - K + 1);
    // images A_phi | A_psi | B of M doubles each.
    // CORR2D_PACK_F64_GAUSS (M <= 128, kg = M / 2, no padding slots): images
    // A | B of 3 kg = 3 M / 2 doubles each (same bytes)
    const int K = H + 1;
    const int img = 3 * M * 8;
    const bool gauss = p.pack_kind == CORR2D_PACK_F64_GAUSS;
#pragma unroll
    for (int k1 = 0; k1 < R && gauss; ++k1) {
      C2 yy[2];
      split(k1, yy[0], yy[1]);
      const int w = k1 + R * k2;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (w > H) continue;
        double* row = reinterpret_cast<double*>(work + (size_t)(2 * warp + e) * img);
        const int kg = M / 2, G = 3 * kg;
        double va, vb;
        if (w < H) {                                  // DC / interior: segments 0 and 1 at slot w
          gauss_values(0, w, M, p.norm, yy[e].x, (double)yy[e].y, va, vb);
          row[w] = va; row[G + w] = vb;
          gauss_values(1, w, M, p.norm, yy[e].x, (double)yy[e].y, va, vb);
          row[kg + w] = va; row[G + kg + w] = vb;
        }
        if (w >= 1) {                                 // interior at w - 1, Nyquist (w = H) at H - 1
          gauss_values(2, w, M, p.norm, yy[e].x, (double)yy[e].y, va, vb);
          row[2 * kg + w - 1] = va; row[G + 2 * kg + w - 1] = vb;
        }
      }
    }
#pragma unroll
    for (int k1 = 0; k1 < R && !gauss; ++k1) {
      C2 yy[2];
      split(k1, yy[0], yy[1]);
      const int w = k1 + R * k2;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (w > H) continue;
        double* row = reinterpret_cast<double*>(work + (size_t)(2 * warp + e) * img);
        const C2 y = yy[e];
        const bool edge = (w == 0 || w == H);
        const double Rv = y.x, Iv = edge ? 0.0 : (double)y.y;
        double nr = p.norm * Rv, ni = p.norm * Iv;
        if (!edge) { nr *= 2.0; ni *= 2.0; }
        row[w] = nr; row[M + w] = ni; row[2 * M + w] = Rv;                  // Re slot s = w
        if (!edge) {
          const int s = K + w - 1;                                          // Im slot
          row[s] = ni; row[M + s] = -nr; row[2 * M + s] = Iv;
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = 2 * warp + e;
      if (c >= nc) continue;
      const double* src = reinterpret_cast<const double*>(work + (size_t)c * img);
      const long long o = (long long)(c0 + c) * p.ld_pack;
      if (gauss) {
        const int G = 3 * (M / 2);
        for (int s = lane; s < G; s += 32) {
          if (p.pack_roles & CORR2D_ROLE_A) static_cast<double*>(p.a_phi)[o + s] = src[s];
          if (p.pack_roles & CORR2D_ROLE_B) static_cast<double*>(p.b)[o + s] = src[G + s];
        }
        continue;
      }
      for (int s = lane; s < M; s += 32) {
        if (p.pack_roles & CORR2D_ROLE_A) {
          static_cast<double*>(p.a_phi)[o + s] = src[s];
          static_cast<double*>(p.a_psi)[o + s] = src[M + s];
        }
        if (p.pack_roles & CORR2D_ROLE_B) static_cast<double*>(p.b)[o + s] = src[2 * M + s];
      }
    }
  }
  mark(3);
  if (p.fast_store) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // images -> async proxy
  __syncthreads();   // row images complete (copied out, or ready for the TMA store)
  if (tma && tid == 0) {
    const int nb = blk + 2 * (int)gridDim.x;
    if (p.fast_store) {
      // one TMA tensor store of the block's 16 row images (box {64, L, 16},
      // SWIZZLE_128B = the images' chunk swizzle); the buffer is reloaded once
      // the store has read it (next iteration)
      if (p.pack_roles & CORR2D_ROLE_A)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n"
                     ::"l"(reinterpret_cast<uint64_t>(&outA)), "r"(0), "r"(0), "r"(c0), "r"(smem_u32(work)) : "memory");
      if (p.pack_roles & CORR2D_ROLE_B)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n"
                     ::"l"(reinterpret_cast<uint64_t>(&outB)), "r"(0), "r"(0), "r"(c0), "r"(smem_u32(work)) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      if (nb < nblk) pend_blk = nb;
    } else if (nb < nblk) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic writes before the TMA overwrite
      fast_issue<M, TIN>(&rawmap, work, &bars[it & 1], nb);
    }
  }
  }  // blocks of this CTA
  if (p.fast_store && tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// CORR2D_PACK_F64_TIME of already-dynamic values (the Hilbert route's
// operands; hilbert.py:92-115) for ANY m -- no FFT, so no shared-memory limit
// on m (the reference's Toeplitz branch above DENSE_LIMIT = 4096, hilbert.py:
// 52-61, is the same matrix): a tiled transpose out[c][s] = Norm * v[s][c]
// (role A) / v[s][c] (role B), zero padded to mp, with the finite count.
__global__ void __launch_bounds__(256) time_pack_kernel(const PrepParams p) {
  __shared__ double tile[32][33];
  const int s0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  int bad = 0;
  for (int r = ty; r < 32; r += 8) {
    const int s = s0 + r, c = c0 + tx;
    double v = 0.0;
    if (s < p.m && c < p.n) {
      const long long o = (long long)s * p.ld_raw + c;
      v = p.in_f32 ? (double)static_cast<const float*>(p.raw)[o] : static_cast<const double*>(p.raw)[o];
      bad += !isfinite(v);
    }
    tile[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int c = c0 + r, s = s0 + tx;
    if (c < p.n && s < p.mp) {
      const double v = tile[tx][r];
      const long long o = (long long)c * p.ld_pack + s;
      if (p.pack_roles & CORR2D_ROLE_A) static_cast<double*>(p.a_phi)[o] = p.norm * v;
      if (p.pack_roles & CORR2D_ROLE_B) static_cast<double*>(p.b)[o] = v;
    }
  }
  bad = warp_sum(bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&p.status[CORR2D_ST_NONFINITE], bad);
}

static bool time_pack_eligible(const PrepParams& p) {
  return p.pack_kind == CORR2D_PACK_F64_TIME && p.resample_kind == CORR2D_RESAMPLE_NONE &&
         p.ref_mode == CORR2D_REF_NONE && p.alpha == 0.0 && !p.values_out && !p.half_out && !p.ref_out &&
         !p.sigma_out && p.m == p.m_in;
}

static bool fast_eligible(const PrepParams& p) {
  if (const char* e = getenv("CORR2D_PREP_FAST"))
    if (e[0] == '0') return false;
  if (p.resample_kind != CORR2D_RESAMPLE_NONE || p.values_out || p.half_out) return false;
  if (p.m != 64 && p.m != 128 && p.m != 256 && p.m != 512) return false;
  if (p.pack_kind == CORR2D_PACK_BF16X2 || p.pack_kind == CORR2D_PACK_F16F8) return p.mp == 3 * (p.m / 2);
  if (p.pack_kind == CORR2D_PACK_F64_GAUSS) return p.m <= 128 && p.mp == 3 * (p.m / 2);
  return p.pack_kind == CORR2D_PACK_F64 && p.m <= 128 && p.mp == p.m;
}

// bytes of one block buffer: the raw block (TMA rows or the register path's
// channel-major copy) and, after it is consumed, the packed row images
static int fast_buf_bytes(const PrepParams& p) {
  const int M = p.m;
  const size_t sz = p.in_f32 ? 4 : 8;
  const size_t raw = (size_t)kFastCh * (M + 1) * sz;
  const bool f64 = p.pack_kind == CORR2D_PACK_F64 || p.pack_kind == CORR2D_PACK_F64_GAUSS;
  const size_t img = !f64 ? (size_t)kFastCh * (6 * (M / 2) * 2 + 128)
                                                    : (size_t)kFastCh * 3 * M * 8;
  const size_t b = raw > img ? raw : img;
  return (int)((b + 1023) / 1024 * 1024);
}

static size_t fast_smem(const PrepParams& p) {
  return (size_t)p.m * sizeof(double2) + 1024 + 2 * (size_t)fast_buf_bytes(p) + 16;
}

static PFN_cuTensorMapEncodeTiled_v12000 prep_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) == cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// TMA map of the raw m x n block matrix: boxes of 16 channels x min(m, 256) rows
// (64-B rows SWIZZLE_64B for fp32, 128-B rows SWIZZLE_128B for fp64); channels
// past n read as zeros.  false when the layout does not allow TMA.
static bool fast_raw_map(const PrepParams& p, CUtensorMap* map) {
  const size_t sz = p.in_f32 ? 4 : 8;
  if (const char* e = getenv("CORR2D_PREP_TMA"))
    if (e[0] == '0') return false;
  if ((reinterpret_cast<uintptr_t>(p.raw) & 15) || ((size_t)p.ld_raw * sz) % 16) return false;
  auto fn = prep_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)p.n, (cuuint64_t)p.m};
  cuuint64_t strides[1] = {(cuuint64_t)p.ld_raw * sz};
  cuuint32_t box[2] = {(cuuint32_t)kFastCh, (cuuint32_t)(p.m < 256 ? p.m : 256)};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, p.in_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
            const_cast<void*>(p.raw), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            p.in_f32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA map of a tensor-core packed operand array viewed as {64 x 2 B, L lines of
// 128 B, n rows}: one box {64, L, 16} = the 16 row images of a block, in the
// SWIZZLE_128B layout the images are written in.
static bool fast_out_map(const PrepParams& p, void* base, CUtensorMap* map) {
  if (!base || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  const int hp = p.m / 2;
  const int L = (12 * hp + 128) / 128;
  if (L > 256 || (long long)p.ld_pack * 2 < (long long)L * 128) return false;
  auto fn = prep_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {64, (cuuint64_t)L, (cuuint64_t)p.n};
  cuuint64_t strides[2] = {128, (cuuint64_t)p.ld_pack * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)L, (cuuint32_t)kFastCh};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename K>
static void launch_fast_kernel(K kern, PrepParams p, size_t smem, cudaStream_t st) {
  const int nblk = (p.n + kFastCh - 1) / kFastCh;
  CUtensorMap map, oa, ob;
  memset(&map, 0, sizeof(map));
  memset(&oa, 0, sizeof(oa));
  memset(&ob, 0, sizeof(ob));
  p.fast_buf = fast_buf_bytes(p);
  p.fast_tma = fast_raw_map(p, &map) ? 1 : 0;
  p.fast_store = 0;
  if (p.fast_tma && (p.pack_kind == CORR2D_PACK_BF16X2 || p.pack_kind == CORR2D_PACK_F16F8)) {
    const char* e = getenv("CORR2D_PREP_TMA_STORE");
    bool ok = !(e && e[0] == '0');
    if (ok && (p.pack_roles & CORR2D_ROLE_A)) ok = fast_out_map(p, p.a_phi, &oa);
    if (ok && (p.pack_roles & CORR2D_ROLE_B)) ok = fast_out_map(p, p.b, &ob);
    p.fast_store = ok ? 1 : 0;
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = nblk;
  if (p.fast_tma) {   // persistent: as many CTAs as fit, never more than the blocks
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFastThreads, smem) != cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    grid = std::min(nblk, per_sm * sms);
  }
  kern<<<grid, kFastThreads, smem, st>>>(p, map, oa, ob);
}

template <int R, bool BF>
static void launch_fast_rb(const PrepParams& p, size_t smem, cudaStream_t st) {
  if (p.in_f32) launch_fast_kernel(prep_fast_kernel<R, float, BF>, p, smem, st);
  else launch_fast_kernel(prep_fast_kernel<R, double, BF>, p, smem, st);
}
template <int R>
static void launch_fast_r(const PrepParams& p, size_t smem, cudaStream_t st) {
  if (p.pack_kind == CORR2D_PACK_BF16X2 || p.pack_kind == CORR2D_PACK_F16F8) launch_fast_rb<R, true>(p, smem, st);
  else if constexpr (R <= 4) launch_fast_rb<R, false>(p, smem, st);   // F64 packing: m <= 128
}

static int fft_factorize(int m, int* f, int maxf) {
  int k = 0;
  for (int r : {8, 4, 2}) {
    while (m % r == 0 && m > 1) {
      if (k >= maxf) return -1;
      f[k++] = r;
      m /= r;
    }
  }
  for (int q = 3; m > 1; q += 2) {
    while (m % q == 0) {
      if (k >= maxf) return -1;
      f[k++] = q;
      m /= q;
    }
    if ((long long)q * q > m && m > 1) {  // remaining m is prime
      if (k >= maxf) return -1;
      f[k++] = m;
      m = 1;
    }
  }
  return k;
}

static size_t prep_smem_bytes(int m, int m_in, int C, bool resample, int in_bytes) {
  const size_t CPc = C / 2 + 1;
  size_t b = 2 * (size_t)m * CPc * sizeof(double2) + (size_t)m * sizeof(double2);
  if (resample) b += (size_t)m_in * (C + 1) * sizeof(double);
  b += 2 * (size_t)C * sizeof(double);
  b += (size_t)m_in * C * in_bytes;  // cp.async landing zone of the raw block
  return b;
}

}  // namespace corr2d

using namespace corr2d;

extern "C" int corr2d_fft_factors(int m, int* factors, int max_factors) {
  if (m < 1) return fail(CORR2D_ERR_DATA, "fft length must be >= 1");
  int tmp[kMaxFactors];
  int k = fft_factorize(m, tmp, kMaxFactors);
  if (k < 0) return fail(CORR2D_ERR_UNSUPPORTED, "too many FFT factors");
  for (int i = 0; i < k && i < max_factors; ++i) factors[i] = tmp[i];
  return k;
}

extern "C" int corr2d_packed_depth(int m, int pack_kind) {
  if (m < 2) return fail(CORR2D_ERR_DATA, "need m >= 2");
  if (pack_kind == CORR2D_PACK_BF16X2 || pack_kind == CORR2D_PACK_F16F8) {
    const int h = (m % 2 == 0) ? m / 2 : (m + 1) / 2;
    return 3 * ((h + 31) / 32 * 32);
  }
  if (pack_kind == CORR2D_PACK_F64_GAUSS) return 3 * gauss_kg(m);
  return (m + 3) / 4 * 4;
}

extern "C" int corr2d_prep(
    int in_dtype, const void* raw, int64_t ld_raw, int m_in, int n,
    int resample_kind, const int32_t* lin_idx, const double* lin_frac,
    const double* resample_matrix, int m,
    int ref_mode, const double* ref_in, const double* sigma_in, double alpha, int substitute_zero_var,
    double norm_const, int pack_kind, int pack_roles,
    void* a_phi, void* a_psi, void* b, int64_t ld_pack, int64_t split_plane,
    double* values_out, int64_t ld_values, double* half_out,
    double* ref_out, double* sigma_out, int32_t* status, void* stream) {
  if (!raw || !status) return fail(CORR2D_ERR_DATA, "corr2d_prep: raw and status are required");
  if (m_in < 2 || n < 1 || m < 2) return fail(CORR2D_ERR_DATA, "corr2d_prep: need m >= 2 and n >= 1");
  if (in_dtype != CORR2D_F64 && in_dtype != CORR2D_F32) return fail(CORR2D_ERR_DATA, "corr2d_prep: bad dtype");
  if (resample_kind == CORR2D_RESAMPLE_NONE && m != m_in)
    return fail(CORR2D_ERR_DATA, "corr2d_prep: m != m_in without resampling");
  if (resample_kind == CORR2D_RESAMPLE_LINEAR && (!lin_idx || !lin_frac))
    return fail(CORR2D_ERR_DATA, "corr2d_prep: linear resampling needs idx/frac");
  if (resample_kind == CORR2D_RESAMPLE_MATRIX && !resample_matrix)
    return fail(CORR2D_ERR_DATA, "corr2d_prep: matrix resampling needs the matrix");
  if (ld_raw < n) return fail(CORR2D_ERR_DATA, "corr2d_prep: ld_raw < n");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(CORR2D_ERR_DATA, "scaling exponent must lie in [0, 1]");

  PrepParams p{};
  p.raw = raw; p.in_f32 = (in_dtype == CORR2D_F32); p.ld_raw = ld_raw; p.m_in = m_in; p.n = n;
  p.resample_kind = resample_kind; p.lin_idx = lin_idx; p.lin_frac = lin_frac; p.rs_mat = resample_matrix;
  if (ref_mode < CORR2D_REF_MEAN || ref_mode > CORR2D_REF_NONE) return fail(CORR2D_ERR_DATA, "corr2d_prep: bad ref_mode");
  if (ref_mode == CORR2D_REF_PROVIDED && !ref_in) return fail(CORR2D_ERR_DATA, "corr2d_prep: provided reference missing");
  p.m = m; p.ref_mode = ref_mode; p.ref_in = ref_in; p.sigma_in = sigma_in; p.alpha = alpha;
  p.substitute = substitute_zero_var; p.norm = norm_const;
  p.pack_kind = pack_kind; p.pack_roles = pack_roles;
  p.a_phi = a_phi; p.a_psi = a_psi; p.b = b; p.ld_pack = ld_pack; p.split_plane = split_plane;
  p.values_out = values_out; p.ld_values = ld_values; p.half_out = half_out;
  p.ref_out = ref_out; p.sigma_out = sigma_out; p.status = status;
  if (pack_kind < CORR2D_PACK_NONE || pack_kind > CORR2D_PACK_F64_GAUSS)
    return fail(CORR2D_ERR_DATA, "corr2d_prep: bad pack_kind");
  const bool tc_pack = pack_kind == CORR2D_PACK_BF16X2 || pack_kind == CORR2D_PACK_F16F8;
  p.do_fft = (half_out != nullptr) || pack_kind == CORR2D_PACK_F64 || pack_kind == CORR2D_PACK_F64_GAUSS || tc_pack;
  if (pack_kind != CORR2D_PACK_NONE) {
    p.mp = corr2d_packed_depth(m, pack_kind);
    if (tc_pack) {
      if (ld_pack < 2 * (long long)p.mp + 64 || ld_pack % 64)
        return fail(CORR2D_ERR_DATA, "corr2d_prep: bf16 / f16f8 ld_pack must be >= 2 * packed depth + 64 and a multiple of 64");
    } else if (ld_pack < p.mp) {
      return fail(CORR2D_ERR_DATA, "corr2d_prep: ld_pack < packed depth");
    }
    if ((pack_roles & CORR2D_ROLE_A) && (!a_phi || (pack_kind == CORR2D_PACK_F64 && !a_psi)))
      return fail(CORR2D_ERR_DATA, "corr2d_prep: A operands missing");
    if ((pack_roles & CORR2D_ROLE_B) && !b) return fail(CORR2D_ERR_DATA, "corr2d_prep: B operand missing");
  }
  if (values_out && ld_values < n) return fail(CORR2D_ERR_DATA, "corr2d_prep: ld_values < n");
  p.nfactors = fft_factorize(m, p.factors, kMaxFactors);
  if (p.nfactors < 0) return fail(CORR2D_ERR_UNSUPPORTED, "corr2d_prep: FFT factorisation failed");

  if (small_eligible(p)) {
    return launch_prep_small(p, static_cast<cudaStream_t>(stream));
  }
  if (fast_eligible(p)) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    static long long* ftrace = nullptr;
    const char* ftrc = getenv("CORR2D_PREP_TRACE");
    if (ftrc && ftrc[0] == '1') {
      if (!ftrace) cudaMalloc(&ftrace, 16 * sizeof(long long));
      cudaMemsetAsync(ftrace, 0, 16 * sizeof(long long), st);
      p.trace = ftrace;
    }
    if (cudaMemsetAsync(status, 0, 4 * sizeof(int32_t), st) != cudaSuccess) return check_launch("status reset");
    const size_t smem = fast_smem(p);
    switch (m) {
      case 64: launch_fast_r<2>(p, smem, st); break;
      case 128: launch_fast_r<4>(p, smem, st); break;
      case 256: launch_fast_r<8>(p, smem, st); break;
      default: launch_fast_r<16>(p, smem, st); break;
    }
    if (p.trace) {
      long long h[16];
      cudaMemcpyAsync(h, p.trace, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const double g = (double)((n + kFastCh - 1) / kFastCh);
      fprintf(stderr, "prep fast trace (cycles/CTA, grid=%.0f): load %.0f stats %.0f fft %.0f pack %.0f\n", g,
              h[0] / g, h[1] / g, h[2] / g, h[3] / g);
    }
    return check_launch("prep_fast_kernel");
  }

  if (time_pack_eligible(p)) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(status, 0, 4 * sizeof(int32_t), st) != cudaSuccess) return check_launch("status reset");
    const dim3 grid((n + 31) / 32, (p.mp + 31) / 32);
    time_pack_kernel<<<grid, 256, 0, st>>>(p);
    return check_launch("time_pack_kernel");
  }
  const bool resample = resample_kind != CORR2D_RESAMPLE_NONE;
  int C = 64;
  const int in_bytes = (in_dtype == CORR2D_F32) ? 4 : 8;
  const size_t budget = 110 * 1024;
  while (C > 2 && prep_smem_bytes(m, m_in, C, resample, in_bytes) > budget) C /= 2;
  {
    // small n (cfg1 / cfg2: 1000 - 2000 channels): fewer channels per CTA so the
    // grid covers the SMs; not below 8 -- the per-CTA fixed cost then wins
    // (cfg1 K1: C 64 11.7 us, C 8 10.0 us, C 2 14.5 us).  Any even C gives the
    // same bits (each channel pair is transformed on its own).
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    while (C > 8 && (n + C - 1) / C < sms) C /= 2;
  }
  if (const char* e = getenv("CORR2D_PREP_C")) {  // experiments: channels per CTA
    const int forced = atoi(e);
    if (forced >= 2 && forced <= 64 && (forced & (forced - 1)) == 0) C = forced;
  }
  size_t smem = prep_smem_bytes(m, m_in, C, resample, in_bytes);
  if (smem > 220 * 1024)
    return fail(CORR2D_ERR_UNSUPPORTED, "corr2d_prep: m too large for the shared-memory FFT (m <= ~4096)");
  p.C = C;
  cudaFuncSetAttribute(prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(status, 0, 4 * sizeof(int32_t), st) != cudaSuccess) return check_launch("status reset");
  const int grid = (n + C - 1) / C;
  static long long* trace_buf = nullptr;
  const char* trc = getenv("CORR2D_PREP_TRACE");
  if (trc && trc[0] == '1') {
    if (!trace_buf) cudaMalloc(&trace_buf, 16 * sizeof(long long));
    cudaMemsetAsync(trace_buf, 0, 16 * sizeof(long long), st);
    p.trace = trace_buf;
  }
  prep_kernel<<<grid, kPrepThreads, smem, st>>>(p);
  if (p.trace) {
    long long h[16];
    cudaMemcpyAsync(h, p.trace, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "prep trace (cycles/CTA, C=%d grid=%d): issue %.0f wait %.0f convert %.0f stats %.0f normalise %.0f "
            "fft %.0f pack %.0f\n", C, grid, (double)h[0] / grid, (double)h[1] / grid, (double)h[2] / grid,
            (double)h[3] / grid, (double)h[4] / grid, (double)h[5] / grid, (double)h[6] / grid);
  }
  return check_launch("prep_kernel");
}
