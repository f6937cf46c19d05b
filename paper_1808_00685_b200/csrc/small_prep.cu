// Small-m K1 (m <= 32, no resampling, CORR2D_PACK_F64 operands): prep_small_kernel,
// one warp per channel pair (corr2d_prep; the one-launch correlation of these
// shapes is small_fused.cu).
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

}  // namespace corr2d
