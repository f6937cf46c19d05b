// K1 launch parameters, shared by prep.cu (generic / fast kernels) and
// small.cu (small-m kernel and the fused small-m correlation).
#pragma once

#include "common.cuh"

namespace corr2d {

constexpr int kMaxFactors = 24;

struct PrepParams {
  const void* raw;
  int in_f32;
  long long ld_raw;
  int m_in, n;
  int resample_kind;
  const int* lin_idx;
  const double* lin_frac;
  const double* rs_mat;
  int m;
  int ref_mode;            // CORR2D_REF_MEAN / _PROVIDED / _NONE
  const double* ref_in;
  const double* sigma_in;  // optional provided sigma (apply_scaling)
  double alpha;
  int substitute;
  double norm;
  int pack_kind, pack_roles;
  void* a_phi;
  void* a_psi;
  void* b;
  long long ld_pack, split_plane;
  int mp;
  double* values_out;
  long long ld_values;
  double* half_out;
  double* ref_out;
  double* sigma_out;
  int* status;
  int do_fft;
  long long* trace;        // profiling (CORR2D_PREP_TRACE=1): per-phase cycles, summed over CTAs
  int fast_tma;            // fast kernel: persistent CTAs, raw blocks double-buffered by TMA
  int fast_buf;            // fast kernel: bytes per block buffer (multiple of 1024)
  int fast_store;          // fast kernel (tensor-core packing, TMA mode): row images leave by one TMA store
  int C;
  int nfactors;
  int factors[kMaxFactors];
};

// ---- CORR2D_PACK_F64_GAUSS (corr2d.h): three real products per bin.
// Interior bins (neither DC nor Nyquist): 1 .. gauss_interior(m).
__host__ __device__ __forceinline__ int gauss_interior(int m) { return (m - 1) / 2; }
// Slots per segment: the DC / Nyquist bin plus the interior bins, rounded up to
// a multiple of 4 (the DMMA k-step).
__host__ __device__ __forceinline__ int gauss_kg(int m) { return (gauss_interior(m) + 1 + 3) / 4 * 4; }
// The bin segment `seg` (0, 1, 2) carries in slot j, or -1 for a zero pad.
__host__ __device__ __forceinline__ int gauss_bin(int seg, int j, int m) {
  const int I = gauss_interior(m);
  if (seg < 2) return j <= I ? j : -1;                 // DC at slot 0, interior bins at 1..I
  if (j < I) return j + 1;                             // interior bins at 0..I-1
  return (j == I && (m % 2) == 0) ? m / 2 : -1;        // Nyquist (even m) at slot I
}
// Operand values of bin w (spectrum R + i Iraw) in segment seg: with
// a = Norm w R, b = Norm w I, c = R, d = -I:  seg 0 (a + b, c), seg 1 (a, d - c),
// seg 2 (-b, c + d) -- or (a, c) for the real Nyquist bin.  Norm and the
// half-spectrum weight are applied in the order of the CORR2D_PACK_F64 slots.
__device__ __forceinline__ void gauss_values(int seg, int w, int m, double norm, double R, double Iraw,
                                             double& va, double& vb) {
  const bool edge = (w == 0 || ((m % 2) == 0 && w == m / 2));
  const double I = edge ? 0.0 : Iraw;
  double a = norm * R, b = norm * I;
  if (!edge) { a *= 2.0; b *= 2.0; }
  const double c = R, d = -I;
  if (seg == 0) { va = a + b; vb = c; }
  else if (seg == 1) { va = a; vb = d - c; }
  else if (edge) { va = a; vb = c; }
  else { va = -b; vb = c + d; }
}

// Small-m K1 (m <= 32, no resampling, fp64 packing), small.cu.
bool small_eligible(const PrepParams& p);
int launch_prep_small(const PrepParams& p, cudaStream_t st);

}  // namespace corr2d
