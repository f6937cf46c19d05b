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

// Small-m K1 (m <= 32, no resampling, fp64 packing), small.cu.
bool small_eligible(const PrepParams& p);
int launch_prep_small(const PrepParams& p, cudaStream_t st);

}  // namespace corr2d
