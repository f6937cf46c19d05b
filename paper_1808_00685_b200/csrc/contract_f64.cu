// K2 (fp64) -- packed-spectrum contraction  sync = A_phi . B^T,  async = A_psi . B^T.
//
// Restates the hot loop of correlate_ft (fourier.py:107-123): the weighted
// half-spectrum complex cross sum  Norm * sum_w weight(w) Y1(nu1,w) conj(Y2(nu2,w))
// in OpenBLAS zgemm row blocks (engine_core.py:114-127), then the Re/Im split.
// Here the complex contraction over K bins is an exact real contraction over
// the packed depth m (see include/corr2d.h), done on the FP64 tensor pipe
// (mma.sync m16n8k4 f64 -> SASS DMMA.8x8x4; B200 has no tcgen05 f64 kind).
//
// CTA tile 64 x 64 output elements of BOTH planes, 4 warps of 32 x 32.
// Operands stream through shared memory in depth chunks of 64 (cp.async);
// the epilogue stages both planes in shared memory and writes them as
// coalesced 256 B row segments -- and, for homo tiles above the diagonal,
// also the mirrored tile (sync^T, -async^T), so the result is exactly
// symmetric / skew-symmetric (dataset.py:159-170) and half the tiles are
// never computed.  Finite check and max|.| are fused into the same pass
// (engine_core.py:139-140).
#include "common.cuh"

#include <cmath>
#include <cstdlib>

namespace corr2d {

constexpr int kBM = 64;
constexpr int kBN = 64;
// depth chunk 32 + at least 3 CTAs / SM: the DMMA accumulate chains are
// latency-bound (ncu: "wait" stalls), so resident warps matter more than
// depth per chunk -- measured cfg3 1.91 -> 1.61 ms, cfg4 0.51 -> 0.42 ms
#ifndef CORR2D_F64_KC
#define CORR2D_F64_KC 32
#endif
#ifndef CORR2D_F64_MINB
#define CORR2D_F64_MINB 3
#endif
constexpr int kKC = CORR2D_F64_KC; // depth chunk
#ifndef CORR2D_F64_NBUF
#define CORR2D_F64_NBUF 1
#endif
constexpr int kNBuf = CORR2D_F64_NBUF;                // operand buffers (2: double buffering)
constexpr int kKS = kKC + 4;       // smem row stride (doubles): conflict-free fragments
constexpr int kCS = kBN + 1;       // epilogue staging stride
constexpr int kBufStride = 3 * 64 * (kKC + 4);   // doubles per operand buffer (A_phi, A_psi, B)
// MT m16 row tiles per warp: 2 -> 4 warps of 32 x 32 (128 threads); 1 -> 8 warps
// of 16 x 32 (256 threads, half the accumulator registers per thread)
#ifndef CORR2D_F64_MT
#define CORR2D_F64_MT 2
#endif
constexpr int kMT = CORR2D_F64_MT;
constexpr int kThreads = 32 * 2 * (64 / (16 * kMT));

// kTransOnly: a tile left of the shard's diagonal square is computed as its
// globally-upper mirror (operand tiles swapped) and only the transpose is
// written, so every element has the value the unsharded call computes.
enum TileMode { kPlain = 0, kMirror = 1, kDiag = 2, kTransOnly = 3 };

struct ContractParams {
  const double* a_phi;
  const double* a_psi;
  const double* b;
  long long ld_pack;
  int n1, n2, mp;
  int kg;           // Gauss operands (CORR2D_PACK_F64_GAUSS): slots per segment, mp = 3 kg
  int dbg;          // profiling builds only (-DCORR2D_PROFILING): 1 = no output stores, 2 = no MMAs
  int homo;
  int row0, row1;
  int I0, I1, T;  // row-tile range of the shard, number of column tiles
  long long tile0;  // first tile of this launch (tile-range partition)
  int vec_direct;   // planes 16-B aligned with an even ld_out: direct tiles from registers
  double* phi;
  double* psi;
  long long ld_out;
  unsigned long long* stats;
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gsrc), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Decode the linear block index into (row tile I, column tile J, mode).
__device__ __forceinline__ void decode_tile(const ContractParams& p, int& I, int& J, int& mode) {
  const long long b = p.tile0 + blockIdx.x;
  if (!p.homo) {
    I = p.I0 + (int)(b / p.T);
    J = (int)(b % p.T);
    mode = kPlain;
    return;
  }
  // row tile I0 + d owns columns [0, I0) U [I0 + d, T): count T - d.
  // S(d) = d T - d (d - 1) / 2 tiles precede it.
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
    J = I;           // own rows: written through the transpose
    I = (int)o;      // row-operand tile outside the shard
    mode = kTransOnly;
  } else {
    J = I + (int)(o - p.I0);
    mode = (J == I) ? kDiag : (J < p.I1 ? kMirror : kPlain);
  }
}

// Both planes of a staged 64 x 64 tile (row pitch kCS) -> global memory as
// coalesced 256-B row segments, plus the mirrored tile (sync^T, -async^T) of
// homo tiles above the diagonal; fused max|.| / finite check into p.stats.
// direct_done: the direct tile was already written from registers by the
// caller, whose max / finite partials come in through mphi0 / mpsi0 / bad0.
// max|x| and the finite check on the INTEGER pipe: |x|'s bit pattern orders
// like |x| and Inf / NaN patterns exceed every finite one.  (fp64 fmax / fabs /
// isfinite would queue on the FP64 pipe behind the DMMAs of the co-resident CTAs.)
constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;
__device__ __forceinline__ unsigned long long absbits(double x) { return abs_bits(x); }
__device__ __forceinline__ double dneg(double x) { return neg_bits(x); }   // sign flip, integer pipe

__device__ __forceinline__ void write_tile(const ContractParams& p, int mode, int i0, int j0,
                                           const double* Cphi, const double* Cpsi, int tid, int nthreads,
                                           int lane, bool direct_done = false, unsigned long long bphi0 = 0,
                                           unsigned long long bpsi0 = 0) {
  unsigned long long bphi = bphi0, bpsi = bpsi0;
  for (int idx = tid; idx < kBM * kBN; idx += nthreads) {
    if (mode == kTransOnly || direct_done) break;
    const int r = idx >> 6, c = idx & 63;
    const int gi = i0 + r, gj = j0 + c;
    if (gi >= p.row1 || gj >= p.n2) continue;
    double vphi, vpsi;
    if (mode == kDiag) {
      if (r <= c) { vphi = Cphi[r * kCS + c]; } else { vphi = Cphi[c * kCS + r]; }
      if (r < c) vpsi = Cpsi[r * kCS + c];
      else if (r == c) vpsi = 0.0;
      else vpsi = dneg(Cpsi[c * kCS + r]);
    } else {
      vphi = Cphi[r * kCS + c];
      vpsi = Cpsi[r * kCS + c];
    }
    const long long o = (long long)(gi - p.row0) * p.ld_out + gj;
    __stcs(p.phi + o, vphi);
    __stcs(p.psi + o, vpsi);
    bphi = max(bphi, absbits(vphi));
    bpsi = max(bpsi, absbits(vpsi));
  }
  const bool mirror_full = p.vec_direct && j0 >= p.row0 && j0 + kBN <= p.row1 && i0 + kBM <= p.n2;
  if ((mode == kMirror || mode == kTransOnly) && mirror_full && nthreads == 128) {
    // whole mirrored tile in bounds: a thread owns a column pair of the output
    // rows, 16-byte stores, pointer steps (a third of the generic loop's issue)
    const int c0 = 2 * (tid & 31), r4 = tid >> 5;
    const long long step = 4 * p.ld_out;
    double* dphi = p.phi + (long long)(j0 + r4 - p.row0) * p.ld_out + i0 + c0;
    double* dpsi = p.psi + (dphi - p.phi);
#pragma unroll 4
    for (int k = 0; k < kBN / 4; ++k) {
      const int rr = r4 + 4 * k;
      const double a0 = Cphi[c0 * kCS + rr], a1 = Cphi[(c0 + 1) * kCS + rr];
      const double b0 = dneg(Cpsi[c0 * kCS + rr]), b1 = dneg(Cpsi[(c0 + 1) * kCS + rr]);
      __stcs(reinterpret_cast<double2*>(dphi), make_double2(a0, a1));
      __stcs(reinterpret_cast<double2*>(dpsi), make_double2(b0, b1));
      if (mode == kTransOnly) {
        bphi = max(bphi, max(absbits(a0), absbits(a1)));
        bpsi = max(bpsi, max(absbits(b0), absbits(b1)));
      }
      dphi += step;
      dpsi += step;
    }
  } else if (mode == kMirror || mode == kTransOnly) {
    // out[j][i] = sync[i][j], -async[i][j] for the tile below the diagonal
    for (int idx = tid; idx < kBM * kBN; idx += nthreads) {
      const int rr = idx >> 6, cc = idx & 63;   // rr: column of C, cc: row of C
      const int gi = j0 + rr, gj = i0 + cc;
      if (gi >= p.row1 || gj >= p.n2 || gi < p.row0) continue;
      const long long o = (long long)(gi - p.row0) * p.ld_out + gj;
      const double vphi = Cphi[cc * kCS + rr], vpsi = dneg(Cpsi[cc * kCS + rr]);
      __stcs(p.phi + o, vphi);
      __stcs(p.psi + o, vpsi);
      if (mode == kTransOnly) {
        bphi = max(bphi, absbits(vphi));
        bpsi = max(bpsi, absbits(vpsi));
      }
    }
  }
  int bad = (bphi >= kInfBits) + (bpsi >= kInfBits);   // lanes holding a non-finite value
  bphi = min(bphi, kInfBits);
  bpsi = min(bpsi, kInfBits);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {   // integer max of the bit patterns (fmax would use the FP64 pipe)
    bphi = max(bphi, (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)bphi, o));
    bpsi = max(bpsi, (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)bpsi, o));
  }
  bad = warp_sum(bad);
  // one set of atomics per CTA (tens of thousands of CTAs hit the same three
  // words); the max stays on bit patterns (non-negative doubles order like them)
  __shared__ unsigned long long red_m[2][8];
  __shared__ int red_b[8];
  const int w = tid >> 5, nw = nthreads >> 5;
  if (lane == 0) {
    red_m[0][w] = bphi;
    red_m[1][w] = bpsi;
    red_b[w] = bad;
  }
  __syncthreads();
  if (tid == 0) {
    for (int i = 1; i < nw; ++i) {
      bphi = max(bphi, red_m[0][i]);
      bpsi = max(bpsi, red_m[1][i]);
      bad += red_b[i];
    }
    if (bphi) atomicMax(&p.stats[0], bphi);
    if (bpsi) atomicMax(&p.stats[1], bpsi);
    if (bad) atomicAdd(&p.stats[2], (unsigned long long)bad);
  }
}

// One depth chunk [k0, k0 + kc) of ONE operand pair (Gauss segment) into ONE
// accumulator set: A rows from As, B rows from Bs (row stride kKS).
__device__ __forceinline__ void mma_chunk1(double (&acc)[kMT][4][4], const double* A, const double* B, int kc,
                                           int wm, int wn, int lr, int lk) {
#pragma unroll 4
  for (int kk = 0; kk < kc; kk += 4) {
    double ap[2][2], bf[4];
#pragma unroll
    for (int mt = 0; mt < kMT; ++mt) {
      const int r = wm * 16 * kMT + mt * 16 + lr;
      ap[mt][0] = A[r * kKS + kk + lk];
      ap[mt][1] = A[(r + 8) * kKS + kk + lk];
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[nt] = B[(wn * 32 + nt * 8 + lr) * kKS + kk + lk];
#pragma unroll
    for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma_16x8x4(acc[mt][nt], ap[mt][0], ap[mt][1], bf[nt]);
  }
}

// Two operand pairs, two accumulator sets, interleaved per k-step: 16
// independent DMMAs per warp and k-step.
__device__ __forceinline__ void mma_chunk2(double (&acc0)[kMT][4][4], double (&acc1)[kMT][4][4],
                                           const double* A0, const double* B0, const double* A1, const double* B1,
                                           int kc, int wm, int wn, int lr, int lk) {
#pragma unroll 2
  for (int kk = 0; kk < kc; kk += 4) {
    double a0[2][2], a1[2][2], b0[4], b1[4];
#pragma unroll
    for (int mt = 0; mt < kMT; ++mt) {
      const int r = wm * 16 * kMT + mt * 16 + lr;
      a0[mt][0] = A0[r * kKS + kk + lk];
      a0[mt][1] = A0[(r + 8) * kKS + kk + lk];
      a1[mt][0] = A1[r * kKS + kk + lk];
      a1[mt][1] = A1[(r + 8) * kKS + kk + lk];
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      b0[nt] = B0[(wn * 32 + nt * 8 + lr) * kKS + kk + lk];
      b1[nt] = B1[(wn * 32 + nt * 8 + lr) * kKS + kk + lk];
    }
#pragma unroll
    for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        dmma_16x8x4(acc0[mt][nt], a0[mt][0], a0[mt][1], b0[nt]);
        dmma_16x8x4(acc1[mt][nt], a1[mt][0], a1[mt][1], b1[nt]);
      }
  }
}

__device__ __forceinline__ int f64_dbg(const ContractParams& p) {
#ifdef CORR2D_PROFILING
  return p.dbg;
#else
  (void)p;
  return 0;
#endif
}

template <bool GAUSS>
__global__ void __launch_bounds__(kThreads, CORR2D_F64_MINB) contract_f64_kernel(const ContractParams p) {
  extern __shared__ __align__(16) double sm[];
  double* As = sm;                     // [kNBuf][kBM][kKS]  A_phi (buffer stride kBufStride)
  double* Ps = As + kBM * kKS;         // A_psi
  double* Bs = Ps + kBM * kKS;         // B

  int I, J, mode;
  decode_tile(p, I, J, mode);
  const int i0 = I * kBM, j0 = J * kBN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;   // rows wm * 16 MT .., columns wn * 32 ..
  const int lr = lane >> 2, lk = lane & 3;

  double acc_phi[kMT][4][4], acc_psi[kMT][4][4];
#pragma unroll
  for (int a = 0; a < kMT; ++a)
#pragma unroll
    for (int bq = 0; bq < 4; ++bq)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc_phi[a][bq][c] = acc_psi[a][bq][c] = 0.0;

  if constexpr (GAUSS) {
    // three products per bin (corr2d.h CORR2D_PACK_F64_GAUSS), 3 kg
    // multiply-adds per element instead of 2 m.  Phase A runs two independent
    // accumulator chains per k-step (DMMA latency hidden as in the four-product
    // kernel): segment 0 (P1) into the async set and segment 2 (-P3) into the
    // sync set; then sync += async gives P1 - P3, and phase B adds segment 1
    // (P2) to the async set: P1 + P2.
    constexpr int kTile = kBM * kKS;                 // doubles per operand tile
    auto issue = [&](int seg, int k0, int slot) {
      const int kc = min(kKC, p.kg - k0);
      const int vec = kc / 2;
      const int kbase = seg * p.kg + k0;
      double* A = sm + 2 * slot * kTile;
      double* B = A + kTile;
      for (int idx = tid; idx < kBM * vec; idx += kThreads) {
        const int r = kc == kKC ? idx / (kKC / 2) : idx / vec;
        const int v = idx - r * vec;
        const int gi = i0 + r, gj = j0 + r;
        const bool va = gi < p.n1, vb = gj < p.n2;
        cp_async16(A + r * kKS + 2 * v, p.a_phi + (long long)(va ? gi : 0) * p.ld_pack + kbase + 2 * v, va);
        cp_async16(B + r * kKS + 2 * v, p.b + (long long)(vb ? gj : 0) * p.ld_pack + kbase + 2 * v, vb);
      }
    };
    for (int k0 = 0; k0 < p.kg; k0 += kKC) {          // phase A: segments 0 and 2 together
      issue(0, k0, 0);
      issue(2, k0, 1);
      cp_async_wait_all();
      __syncthreads();
      const int kc = min(kKC, p.kg - k0);
      if (!(f64_dbg(p) & 2)) mma_chunk2(acc_psi, acc_phi, sm, sm + kTile, sm + 2 * kTile, sm + 3 * kTile, kc, wm, wn, lr, lk);
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < kMT; ++a)
#pragma unroll
      for (int bq = 0; bq < 4; ++bq)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc_phi[a][bq][c] += acc_psi[a][bq][c];
    for (int k0 = 0; k0 < p.kg; k0 += kKC) {          // phase B: segment 1
      issue(1, k0, 0);
      cp_async_wait_all();
      __syncthreads();
      if (!(f64_dbg(p) & 2)) mma_chunk1(acc_psi, sm, sm + kTile, min(kKC, p.kg - k0), wm, wn, lr, lk);
      __syncthreads();
    }
  } else {

  // depth chunks through NBUF shared-memory buffers (CORR2D_F64_NBUF = 2: the
  // next chunk's cp.async overlaps this chunk's DMMAs)
  auto issue = [&](int k0, int buf) {
    const int kc = min(kKC, p.mp - k0);  // multiple of 4
    const int vec = kc / 2;              // 16-byte chunks per row
    double* A = As + buf * kBufStride;
    double* Pq = Ps + buf * kBufStride;
    double* B = Bs + buf * kBufStride;
    for (int idx = tid; idx < kBM * vec; idx += kThreads) {
      // full chunks: vec = kKC / 2 is a power of two (shifts, not a division)
      const int r = kc == kKC ? idx / (kKC / 2) : idx / vec;
      const int v = idx - r * vec;
      const int gi = i0 + r, gj = j0 + r;
      const bool va = gi < p.n1, vb = gj < p.n2;
      const long long oa = (long long)(va ? gi : 0) * p.ld_pack + k0 + 2 * v;
      const long long ob = (long long)(vb ? gj : 0) * p.ld_pack + k0 + 2 * v;
      cp_async16(A + r * kKS + 2 * v, p.a_phi + oa, va);
      cp_async16(Pq + r * kKS + 2 * v, p.a_psi + oa, va);
      cp_async16(B + r * kKS + 2 * v, p.b + ob, vb);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  issue(0, 0);
  for (int k0 = 0, c = 0; k0 < p.mp; k0 += kKC, ++c) {
    const int kc = min(kKC, p.mp - k0);
    const int buf = c % kNBuf;
    if (kNBuf > 1 && k0 + kKC < p.mp) {
      issue(k0 + kKC, (c + 1) % kNBuf);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* A = As + buf * kBufStride;
    const double* Pq = Ps + buf * kBufStride;
    const double* B = Bs + buf * kBufStride;
#pragma unroll 4
    for (int kk = 0; kk < kc; kk += 4) {
      double ap[2][2], as[2][2], bf[4];
#pragma unroll
      for (int mt = 0; mt < kMT; ++mt) {
        const int r = wm * 16 * kMT + mt * 16 + lr;
        ap[mt][0] = A[r * kKS + kk + lk];
        ap[mt][1] = A[(r + 8) * kKS + kk + lk];
        as[mt][0] = Pq[r * kKS + kk + lk];
        as[mt][1] = Pq[(r + 8) * kKS + kk + lk];
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = B[(wn * 32 + nt * 8 + lr) * kKS + kk + lk];
#pragma unroll
      for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          dmma_16x8x4(acc_phi[mt][nt], ap[mt][0], ap[mt][1], bf[nt]);
          dmma_16x8x4(acc_psi[mt][nt], as[mt][0], as[mt][1], bf[nt]);
        }
    }
    if (kNBuf == 1 || k0 + kKC < p.mp) __syncthreads();   // buffer free before it is refilled
    if (kNBuf == 1 && k0 + kKC < p.mp) issue(k0 + kKC, 0);
  }
  }  // !GAUSS

#ifdef CORR2D_PROFILING
  if (p.dbg & 1) {                    // profiling: everything but the output stores
    unsigned long long z = 0;
    for (int a = 0; a < kMT; ++a)
      for (int b = 0; b < 4; ++b)
        for (int c = 0; c < 4; ++c) z ^= abs_bits(acc_phi[a][b][c]) ^ abs_bits(acc_psi[a][b][c]);
    if (z == 0x123456789ull) p.stats[3] = z;
    return;
  }
#endif
  // ---- epilogue.  Plain / mirrored tiles write their direct part straight
  //      from the DMMA fragments (a thread holds 2 adjacent columns of 2 rows:
  //      16-byte stores, 8 x 64-B row segments per warp instruction); the planes
  //      are staged in shared memory for the transposed mirror and for the
  //      symmetrised diagonal tiles, then written as coalesced rows ----
  const bool reg_direct = p.vec_direct && (mode == kPlain || mode == kMirror);
  unsigned long long dphi = 0, dpsi = 0;
  if (reg_direct) {
#pragma unroll
    for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gi = i0 + wm * 16 * kMT + mt * 16 + lr + 8 * h;
          const int gj = j0 + wn * 32 + nt * 8 + 2 * lk;
          if (gi >= p.row1 || gj >= p.n2) continue;
          const double f0 = acc_phi[mt][nt][2 * h], f1 = acc_phi[mt][nt][2 * h + 1];
          const double s0 = acc_psi[mt][nt][2 * h], s1 = acc_psi[mt][nt][2 * h + 1];
          const long long o = (long long)(gi - p.row0) * p.ld_out + gj;
          if (gj + 1 < p.n2) {
            __stcs(reinterpret_cast<double2*>(p.phi + o), make_double2(f0, f1));
            __stcs(reinterpret_cast<double2*>(p.psi + o), make_double2(s0, s1));
            dphi = max(dphi, max(absbits(f0), absbits(f1)));
            dpsi = max(dpsi, max(absbits(s0), absbits(s1)));
          } else {
            __stcs(p.phi + o, f0);
            __stcs(p.psi + o, s0);
            dphi = max(dphi, absbits(f0));
            dpsi = max(dpsi, absbits(s0));
          }
        }
#ifndef CORR2D_F64_REG_MIRROR
#define CORR2D_F64_REG_MIRROR 1
#endif
#if CORR2D_F64_REG_MIRROR
    // whole mirrored tile in bounds: the transpose also leaves straight from the
    // fragments (8-byte stores, 4 rows x 64 B per warp instruction) -- no
    // shared-memory staging, no barriers
    if (mode == kMirror && j0 >= p.row0 && j0 + kBN <= p.row1 && i0 + kBM <= p.n2) {
#pragma unroll
      for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gi = i0 + wm * 16 * kMT + mt * 16 + lr + 8 * h;
            const int gj = j0 + wn * 32 + nt * 8 + 2 * lk;
            const long long o = (long long)(gj - p.row0) * p.ld_out + gi;
            __stcs(p.phi + o, acc_phi[mt][nt][2 * h]);
            __stcs(p.psi + o, dneg(acc_psi[mt][nt][2 * h]));
            __stcs(p.phi + o + p.ld_out, acc_phi[mt][nt][2 * h + 1]);
            __stcs(p.psi + o + p.ld_out, dneg(acc_psi[mt][nt][2 * h + 1]));
          }
      write_tile(p, kPlain, i0, j0, nullptr, nullptr, tid, kThreads, lane, true, dphi, dpsi);
      return;
    }
#endif
    if (mode == kPlain) {       // nothing left to stage
      write_tile(p, kPlain, i0, j0, nullptr, nullptr, tid, kThreads, lane, true, dphi, dpsi);
      return;
    }
  }
  __syncthreads();
  double* Cphi = sm;                   // [kBM][kCS]
  double* Cpsi = sm + kBM * kCS;       // [kBM][kCS]
#pragma unroll
  for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int r = wm * 16 * kMT + mt * 16 + lr;
      const int c = wn * 32 + nt * 8 + 2 * lk;
      Cphi[r * kCS + c] = acc_phi[mt][nt][0];
      Cphi[r * kCS + c + 1] = acc_phi[mt][nt][1];
      Cphi[(r + 8) * kCS + c] = acc_phi[mt][nt][2];
      Cphi[(r + 8) * kCS + c + 1] = acc_phi[mt][nt][3];
      Cpsi[r * kCS + c] = acc_psi[mt][nt][0];
      Cpsi[r * kCS + c + 1] = acc_psi[mt][nt][1];
      Cpsi[(r + 8) * kCS + c] = acc_psi[mt][nt][2];
      Cpsi[(r + 8) * kCS + c + 1] = acc_psi[mt][nt][3];
    }
  __syncthreads();

  write_tile(p, mode, i0, j0, Cphi, Cpsi, tid, kThreads, lane, reg_direct, dphi, dpsi);
}

}  // namespace corr2d

using namespace corr2d;

static int launch_contract(ContractParams p, bool gauss, int64_t tile0, int64_t tile1, void* stream,
                           const char* who) {
  long long tiles;
  const long long R = p.I1 - p.I0;
  if (p.homo) tiles = R * p.T - R * (R - 1) / 2;   // sum_{d<R} (T - d)
  else tiles = R * p.T;
  if (tile1 < 0 || tile1 > tiles) tile1 = tiles;
  if (tile0 < 0 || tile0 > tile1) return fail(CORR2D_ERR_DATA, std::string(who) + ": bad tile range");
  p.tile0 = tile0;
#ifdef CORR2D_PROFILING
  if (const char* e = getenv("CORR2D_DEBUG_SKIP")) p.dbg = atoi(e);
#endif
  tiles = tile1 - tile0;
  if (tiles > 0x7fffffffLL) return fail(CORR2D_ERR_UNSUPPORTED, std::string(who) + ": tile count out of range");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(p.stats, 0, 3 * sizeof(unsigned long long), st) != cudaSuccess) return check_launch("stats reset");
  if (tiles == 0) return CORR2D_OK;
  const size_t smem_ops = gauss ? (size_t)4 * kBM * kKS * sizeof(double) : (size_t)kNBuf * kBufStride * sizeof(double);  // gauss: A0 B0 A2 B2
  const size_t smem_epi = 2 * (size_t)kBM * kCS * sizeof(double);
  const size_t smem = smem_ops > smem_epi ? smem_ops : smem_epi;
  if (gauss) {
    cudaFuncSetAttribute(contract_f64_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    contract_f64_kernel<true><<<(unsigned)tiles, kThreads, smem, st>>>(p);
    return check_launch("contract_f64_kernel<gauss>");
  }
  cudaFuncSetAttribute(contract_f64_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  contract_f64_kernel<false><<<(unsigned)tiles, kThreads, smem, st>>>(p);
  return check_launch("contract_f64_kernel");
}

static int check_common(const char* who, int n1, int n2, int homo, int row0, int row1, int64_t ld_out) {
  if (n1 < 1 || n2 < 1) return fail(CORR2D_ERR_DATA, std::string(who) + ": bad sizes");
  if (row0 < 0 || row1 > n1 || row0 >= row1) return fail(CORR2D_ERR_DATA, std::string(who) + ": bad row range");
  if (ld_out < n2) return fail(CORR2D_ERR_DATA, std::string(who) + ": ld_out < n2");
  if (homo && n1 != n2) return fail(CORR2D_ERR_DATA, std::string(who) + ": homo needs n1 == n2");
  if (row0 % kBM != 0 || (row1 != n1 && row1 % kBM != 0))
    return fail(CORR2D_ERR_DATA, std::string(who) + ": row shard bounds must be multiples of 64 (or n1)");
  return CORR2D_OK;
}

static ContractParams make_params(int n1, int n2, int homo, int row0, int row1, double* phi, double* psi,
                                  int64_t ld_out, unsigned long long* stats) {
  ContractParams p{};
  p.n1 = n1; p.n2 = n2; p.homo = homo; p.row0 = row0; p.row1 = row1;
  p.I0 = row0 / kBM; p.I1 = (row1 + kBM - 1) / kBM; p.T = (n2 + kBN - 1) / kBN;
  p.phi = phi; p.psi = psi; p.ld_out = ld_out; p.stats = stats;
  p.vec_direct = (ld_out % 2 == 0) && ((reinterpret_cast<uintptr_t>(phi) | reinterpret_cast<uintptr_t>(psi)) & 15) == 0;
  return p;
}

extern "C" int corr2d_contract_f64(
    const double* a_phi, const double* a_psi, const double* b, int64_t ld_pack,
    int n1, int n2, int mp, int homo, int row0, int row1, int64_t tile0, int64_t tile1,
    double* phi, double* psi, int64_t ld_out, unsigned long long* stats, void* stream) {
  if (!a_phi || !a_psi || !b || !phi || !psi || !stats)
    return fail(CORR2D_ERR_DATA, "corr2d_contract_f64: null pointer");
  if (mp < 4 || (mp % 4) != 0)
    return fail(CORR2D_ERR_DATA, "corr2d_contract_f64: bad sizes (mp must be a positive multiple of 4)");
  if (ld_pack < mp || (ld_pack % 2) != 0)
    return fail(CORR2D_ERR_DATA, "corr2d_contract_f64: ld_pack must be even and >= mp");
  if (int rc = check_common("corr2d_contract_f64", n1, n2, homo, row0, row1, ld_out)) return rc;
  ContractParams p = make_params(n1, n2, homo, row0, row1, phi, psi, ld_out, stats);
  p.a_phi = a_phi; p.a_psi = a_psi; p.b = b; p.ld_pack = ld_pack; p.mp = mp;
  return launch_contract(p, false, tile0, tile1, stream, "corr2d_contract_f64");
}

extern "C" int corr2d_contract_f64_gauss(
    const double* a, const double* b, int64_t ld_pack, int n1, int n2, int kg, int homo,
    int row0, int row1, int64_t tile0, int64_t tile1,
    double* phi, double* psi, int64_t ld_out, unsigned long long* stats, void* stream) {
  if (!a || !b || !phi || !psi || !stats) return fail(CORR2D_ERR_DATA, "corr2d_contract_f64_gauss: null pointer");
  if (kg < 4 || (kg % 4) != 0)
    return fail(CORR2D_ERR_DATA, "corr2d_contract_f64_gauss: kg must be a positive multiple of 4");
  if (ld_pack < 3LL * kg || (ld_pack % 2) != 0)
    return fail(CORR2D_ERR_DATA, "corr2d_contract_f64_gauss: ld_pack must be even and >= 3 kg");
  if (int rc = check_common("corr2d_contract_f64_gauss", n1, n2, homo, row0, row1, ld_out)) return rc;
  ContractParams p = make_params(n1, n2, homo, row0, row1, phi, psi, ld_out, stats);
  p.a_phi = a; p.a_psi = a; p.b = b; p.ld_pack = ld_pack; p.mp = 3 * kg; p.kg = kg;
  return launch_contract(p, true, tile0, tile1, stream, "corr2d_contract_f64_gauss");
}
