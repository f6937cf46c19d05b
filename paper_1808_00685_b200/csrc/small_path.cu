// The whole small-m correlation (corr2d_correlate_small_f64): fp64,
// 2 <= m <= 32, no resampling -- the cfg1 (m = 11) and cfg2 (m = 21) shapes,
// where a step is bound by latency, one DRAM round trip and the output write
// (cfg1: 16 MB of planes, cfg2: 48 MB).  Every kernel here is launched with
// programmatic dependent launch.  Single calls order memory with
// griddepcontrol.wait; pipelined calls (corr2d_correlate_small_f64_slot) with
// monotonic tickets (see kPClaim below).
//
// Calls without operand scratch: small_fused_kernel -- ONE kernel: each CTA
//   centres its blocks' channels, builds their Gauss operand rows with one
//   FP64 tensor-core product per role, contracts them and writes both planes
//   (+ the homo mirror) by TMA tensor stores.
// Otherwise (the default) two kernels.
//   small_rows_kernel -- K1 once per channel: 64 channels per CTA, the
//   reference's statistics in its order (one lane per channel, sequential
//   sums: bitwise-equal reference / sigma / values), then the
//   CORR2D_PACK_F64_GAUSS operand rows of every role as ONE FP64 tensor-core
//   product (the rfft rows already combined into the Gauss slots), copied out
//   by one bulk copy per warp and role.  It only reads global memory before
//   its griddepcontrol.wait, so it overlaps the previous call's contraction.
//   small_stream_kernel -- persistent contraction, two CTAs per SM, each
//   walking a contiguous run of 64 x 64 blocks: operand rows by cp.async
//   (issued as soon as the block's DMMAs have read the buffer), the Gauss
//   contraction with two accumulator chains, both planes staged swizzled and
//   written by TMA tensor stores issued by one thread (no warp waits on its
//   own stores); max|.| / finite folded into the fragments.
//   small_contract_kernel -- one CTA per block with plain stores, for planes
//   that are not 16-B aligned with an even row pitch.
// Status / stat words are self-resetting.  Within one call no CTA waits for
// another; pipelined calls (corr2d_correlate_small_f64_slot) order themselves
// through monotonic tickets, waiting only on grids whose CTAs are resident.
//
// Reference path: preprocess.py:123-137, :198-259 (reference, sigma, scaling),
// fourier.py:61-82 (rfft along the perturbation axis), fourier.py:107-123
// (weighted half-spectrum cross sum x Norm, split into sync / async),
// engine_core.py:139-140 (finite check), dataset.py:159-170 (homo symmetry).
#include "prep_params.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <string>
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
  int mpad;                 // m rounded up to 4 (the DMMA k-step); samples past m are 0
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
  long long tiles;          // streamed contraction: 64 x 64 blocks, CTAs, 64-KB staging slots
  int nctas, nslots;
  int dbg;                  // profiling builds only (CORR2D_DEBUG_SKIP): 1 no stores, 2 no DMMAs
  int tma_ops;              // streamed contraction, one buffer: operand rows by bulk copy (else cp.async)
  const double* G;          // small_rows_kernel: [2][nsp][gp] Gauss-row table (fused_table), gp = mpad + 2
  int slot;                 // pipelined calls: this call's scratch slot (0 / 1) ...
  unsigned long long* pipe; // ... and the plan's uint64[16] pipeline words (kP*; NULL: not pipelined)
  int k1_ctas;              // pipelined calls: K1's grid (every K1 CTA takes one ticket per counter)
};

// Pipelined calls (corr2d_correlate_small_f64_slot with a pipe): consecutive
// calls of one plan alternate between two scratch slots (operand rows, stats,
// work and status words), and no kernel waits for a whole earlier grid
// (griddepcontrol.wait would: a grid launched early still completes in stream
// order, so the next call could never overlap this one).  Ordering comes from
// monotonic 64-bit counters instead (uint64 words of the plan's pipe).  A
// kernel's CTAs take their tickets BEFORE griddepcontrol.launch_dependents, so
// all of a call's tickets precede the next call's, and ticket / (grid CTAs) is
// the call's index on that counter:
//   kPClaim + s   K1 tickets on slot s -> use index u of the slot;
//   kPGen + s     completed uses of slot s: K1 writes its slot only when it
//                 equals u (the slot's previous user has finished with it);
//   kPReady + s   K1 CTAs of slot s that have written their rows, statistics
//                 and status words (never reset): use u of the slot is
//                 complete at (K1 CTAs) * (u + 1);
//   kPSClaim + s  contraction tickets on slot s -> its use index, so it waits
//                 for ITS K1 (not a stale count of the slot's previous use);
//   kPSCall       contraction tickets on the plan -> call index c;
//   kPPlanes      calls whose contraction has completed all its stores: a
//                 contraction issues its first store only when it equals c
//                 (every call writes the same planes: they land in call order);
//   kPArrive + s  contraction CTAs done; the last one advances kPGen + s and
//                 kPPlanes.
// Every wait is on a grid whose CTAs have all passed
// griddepcontrol.launch_dependents, i.e. are resident (or done), so it cannot
// wait for a CTA that is not running.  A wait that outlives ~8 s gives up and
// flags the call (stats[2], the non-finite-output count).
constexpr int kPClaim = 0, kPGen = 2, kPReady = 4, kPSClaim = 6, kPSCall = 8, kPPlanes = 9, kPArrive = 10;
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* w) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];\n" : "=l"(v) : "l"(w) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* w, unsigned long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;\n" ::"l"(w), "l"(v) : "memory");
}
__device__ __noinline__ void pipe_wait_at_least(const SmallParams& p, const unsigned long long* w,
                                                unsigned long long value) {
  for (long long i = 0; i < (1LL << 23); ++i) {
    if (ld_acquire(w) >= value) return;
    __nanosleep(64);
  }
  atomicAdd(&p.stats[2], 1ull);                        // never expected: the call reports bad output
}
// counters only grow: "equals" is "reached"
__device__ __forceinline__ void pipe_wait_value(const SmallParams& p, const unsigned long long* w,
                                                unsigned long long value) {
  pipe_wait_at_least(p, w, value);
}
// The last CTA of a pipelined contraction, once every CTA's stores have
// performed: one more completed use of the slot and one more completed call.
__device__ __forceinline__ void pipe_release(const SmallParams& p, int tid, unsigned long long call) {
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;\nfence.proxy.async.global;\n" ::: "memory");
  __threadfence();
  __syncthreads();
  if (tid == 0 && atomicAdd(p.pipe + kPArrive + p.slot, 1ull) == (unsigned long long)p.nctas - 1) {
    p.pipe[kPArrive + p.slot] = 0;
    __threadfence();
    atomicAdd(p.pipe + kPGen + p.slot, 1ull);
    __threadfence();
    st_release(p.pipe + kPPlanes, call + 1);
  }
}

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
// kernels in the reference's order.  No global writes (K1 computes before its
// griddepcontrol.wait); lane_report publishes the channel's status /
// reference / sigma afterwards.
struct LaneStat {
  double ref, sigma;
  int bad;
};
template <int kYS>                                     // the column's sample pitch (doubles)
__device__ __forceinline__ LaneStat lane_stats(const SmallParams& p, int set, int c, bool valid, double* ys) {
  const int m = p.m;
  const int ref_mode = set ? p.ref_mode2 : p.ref_mode1;
  LaneStat st{0.0, 0.0, 0};
  double ref = 0.0, scale = 1.0;
  int bad = 0;
  double sum = 0.0;                                    // left to right (numpy's axis-0 order)
#pragma unroll 4
  for (int t = 0; t < m; ++t) {
    const double v = ys[t * kYS];
    bad += !isfinite(v);
    sum = __dadd_rn(sum, v);
  }
  st.bad = bad;
  if (ref_mode == CORR2D_REF_PROVIDED) {
    ref = valid ? __ldg((set ? p.ref_in2 : p.ref_in1) + c) : 0.0;
  } else if (ref_mode == CORR2D_REF_MEAN) {
    ref = __ddiv_rn(sum, (double)m);
  }
  st.ref = ref;
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
    st.sigma = sigma;
    if (sigma == 0.0 && p.substitute) sigma = 1.0;
    scale = (p.alpha == 0.5) ? __dsqrt_rn(sigma) : (p.alpha == 1.0 ? sigma : pow(sigma, p.alpha));
  }
  const bool sub = ref_mode != CORR2D_REF_NONE, div = p.alpha > 0.0;
  if (!div) {
#pragma unroll 4
    for (int t = 0; t < m; ++t) {
      const double v = ys[t * kYS];
      ys[t * kYS] = valid ? (sub ? __dsub_rn(v, ref) : v) : 0.0;
    }
    return st;
  }
  for (int t = 0; t < m; ++t) {
    double v = ys[t * kYS];
    if (sub) v = __dsub_rn(v, ref);
    v = __ddiv_rn(v, scale);
    ys[t * kYS] = valid ? v : 0.0;
  }
  return st;
}

// The channel's status words, sigma and reference (after griddepcontrol.wait).
__device__ __forceinline__ void lane_report(const SmallParams& p, int set, int c, const LaneStat& st) {
  int* status = p.work + (set ? kWStatus2 : kWStatus1);
  if (st.bad) atomicAdd(&status[CORR2D_ST_NONFINITE], st.bad);
  if (p.alpha > 0.0) {
    double* so = set ? p.sigma_out2 : p.sigma_out1;
    if (so) so[c] = st.sigma;
    if (st.sigma == 0.0) {
      atomicAdd(&status[CORR2D_ST_ZEROVAR], 1);
      atomicMax(&status[CORR2D_ST_FIRST_ZEROVAR], INT_MAX - c);
    }
  }
  if ((set ? p.ref_mode2 : p.ref_mode1) != CORR2D_REF_NONE) {
    double* ro = set ? p.ref_out2 : p.ref_out1;
    if (ro) ro[c] = st.ref;
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

// =====================================================================
// The fused small-m path (default): ONE persistent kernel, no operand rows in
// global memory and no kernel boundary between the per-channel work and the
// contraction.  CTA c owns a contiguous run of the 64 x 64 output blocks
// (homo: the upper triangle, row by row) and, per block,
//   * loads the raw samples of the block's 64 row channels (only when the
//     row block changes) and 64 column channels (cp.async, prefetched during
//     the previous block's contraction),
//   * centres / scales them in the reference's order (lane per channel),
//   * turns them into the CORR2D_PACK_F64_GAUSS operand rows with ONE FP64
//     tensor-core product per role: rows[ch][s] = sum_t y[t][ch] G[s][t], G the
//     DFT rows already combined into the three Gauss segments (the rfft of
//     fourier.py:73 and the slot algebra of gauss_values, folded on the host),
//   * contracts them (two accumulator chains) and stages both planes in shared
//     memory, from where they leave by bulk asynchronous copies (one per row):
//     no warp ever waits on its own output stores, so the next block's loads,
//     centring and DMMAs overlap the previous block's HBM write stream.
// Status / stat words: owner CTAs (tile (I, first column) for the rows, tile
// (0, J) for a hetero column block) report each channel's status once; the
// last CTA to arrive (an arrival counter, never a wait) publishes and
// re-zeroes the accumulators.
// =====================================================================
constexpr int kFYP = 68;   // sample pitch (doubles): [t][64 channels + 4]
constexpr int kWFStat1 = 0, kWFStat2 = 4, kWFAcc = 8 /* 3 x u64 at byte 32 */, kWFCount = 14;

struct FusedParams {
  const void* raw1;
  const void* raw2;
  long long ld1, ld2;
  int in_f32;
  int al1, al2;             // fp64 rows of raw1 / raw2 16-B aligned (16-byte sample copies)
  int mirror_buf;           // homo: a second staging buffer for the mirrored block
  int m, mpad, gp, n1, n2, homo;
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
  const double* G;          // [2][nsp][gp]: role-A rows (x Norm in the kernel), then role-B rows
  int kg, ns, nsp, ks;      // Gauss slots per segment, 3 kg, 3 kg rounded to 8, operand row pitch
  int T1, T2;
  long long tiles;
  int nctas;
  double* phi;
  double* psi;
  long long ld_out;
  int vec;
  int* status1;
  int* status2;
  unsigned long long* stats;
  int* work;
  unsigned long long* trace;
};

__device__ __forceinline__ void fused_decode(const FusedParams& p, long long b, int& I, int& J) {
  if (!p.homo) {
    I = (int)(b / p.T2);
    J = (int)(b - (long long)I * p.T2);
    return;
  }
  const long long T = p.T1;
  const long long t2 = 2 * T + 1;
  const long long disc = t2 * t2 - 8 * b;
  long long d = (long long)((float)t2 - sqrtf((float)(disc > 0 ? disc : 0))) / 2;
  auto S = [&](long long dd) { return dd * T - dd * (dd - 1) / 2; };
  if (d < 0) d = 0;
  while (d > 0 && S(d) > b) --d;
  while (S(d + 1) <= b) ++d;
  I = (int)d;
  J = I + (int)(b - S(d));
}

// first tile of row block I in the enumeration (homo: the diagonal block)
__device__ __forceinline__ long long fused_row_start(const FusedParams& p, int I) {
  const long long d = I;
  return p.homo ? d * p.T1 - d * (d - 1) / 2 : d * p.T2;
}

#ifdef CORR2D_PROFILING
#define FUSED_STAMP(k)                                                                         \
  do {                                                                                         \
    if (p.trace && threadIdx.x == 0) {                                                         \
      unsigned long long t_;                                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
      p.trace[16 * blockIdx.x + (k)] = t_;                                                     \
    }                                                                                          \
  } while (0)
#else
#define FUSED_STAMP(k) do { } while (0)
#endif

// Raw samples of 64 channels [c0, c0 + 64) of dataset `set` -> ys[t][ch]
// (cp.async, zero-filled past n; fp32 inputs land in the low half of the slot).
__device__ __forceinline__ void fused_load(const FusedParams& p, int set, int c0, double* ys) {
  const int n = set ? p.n2 : p.n1;
  const long long ld = set ? p.ld2 : p.ld1;
  const void* raw = set ? p.raw2 : p.raw1;
  const int tid = threadIdx.x;
  if (!p.in_f32 && (set ? p.al2 : p.al1) && c0 + 64 <= n) {
    // whole block, 16-B aligned rows: a thread copies channel pairs of rows t, t + 4, ...
    const double* src = static_cast<const double*>(raw) + c0 + 2 * (tid & 31) + (long long)(tid >> 5) * ld;
    unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(ys + 2 * (tid & 31) + (tid >> 5) * kFYP));
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
#pragma unroll 1
    for (int t = tid >> 5; t < p.m; t += 4, src += 4 * ld, dst += 8u * 4 * kFYP)
      asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "l"(pol)
                   : "memory");
  } else {
    const int total = p.m * 64;
#pragma unroll 1
    for (int idx = tid; idx < total; idx += kSThreads) {
      const int t = idx >> 6, ch = idx & 63, c = c0 + ch;
      const bool v = c < n;
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(ys + t * kFYP + ch));
      if (p.in_f32) {
        const float* src = static_cast<const float*>(raw) + (long long)t * ld + (v ? c : 0);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 4 : 0) : "memory");
      } else {
        const double* src = static_cast<const double*>(raw) + (long long)t * ld + (v ? c : 0);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0) : "memory");
      }
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// One channel's statistics and dynamic values in place in its column
// ys[t * kFYP] -- the IEEE operations of the other K1 kernels in the
// reference's order (preprocess.py:123-137, :198-259).  The owner lane reports
// status / reference / sigma.
__device__ __noinline__ void fused_f32_column(double* ys, int m) {
  for (int t = 0; t < m; ++t) ys[t * kFYP] = (double)reinterpret_cast<const float*>(ys + t * kFYP)[0];
}

// sigma about ref (preprocess.py:198-211) -> the division scale sigma**alpha
// (:214-259), in place; the owner lane reports sigma and zero variance.
__device__ __noinline__ void fused_scale_column(const FusedParams& p, int set, int c, bool valid, bool report,
                                                double ref, bool sub, double* ys) {
  const int m = p.m;
  const double* sigma_in = set ? p.sigma_in2 : p.sigma_in1;
  int* status = p.work + (set ? kWFStat2 : kWFStat1);
  double sigma;
  if (sigma_in) {
    sigma = valid ? __ldg(sigma_in + c) : 1.0;
  } else {
    double ss = 0.0;
    for (int t = 0; t < m; ++t) {
      const double d = __dsub_rn(ys[t * kFYP], ref);
      ss = __dadd_rn(ss, __dmul_rn(d, d));
    }
    sigma = __dsqrt_rn(__ddiv_rn(ss, (double)(m - 1)));
  }
  if (report) {
    double* so = set ? p.sigma_out2 : p.sigma_out1;
    if (so) so[c] = sigma;
    if (sigma == 0.0) {
      atomicAdd(&status[CORR2D_ST_ZEROVAR], 1);
      atomicMax(&status[CORR2D_ST_FIRST_ZEROVAR], INT_MAX - c);
      __threadfence();
    }
  }
  if (sigma == 0.0 && p.substitute) sigma = 1.0;
  const double scale = (p.alpha == 0.5) ? __dsqrt_rn(sigma) : (p.alpha == 1.0 ? sigma : pow(sigma, p.alpha));
  for (int t = 0; t < m; ++t) {
    double v = ys[t * kFYP];
    if (sub) v = __dsub_rn(v, ref);
    ys[t * kFYP] = valid ? __ddiv_rn(v, scale) : 0.0;
  }
}

// One channel's statistics and dynamic values in place in its column
// ys[t * kFYP] -- the IEEE operations of the other K1 kernels in the
// reference's order (preprocess.py:123-137, :198-259).  The owner lane reports
// status / reference / sigma.  Scaling and fp32 inputs are out of line.
__device__ __forceinline__ void fused_stats(const FusedParams& p, int set, int c, bool valid, bool owner,
                                            double* ys) {
  const int m = p.m;
  if (p.in_f32) fused_f32_column(ys, m);
  const int ref_mode = set ? p.ref_mode2 : p.ref_mode1;
  double ref = 0.0;
  int bad = 0;
  double sum = 0.0;                                    // left to right (numpy's axis-0 order)
#pragma unroll 4
  for (int t = 0; t < m; ++t) {
    const double v = ys[t * kFYP];
    bad += (unsigned)(__double2hiint(v) & 0x7ff00000) == 0x7ff00000u;   // !isfinite, integer pipe
    sum = __dadd_rn(sum, v);
  }
  const bool report = owner && valid;
  if (report && bad) {
    atomicAdd(&p.work[(set ? kWFStat2 : kWFStat1) + CORR2D_ST_NONFINITE], bad);
    __threadfence();
  }
  if (ref_mode == CORR2D_REF_PROVIDED) {
    ref = valid ? __ldg((set ? p.ref_in2 : p.ref_in1) + c) : 0.0;
  } else if (ref_mode == CORR2D_REF_MEAN) {
    ref = __ddiv_rn(sum, (double)m);
  }
  if (report && ref_mode != CORR2D_REF_NONE) {
    double* ro = set ? p.ref_out2 : p.ref_out1;
    if (ro) ro[c] = ref;
  }
  const bool sub = ref_mode != CORR2D_REF_NONE;
  if (p.alpha > 0.0) {
    fused_scale_column(p, set, c, valid, report, ref, sub, ys);
    return;
  }
#pragma unroll 4
  for (int t = 0; t < m; ++t) {
    const double v = ys[t * kFYP];
    ys[t * kFYP] = valid ? (sub ? __dsub_rn(v, ref) : v) : 0.0;
  }
}

// Compile-time shape of the Gauss rows for KG slots per segment (KG = gauss_kg(m)
// in {4, 8, 12, 16}): NS = 3 KG slots, padded to NSP (whole 8-column DMMA tiles),
// operand row pitch KS = NSP + 4 doubles (conflict-free fragment loads).
// Row pitch (doubles) of the small path's Gauss operand rows in global and
// shared memory: 3 kg slots, padded to 4 or 12 mod 16 (conflict-free DMMA
// fragment loads straight from the dense rows)
__host__ __device__ constexpr int small_ops_pitch(int kg) { return 3 * kg + ((3 * kg) % 16 == 0 || (3 * kg) % 16 == 8 ? 4 : 0); }

template <int KG>
struct FShape {
  static constexpr int NS = 3 * KG, NSP = (NS + 7) / 8 * 8, NNT = NSP / 8, KS = NSP + 4;
};

// Gauss operand rows of 64 channels: out[ch][s] = scale * sum_t ys[t][ch] G[s][t]
// on the FP64 tensor pipe (warp w: channels 16 w .. 16 w + 15, all slots).
template <int KG>
__device__ __forceinline__ void fused_transform(int mpad, int gp, const double* ys, const double* Gt, double* out,
                                                double scale, int warp, int lr, int lk) {
  using S = FShape<KG>;
  double acc[S::NNT][4];
#pragma unroll
  for (int a = 0; a < S::NNT; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[a][q] = 0.0;
  const int ch = 16 * warp + lr;
  const double* y = ys + lk * kFYP + ch;
  const double* g = Gt + lr * gp + lk;
#pragma unroll 2
  for (int kk = 0; kk < mpad; kk += 4) {
    const double a0 = y[kk * kFYP];
    const double a1 = y[kk * kFYP + 8];
#pragma unroll
    for (int nt = 0; nt < S::NNT; ++nt) dmma(acc[nt], a0, a1, g[nt * 8 * gp + kk]);
  }
#pragma unroll
  for (int nt = 0; nt < S::NNT; ++nt) {
    const int c = nt * 8 + 2 * lk;
    *reinterpret_cast<double2*>(out + ch * S::KS + c) = make_double2(acc[nt][0] * scale, acc[nt][1] * scale);
    *reinterpret_cast<double2*>(out + (ch + 8) * S::KS + c) = make_double2(acc[nt][2] * scale, acc[nt][3] * scale);
  }
}

// Both roles at once (independent accumulator chains interleaved): A rows
// (x scaleA) from ysA, B rows from ysB.
template <int KG>
__device__ __forceinline__ void fused_transform2(int mpad, int gp, const double* ysA, const double* GA, double* outA,
                                                 double scaleA, const double* ysB, const double* GB, double* outB,
                                                 int warp, int lr, int lk) {
  using S = FShape<KG>;
  double acc[2][S::NNT][4];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int a = 0; a < S::NNT; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][a][q] = 0.0;
  const int ch = 16 * warp + lr;
  const double* ya = ysA + lk * kFYP + ch;
  const double* yb = ysB + lk * kFYP + ch;
  const double* ga = GA + lr * gp + lk;
  const double* gb = GB + lr * gp + lk;
#pragma unroll 1
  for (int kk = 0; kk < mpad; kk += 4) {
    const double a0 = ya[kk * kFYP], a1 = ya[kk * kFYP + 8];
    const double c0 = yb[kk * kFYP], c1 = yb[kk * kFYP + 8];
#pragma unroll
    for (int nt = 0; nt < S::NNT; ++nt) {
      dmma(acc[0][nt], a0, a1, ga[nt * 8 * gp + kk]);
      dmma(acc[1][nt], c0, c1, gb[nt * 8 * gp + kk]);
    }
  }
#pragma unroll
  for (int nt = 0; nt < S::NNT; ++nt) {
    const int c = nt * 8 + 2 * lk;
    *reinterpret_cast<double2*>(outA + ch * S::KS + c) = make_double2(acc[0][nt][0] * scaleA, acc[0][nt][1] * scaleA);
    *reinterpret_cast<double2*>(outA + (ch + 8) * S::KS + c) = make_double2(acc[0][nt][2] * scaleA, acc[0][nt][3] * scaleA);
    *reinterpret_cast<double2*>(outB + ch * S::KS + c) = make_double2(acc[1][nt][0], acc[1][nt][1]);
    *reinterpret_cast<double2*>(outB + (ch + 8) * S::KS + c) = make_double2(acc[1][nt][2], acc[1][nt][3]);
  }
}

// KG/4 k-steps of one Gauss segment into one accumulator set (32 x 32 warp tile).
template <int KG, int KS = FShape<KG>::KS>
__device__ __forceinline__ void fused_seg1(double (&acc)[2][4][4], const double* A, const double* B) {
#pragma unroll
  for (int kk = 0; kk < KG; kk += 4) {
    double ap[2][2], bf[4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      ap[mt][0] = A[(mt * 16) * KS + kk];
      ap[mt][1] = A[(mt * 16 + 8) * KS + kk];
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[nt] = B[(nt * 8) * KS + kk];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], ap[mt][0], ap[mt][1], bf[nt]);
  }
}
// Two segments (operand offsets o0 / o1) into two accumulator sets, interleaved:
// 16 independent DMMAs per warp and k-step.
template <int KG, int KS = FShape<KG>::KS>
__device__ __forceinline__ void fused_seg2(double (&acc0)[2][4][4], double (&acc1)[2][4][4], const double* A,
                                           const double* B, int o0, int o1) {
#pragma unroll
  for (int kk = 0; kk < KG; kk += 4) {
    double a0[2][2], a1[2][2], b0[4], b1[4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      a0[mt][0] = A[(mt * 16) * KS + o0 + kk];
      a0[mt][1] = A[(mt * 16 + 8) * KS + o0 + kk];
      a1[mt][0] = A[(mt * 16) * KS + o1 + kk];
      a1[mt][1] = A[(mt * 16 + 8) * KS + o1 + kk];
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      b0[nt] = B[(nt * 8) * KS + o0 + kk];
      b1[nt] = B[(nt * 8) * KS + o1 + kk];
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

// Staging of one 64 x 64 fp64 plane as the four 64-row x 16-column boxes of a
// SWIZZLE_128B tensor map (box q = columns 16 q .. 16 q + 15; the 16-byte
// chunk of each 128-B box row XORed with the row): conflict-free fragment
// writes, and one TMA tensor store per box.
__device__ __forceinline__ int swz(int r, int c) {
  return ((c >> 4) << 10) + (r << 4) + ((((c >> 1) & 7) ^ (r & 7)) << 1) + (c & 1);
}

// The planes stream out with an evict-first L2 policy, so they do not push the
// raw samples (re-read by every block of a row / column) out of L2.
__device__ __forceinline__ void tma_store_box(const CUtensorMap* map, unsigned src, int col, int row, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;\n"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(row), "r"(src), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }

// Both staged planes (8 boxes at shared address S) -> output rows r0..,
// columns c0.. (TMA clips the boxes at the map's edges).  One thread.
__device__ __forceinline__ void fused_store_tile(const CUtensorMap* mphi, const CUtensorMap* mpsi, unsigned S,
                                                 int r0, int c0) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    tma_store_box(mphi, S + q * 8192, c0 + 16 * q, r0, pol);
    tma_store_box(mpsi, S + 32768 + q * 8192, c0 + 16 * q, r0, pol);
  }
  bulk_commit();
}

// max |.| bit patterns over the in-map fragment elements of an edge or
// diagonal block (diagonal: r <= c for sync, r < c for async).
__device__ __forceinline__ void fused_max_edge(const double (&aphi)[2][4][4], const double (&apsi)[2][4][4], int rows,
                                            int cols, bool diag, int wm, int wn, int lr, int lk,
                                            unsigned long long& mphi, unsigned long long& mpsi) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = wm * 32 + mt * 16 + lr + 8 * (q >> 1), c = wn * 32 + nt * 8 + 2 * lk + (q & 1);
        const bool in = r < rows && c < cols;
        const unsigned long long f = abs_bits(aphi[mt][nt][q]), s = abs_bits(apsi[mt][nt][q]);
        if (in && (!diag || r <= c)) mphi = max(mphi, f);
        if (in && (!diag || r < c)) mpsi = max(mpsi, s);
      }
}

__device__ __noinline__ void fused_publish(const FusedParams& p, unsigned long long mphi, unsigned long long mpsi,
                                           int lane, int warp, int tid);

template <int KG>
__global__ void __launch_bounds__(kSThreads, 1)
small_fused_kernel(const __grid_constant__ FusedParams p, const __grid_constant__ CUtensorMap map_phi,
                   const __grid_constant__ CUtensorMap map_psi) {
  using SH = FShape<KG>;
  constexpr int KS = SH::KS;
  extern __shared__ __align__(1024) double sm_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  const int wm = warp >> 1, wn = warp & 1;
  // staging first, at a 1024-B boundary (SWIZZLE_128B boxes); every region is
  // an offset into the shared array (shared-window loads and stores, no
  // generic addressing)
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(sm_raw));
  double* Cst = sm_raw + (((1024u - (sbase & 1023u)) & 1023u) >> 3);
  const unsigned cst_s = static_cast<unsigned>(__cvta_generic_to_shared(Cst));
  double* const Cmir = Cst + 8192;                     // mirror staging (homo, when it fits)
  const unsigned cmir_s = cst_s + 65536u;
  const int gp = p.gp, mpad = p.mpad;
  double* Gs = Cst + (p.mirror_buf ? 16384 : 8192);    // [2][NSP][gp]
  double* YA = Gs + 2 * SH::NSP * gp;                  // [mpad][kFYP]
  double* YB = YA + mpad * kFYP;
  double* As = YB + mpad * kFYP;                       // [64][KS]
  double* Bs = As + 64 * KS;
  const long long b0 = (long long)blockIdx.x * p.tiles / p.nctas;
  const long long b1 = (long long)(blockIdx.x + 1) * p.tiles / p.nctas;
  FUSED_STAMP(0);
  if (tid == 0 && p.vec) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_phi)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_psi)) : "memory");
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");   // earlier kernels' writes visible, their reads done
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  FUSED_STAMP(1);
  {
    const int nt = SH::NSP * gp;                       // 16-byte pieces of both tables
    for (int i = tid; i < nt; i += kSThreads)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n"
                   ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(Gs + 2 * i))), "l"(p.G + 2 * i) : "memory");
    for (int i = tid; i < (mpad - p.m) * 64; i += kSThreads) {   // sample rows past m stay zero
      const int t = p.m + (i >> 6), ch = i & 63;
      YA[t * kFYP + ch] = 0.0;
      YB[t * kFYP + ch] = 0.0;
    }
  }
  int I, J;
  fused_decode(p, b0, I, J);
  fused_load(p, 0, I * kSB, YA);
  bool diag = p.homo && I == J;
  if (!diag) fused_load(p, p.homo ? 0 : 1, J * kSB, YB);
  int curI = -1;
  unsigned long long mphi = 0, mpsi = 0;
  const double* Aw = As + (wm * 32 + lr) * KS + lk;    // this lane's operand fragment bases
  const double* Bw = Bs + (wn * 32 + lr) * KS + lk;
#pragma unroll 1
  for (long long b = b0; b < b1; ++b) {
    const bool newA = I != curI;
    if (b == b0 + 1) FUSED_STAMP(14);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();                                   // this block's samples (and the tables) landed
    if (b == b0) FUSED_STAMP(2);
    if (b == b0 + 1) FUSED_STAMP(15);
    // ---- centring / scaling: threads 0..63 the row channels, 64..127 the column channels
    if (tid < 64) {
      if (newA) {
        const int c = I * kSB + tid;
        fused_stats(p, 0, c, c < p.n1, fused_row_start(p, I) >= b0, YA + tid);
      }
    } else if (!diag) {
      const int c = J * kSB + tid - 64;
      const int set = p.homo ? 0 : 1;
      const int n = set ? p.n2 : p.n1;
      fused_stats(p, set, c, c < n, !p.homo && I == 0, YB + tid - 64);
    }
    if (b == b0) FUSED_STAMP(8);
    if (b == b0 + 1) FUSED_STAMP(9);
    __syncthreads();
    // ---- operand rows: role A (x Norm) of the row channels, role B of the
    //      column channels (a diagonal block: of the same channels)
    if (newA)
      fused_transform2<KG>(mpad, gp, YA, Gs, As, p.norm, diag ? YA : YB, Gs + SH::NSP * gp, Bs, warp, lr, lk);
    else
      fused_transform<KG>(mpad, gp, YB, Gs + SH::NSP * gp, Bs, 1.0, warp, lr, lk);
    if (b == b0) FUSED_STAMP(10);
    __syncthreads();                                   // operand rows ready, sample buffers free
    if (b == b0) FUSED_STAMP(3);
    if (b == b0 + 1) FUSED_STAMP(11);
    const int i0 = I * kSB, j0 = J * kSB;
    const bool mirror = p.homo && !diag;
    curI = I;
    // ---- prefetch the next block's samples (overlaps this block's contraction and stores)
    int nI = I, nJ = J;
    bool ndiag = diag;
    if (b + 1 < b1) {
      fused_decode(p, b + 1, nI, nJ);
      ndiag = p.homo && nI == nJ;
      if (nI != I) fused_load(p, 0, nI * kSB, YA);
      if (!ndiag) fused_load(p, p.homo ? 0 : 1, nJ * kSB, YB);
    }
    // ---- Gauss contraction: sync = P1 - P3, async = P1 + P2
    double aphi[2][4][4], apsi[2][4][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) aphi[a][q][e] = apsi[a][q][e] = 0.0;
    fused_seg2<KG>(apsi, aphi, Aw, Bw, 0, 2 * KG);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) aphi[a][q][e] += apsi[a][q][e];
    fused_seg1<KG>(apsi, Aw + KG, Bw + KG);
    if (b == b0) FUSED_STAMP(4);
    if (b == b0 + 1) FUSED_STAMP(12);
    // ---- max|.| / finite check from the fragments, on |x|'s bit pattern
    //      (integer pipe; Inf / NaN patterns exceed every finite one, so the
    //      maxima also carry the finite check).  Diagonal blocks: the upper
    //      triangle, which is what gets stored.
    const int rows = min(kSB, p.n1 - i0), cols = min(kSB, p.n2 - j0);
    if (!diag && rows == kSB && cols == kSB) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            mphi = max(mphi, abs_bits(aphi[mt][nt][q]));
            mpsi = max(mpsi, abs_bits(apsi[mt][nt][q]));
          }
    } else {
      fused_max_edge(aphi, apsi, rows, cols, diag, wm, wn, lr, lk, mphi, mpsi);
    }
    // ---- stage both planes (the previous block's stores must have read the staging)
    if (tid == 0) bulk_wait_read();
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wm * 32 + mt * 16 + lr + 8 * h, c = wn * 32 + nt * 8 + 2 * lk;
          const int o = swz(r, c);
          *reinterpret_cast<double2*>(Cst + o) = make_double2(aphi[mt][nt][2 * h], aphi[mt][nt][2 * h + 1]);
          *reinterpret_cast<double2*>(Cst + 4096 + o) = make_double2(apsi[mt][nt][2 * h], apsi[mt][nt][2 * h + 1]);
        }
    if (mirror && p.mirror_buf && p.vec) {   // the transposed block into the second buffer, now
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = wm * 32 + mt * 16 + lr + 8 * (q >> 1), c = wn * 32 + nt * 8 + 2 * lk + (q & 1);
            const int o = swz(c, r);
            Cmir[o] = aphi[mt][nt][q];
            Cmir[4096 + o] = neg_bits(apsi[mt][nt][q]);
          }
    }
    if (diag) {        // below the diagonal: the transpose of the upper triangle (exact symmetry)
      __syncthreads();
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = wm * 32 + mt * 16 + lr + 8 * (q >> 1), c = wn * 32 + nt * 8 + 2 * lk + (q & 1);
            if (r < c) {
              const int o = swz(c, r);
              Cst[o] = aphi[mt][nt][q];
              Cst[4096 + o] = neg_bits(apsi[mt][nt][q]);
            } else if (r == c) {
              Cst[4096 + swz(r, r)] = 0.0;
            }
          }
    }
    if (b == b0) FUSED_STAMP(5);
    if (p.vec) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic-proxy writes -> TMA
      __syncthreads();
      // odd n2: the maps cover the even width (TMA writes whole 16-byte
      // pieces at the right edge), the last column leaves by plain stores
      if ((p.n2 & 1) && j0 + cols == p.n2 && tid < rows) {
        __stcs(p.phi + (long long)(i0 + tid) * p.ld_out + p.n2 - 1, Cst[swz(tid, cols - 1)]);
        __stcs(p.psi + (long long)(i0 + tid) * p.ld_out + p.n2 - 1, Cst[4096 + swz(tid, cols - 1)]);
      }
      if (tid == 0) fused_store_tile(&map_phi, &map_psi, cst_s, i0, j0);
      if (mirror && p.mirror_buf) {
        if (tid == 0) fused_store_tile(&map_phi, &map_psi, cmir_s, j0, i0);   // staged with the block
      } else if (mirror) {   // the transposed block (sync^T, -async^T): rows j0.., columns i0..
        if (tid == 0) bulk_wait_read();                // one staging buffer: wait until it was read
        __syncthreads();
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int r = wm * 32 + mt * 16 + lr + 8 * (q >> 1), c = wn * 32 + nt * 8 + 2 * lk + (q & 1);
              const int o = swz(c, r);
              Cst[o] = aphi[mt][nt][q];
              Cst[4096 + o] = neg_bits(apsi[mt][nt][q]);
            }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (tid == 0) fused_store_tile(&map_phi, &map_psi, cst_s, j0, i0);
      }
    } else {           // planes not 16-B aligned / odd ld_out: plain stores from the staging
      __syncthreads();
#pragma unroll 1
      for (int idx = tid; idx < kSB * kSB; idx += kSThreads) {
        const int r = idx >> 6, c = idx & 63;
        if (r >= rows || c >= cols) continue;
        const double f = Cst[swz(r, c)], s = Cst[4096 + swz(r, c)];
        __stcs(p.phi + (long long)(i0 + r) * p.ld_out + j0 + c, f);
        __stcs(p.psi + (long long)(i0 + r) * p.ld_out + j0 + c, s);
        if (mirror) {
          __stcs(p.phi + (long long)(j0 + c) * p.ld_out + i0 + r, f);
          __stcs(p.psi + (long long)(j0 + c) * p.ld_out + i0 + r, neg_bits(s));
        }
      }
      __syncthreads();                                 // staging reads done before the next block's writes
    }
    if (b == b0) FUSED_STAMP(6);
    if (b == b0 + 1) FUSED_STAMP(13);
    I = nI;
    J = nJ;
    diag = ndiag;
  }
  fused_publish(p, mphi, mpsi, lane, warp, tid);
  if (tid == 0) bulk_wait_read();                     // the staging must outlive the stores' reads
  FUSED_STAMP(7);
}


// One set of atomics per CTA into the accumulator words; the last CTA to
// arrive publishes status / stats and leaves every work word zero.
__device__ __noinline__ void fused_publish(const FusedParams& p, unsigned long long mphi, unsigned long long mpsi,
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
  __shared__ int last;
  if (lane == 0) {
    red[0][warp] = mphi;
    red[1][warp] = mpsi;
    red[2][warp] = (unsigned long long)bad;
  }
  __syncthreads();
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(p.work + kWFAcc);
  if (tid == 0) {
    unsigned long long a0 = 0, a1 = 0, a2 = 0;
    for (int w = 0; w < kSThreads / 32; ++w) {
      a0 = max(a0, red[0][w]);
      a1 = max(a1, red[1][w]);
      a2 += red[2][w];
    }
    if (a0) atomicMax(&acc[0], a0);
    if (a1) atomicMax(&acc[1], a1);
    if (a2) atomicAdd(&acc[2], a2);
    __threadfence();
    last = atomicAdd(&p.work[kWFCount], 1) == p.nctas - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (tid < 3) p.stats[tid] = atomicExch(&acc[tid], 0ull);
  if (tid >= 32 && tid < 36) p.status1[tid - 32] = atomicExch(&p.work[kWFStat1 + tid - 32], 0);
  if (tid >= 64 && tid < 68) {
    const int v = atomicExch(&p.work[kWFStat2 + tid - 64], 0);
    if (p.status2) p.status2[tid - 64] = v;
  }
  if (tid == 96) atomicExch(&p.work[kWFCount], 0);
}

// =====================================================================
// Streamed contraction (maps with more 64 x 64 blocks than SMs, after
// small_prep_kernel): one persistent CTA per SM walks a contiguous run of
// blocks.  Per block the operand rows arrive by one bulk copy per row into one
// of two buffers (the next block's rows land while this block contracts),
// the Gauss contraction runs on the FP64 tensor pipe, and both planes (plus
// the homo mirror) are staged swizzled and leave by TMA tensor stores issued
// by one thread -- no warp waits on its own output stores, so the next
// block's DMMAs overlap this block's HBM write stream.  With two 64-KB staging
// slots, consecutive single-tile blocks alternate between them (the slot is
// reused only after the store two blocks back has read it).
// =====================================================================
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
}

// Operand rows of block (I, J) into buffer (As, Bs) -- the block's 64 rows of
// each role are one contiguous run of the dense operand arrays, so ONE bulk
// copy per role (per-row copies cost ~20 ns of TMA issue each), completing on
// `bar` (count 1: thread 0 arrives with the byte count).  Rows past the map
// are zeroed by the other threads (visible after the consumer's barrier).
template <int KG>
__device__ __forceinline__ void stream_load(const SmallParams& p, int I, int J, double* As, double* Bs, unsigned bar) {
  constexpr int OP = small_ops_pitch(KG);
  const int tid = threadIdx.x;
  const int ra = min(kSB, p.n1 - I * kSB), rb = min(kSB, p.n2 - J * kSB);
  if (tid == 0) {
    const unsigned ba = (unsigned)ra * OP * 8u, bb = (unsigned)rb * OP * 8u;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // earlier generic reads of the buffer
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(ba + bb) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(As))), "l"(p.opsA + (long long)I * kSB * OP),
                   "r"(ba), "r"(bar) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(Bs))), "l"(p.opsB + (long long)J * kSB * OP),
                   "r"(bb), "r"(bar) : "memory");
  }
  if (ra < kSB)
    for (int i = ra * OP + 2 * tid; i < kSB * OP; i += 2 * kSThreads) *reinterpret_cast<double2*>(As + i) = make_double2(0.0, 0.0);
  if (rb < kSB)
    for (int i = rb * OP + 2 * tid; i < kSB * OP; i += 2 * kSThreads) *reinterpret_cast<double2*>(Bs + i) = make_double2(0.0, 0.0);
}

// The same rows by cp.async (16 B per thread and copy, through L1 -- not
// queued behind the SM's outgoing TMA tensor stores), all threads; rows past
// the map zero-filled by a zero source size.  Completion: cp.async.wait_group.
template <int KG>
__device__ __forceinline__ void stream_load_lsu(const SmallParams& p, int I, int J, double* As, double* Bs,
                                                bool loadA = true) {
  constexpr int OP = small_ops_pitch(KG);
  constexpr int kPieces = kSB * OP / 2;                // 16-byte pieces per role
  const int ra = min(kSB, p.n1 - I * kSB), rb = min(kSB, p.n2 - J * kSB);
  const double* ga = p.opsA + (long long)I * kSB * OP;
  const double* gb = p.opsB + (long long)J * kSB * OP;
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(As));
  const unsigned sb = static_cast<unsigned>(__cvta_generic_to_shared(Bs));
#pragma unroll 4
  for (int i = threadIdx.x; i < kPieces; i += kSThreads) {
    const bool va = 2 * i < ra * OP, vb = 2 * i < rb * OP;
    if (loadA)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa + 16u * i), "l"(ga + (va ? 2 * i : 0)),
                   "r"(va ? 16 : 0) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sb + 16u * i), "l"(gb + (vb ? 2 * i : 0)),
                 "r"(vb ? 16 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// Fragments -> one staged tile at Cs (swizzled boxes); transposed: the mirror
// (sync^T, -async^T).
__device__ __forceinline__ void stage_tile(double* Cs, const double (&aphi)[2][4][4], const double (&apsi)[2][4][4],
                                           bool transposed, int wm, int wn, int lr, int lk) {
  if (!transposed) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wm * 32 + mt * 16 + lr + 8 * h, c = wn * 32 + nt * 8 + 2 * lk;
          const int o = swz(r, c);
          *reinterpret_cast<double2*>(Cs + o) = make_double2(aphi[mt][nt][2 * h], aphi[mt][nt][2 * h + 1]);
          *reinterpret_cast<double2*>(Cs + 4096 + o) = make_double2(apsi[mt][nt][2 * h], apsi[mt][nt][2 * h + 1]);
        }
  } else {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = wm * 32 + mt * 16 + lr + 8 * (q >> 1), c = wn * 32 + nt * 8 + 2 * lk + (q & 1);
          const int o = swz(c, r);
          Cs[o] = aphi[mt][nt][q];
          Cs[4096 + o] = neg_bits(apsi[mt][nt][q]);
        }
  }
}

__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); }

// NB operand buffers: 2 (one CTA per SM, the next block's rows prefetched)
// or 1 (two CTAs per SM, each loading its next block once its contraction has
// read the buffer; the other CTA's work covers the load)
template <int KG, int NB>
__global__ void __launch_bounds__(kSThreads, 3 - NB)
small_stream_kernel(const __grid_constant__ SmallParams p, const __grid_constant__ CUtensorMap map_phi,
                    const __grid_constant__ CUtensorMap map_psi) {
  constexpr int KS = small_ops_pitch(KG);
  extern __shared__ __align__(1024) double sm_raw[];
  __shared__ __align__(8) unsigned long long bars[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  // accumulator row lr holds output row lrp (bits 0 and 2 of lr exchanged,
  // through the A fragment rows): the two rows of a 16-B store's 8-lane phase
  // then differ in bit 2, and their SWIZZLE_128B chunks in different halves
  // of the 128-B line (no bank conflict when the planes are staged)
  const int lrp = (lr & 2) | ((lr & 1) << 2) | (lr >> 2);
  const int wm = warp >> 1, wn = warp & 1;
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(sm_raw));
  double* Cst = sm_raw + (((1024u - (sbase & 1023u)) & 1023u) >> 3);   // staging slots (64 KB each)
  const unsigned cst_s = static_cast<unsigned>(__cvta_generic_to_shared(Cst));
  double* Ops = Cst + 8192 * p.nslots;                 // [NB buffers][A | B][64][KS]
  const unsigned bar_s = static_cast<unsigned>(__cvta_generic_to_shared(bars));
  const long long b0 = (long long)blockIdx.x * p.tiles / p.nctas;
  const long long b1 = (long long)(blockIdx.x + 1) * p.tiles / p.nctas;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_s) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_s + 8) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_phi)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_psi)) : "memory");
  }
  __syncthreads();
  __shared__ unsigned long long call_idx;
  if (!p.pipe) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // K1 complete, its operand rows visible
    // the next kernel (the next call's K1) may launch now: everything before
    // this grid completed, and K1 writes nothing before its own wait
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  } else {
    // tickets first; then the next call's K1 may launch at once (it takes its
    // tickets, computes, and writes its slot when that slot's previous use is
    // complete); this call starts when all of its K1's CTAs have counted in
    __shared__ unsigned long long use_idx;
    if (tid == 0) {
      use_idx = atomicAdd(p.pipe + kPSClaim + p.slot, 1ull) / (unsigned long long)p.nctas;
      call_idx = atomicAdd(p.pipe + kPSCall, 1ull) / (unsigned long long)p.nctas;
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (tid == 0) pipe_wait_at_least(p, p.pipe + kPReady + p.slot, (unsigned long long)p.k1_ctas * (use_idx + 1));
    __syncthreads();
  }
  SMALL_STAMP(kTraceK1, 1);
  // K1's status accumulators are final now: CTA 0 publishes them and leaves
  // the words zero for the next call (whose K1 starts after this grid ends)
  if (blockIdx.x == 0 && tid < 4) {
    p.status1[tid] = p.work[kWStatus1 + tid];
    p.work[kWStatus1 + tid] = 0;
    if (p.status2) p.status2[tid] = p.work[kWStatus2 + tid];
    p.work[kWStatus2 + tid] = 0;
  }
#ifdef CORR2D_PROFILING
  if (p.dbg & 4) {                                     // K1 + an empty contraction grid
    if (p.pipe) {
      if (tid == 0) pipe_wait_value(p, p.pipe + kPPlanes, call_idx);
      __syncthreads();
      pipe_release(p, tid, call_idx);
    }
    return;
  }
#endif
  int I, J;
  small_decode(p, b0, I, J);
  const bool lsu = NB == 1 && !p.tma_ops;
  if (lsu) stream_load_lsu<KG>(p, I, J, Ops, Ops + 64 * KS);
  else stream_load<KG>(p, I, J, Ops, Ops + 64 * KS, bar_s);
  unsigned long long mphi = 0, mpsi = 0;
  int prev_mask = 0;                                   // staging slots the most recent store group reads
#pragma unroll 1
  for (long long b = b0; b < b1; ++b) {
    const int k = (int)(b - b0), buf = NB == 2 ? (k & 1) : 0;
    const double* As = Ops + buf * 128 * KS;
    const double* Bs = As + 64 * KS;
    if (lsu) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    else mbar_wait(bar_s + 8 * buf, (k / NB) & 1);
    __syncthreads();                                   // zero-filled rows visible; the other buffer is free
    if (b == b0) SMALL_STAMP(kTraceK1, 2);
    if (b == b0 + 2) SMALL_STAMP(kTraceK1, 6);
    const bool diag = p.homo && I == J;
    const int i0 = I * kSB, j0 = J * kSB;
    int nI = I, nJ = J;
    if (b + 1 < b1) small_decode(p, b + 1, nI, nJ);
    if (NB == 2 && b + 1 < b1) {                       // the next block's rows land during this contraction
      double* nA = Ops + (buf ^ 1) * 128 * KS;
      stream_load<KG>(p, nI, nJ, nA, nA + 64 * KS, bar_s + 8 * (buf ^ 1));
    }
    // ---- Gauss contraction: sync = P1 - P3, async = P1 + P2
    const double* Aw = As + (wm * 32 + lrp) * KS + lk;
    const double* Bw = Bs + (wn * 32 + lr) * KS + lk;
    double aphi[2][4][4], apsi[2][4][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) aphi[a][q][e] = apsi[a][q][e] = 0.0;
#ifdef CORR2D_PROFILING
    if (!(p.dbg & 2)) {
#endif
    fused_seg2<KG, KS>(apsi, aphi, Aw, Bw, 0, 2 * KG);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) aphi[a][q][e] += apsi[a][q][e];
    fused_seg1<KG, KS>(apsi, Aw + KG, Bw + KG);
#ifdef CORR2D_PROFILING
    }
#endif
    if (b == b0 + 2) SMALL_STAMP(kTraceK1, 3);
    // ---- max|.| / finite check on |x|'s bit pattern (diagonal: the upper triangle)
    const int rows = min(kSB, p.n1 - i0), cols = min(kSB, p.n2 - j0);
    if (!diag && rows == kSB && cols == kSB) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            mphi = max(mphi, abs_bits(aphi[mt][nt][q]));
            mpsi = max(mpsi, abs_bits(apsi[mt][nt][q]));
          }
    } else {
      fused_max_edge(aphi, apsi, rows, cols, diag, wm, wn, lrp, lk, mphi, mpsi);
    }
    // ---- staging slots: a mirrored block takes both (or stores twice through one)
    const bool mirror = p.homo && !diag;
    int s0 = 0;
    const bool both = mirror && p.nslots == 2;
    if (tid == 0) {
      if (both || p.nslots == 1 || prev_mask == 3) bulk_wait_read();
      else bulk_wait_read1();                          // the previous block's group may still read its slot
      // pipelined: earlier calls write the same planes -- our first store
      // waits until every earlier call's stores have completed
      if (p.pipe && b == b0) pipe_wait_value(p, p.pipe + kPPlanes, call_idx);
    }
    if (!both && p.nslots == 2 && prev_mask == 1) s0 = 1;
    prev_mask = both ? 3 : (1 << s0);
    __syncthreads();                                   // every warp's DMMAs have read the operand buffer
    if (b == b0 + 2) SMALL_STAMP(kTraceK1, 0);
    // (a run of blocks along one row block keeps its A rows: only B reloads)
    if (lsu && b + 1 < b1) stream_load_lsu<KG>(p, nI, nJ, Ops, Ops + 64 * KS, nI != I);   // lands during the staging
    double* C0 = Cst + 8192 * s0;
    stage_tile(C0, aphi, apsi, false, wm, wn, lrp, lk);
    if (both) stage_tile(Cst + 8192, aphi, apsi, true, wm, wn, lrp, lk);
    if (diag) {        // below the diagonal: the transpose of the upper triangle (exact symmetry)
      __syncthreads();
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = wm * 32 + mt * 16 + lrp + 8 * (q >> 1), c = wn * 32 + nt * 8 + 2 * lk + (q & 1);
            if (r < c) {
              const int o = swz(c, r);
              C0[o] = aphi[mt][nt][q];
              C0[4096 + o] = neg_bits(apsi[mt][nt][q]);
            } else if (r == c) {
              C0[4096 + swz(r, r)] = 0.0;
            }
          }
    }
    if (b == b0 + 2) SMALL_STAMP(kTraceK1, 4);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic-proxy writes -> TMA
    __syncthreads();
    // odd n2: the maps cover the even width, the last column leaves by plain stores
    if ((p.n2 & 1) && j0 + cols == p.n2 && tid < rows) {
      __stcs(p.phi + (long long)(i0 + tid) * p.ld_out + p.n2 - 1, C0[swz(tid, cols - 1)]);
      __stcs(p.psi + (long long)(i0 + tid) * p.ld_out + p.n2 - 1, C0[4096 + swz(tid, cols - 1)]);
    }
#ifdef CORR2D_PROFILING
    if (p.dbg & 1) {
      if (NB == 1 && !lsu && b + 1 < b1) stream_load<KG>(p, nI, nJ, Ops, Ops + 64 * KS, bar_s);
      I = nI; J = nJ;
      continue;
    }
#endif
    if (tid == 0) {
      fused_store_tile(&map_phi, &map_psi, cst_s + 65536u * s0, i0, j0);
      if (both) fused_store_tile(&map_phi, &map_psi, cst_s + 65536u, j0, i0);
    }
    if (mirror && !both) {   // one slot: the mirror goes through it once the direct tile was read
      if (tid == 0) bulk_wait_read();
      __syncthreads();
      stage_tile(C0, aphi, apsi, true, wm, wn, lrp, lk);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncthreads();
      if (tid == 0) fused_store_tile(&map_phi, &map_psi, cst_s, j0, i0);
    }
    // one operand buffer: the next block's rows, issued after this block's
    // proxy fences (a fence.proxy.async in the issuing thread would otherwise
    // wait for the copies to land)
    if (NB == 1 && !lsu && b + 1 < b1) stream_load<KG>(p, nI, nJ, Ops, Ops + 64 * KS, bar_s);
    if (b == b0 + 2) SMALL_STAMP(kTraceK1, 7);
    I = nI;
    J = nJ;
  }
  small_publish(p, mphi, mpsi, lane, warp, tid);
  if (!p.pipe) {
    if (tid == 0) bulk_wait_read();                   // the staging must outlive the stores' reads
  } else {
    // pipelined: every store of this CTA performed, then the slot's arrival
    // count; the last CTA releases the slot (and the next call's stores)
    pipe_release(p, tid, call_idx);
  }
  SMALL_STAMP(kTraceK1, 5);
}

// =====================================================================
// K1 of the two-kernel path, operand rows by ONE tensor-core product: 64
// channels per CTA (one lane each for the statistics), then per role
// rows[ch][s] = scale * sum_t y[t][ch] G[s][t] on the FP64 tensor pipe (G =
// the rfft rows of fourier.py:73 already combined into the Gauss slots, the
// table of the fused kernel), written in the rows' global layout (pitch
// small_ops_pitch) and copied out with one bulk copy per warp and role.
// Everything before griddepcontrol.wait only reads global memory (see
// small_prep_kernel).
// =====================================================================
template <int KG>
__device__ __forceinline__ void rows_transform(int mpad, int gp, const double* ys, const double* Gt, double* out,
                                               double scale, int warp, int lr, int lk) {
  using S = FShape<KG>;
  constexpr int OP = small_ops_pitch(KG);
  double acc[S::NNT][4];
#pragma unroll
  for (int a = 0; a < S::NNT; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[a][q] = 0.0;
  const int ch = 16 * warp + lr;
  const double* y = ys + lk * kFYP + ch;
  const double* g = Gt + lr * gp + lk;
#pragma unroll 2
  for (int kk = 0; kk < mpad; kk += 4) {
    const double a0 = y[kk * kFYP];
    const double a1 = y[kk * kFYP + 8];
#pragma unroll
    for (int nt = 0; nt < S::NNT; ++nt) dmma(acc[nt], a0, a1, g[nt * 8 * gp + kk]);
  }
#pragma unroll
  for (int nt = 0; nt < S::NNT; ++nt) {
    const int c = nt * 8 + 2 * lk;
    if (c < 3 * KG) {                                  // slots past 3 kg: the row's pad (zeroed by the caller)
      *reinterpret_cast<double2*>(out + ch * OP + c) = make_double2(acc[nt][0] * scale, acc[nt][1] * scale);
      *reinterpret_cast<double2*>(out + (ch + 8) * OP + c) = make_double2(acc[nt][2] * scale, acc[nt][3] * scale);
    }
  }
}

template <int KG>
__global__ void __launch_bounds__(kSThreads) small_rows_kernel(const __grid_constant__ SmallParams p) {
  using SH = FShape<KG>;
  constexpr int OP = small_ops_pitch(KG);
  extern __shared__ __align__(16) double sm[];
  const int m = p.m, mpad = p.mpad, gp = p.mpad + 2;
  double* Gs = sm;                                     // [2][NSP][gp]
  double* ys = Gs + 2 * SH::NSP * gp;                  // [mpad][kFYP]
  double* rowsA = ys + mpad * kFYP;                    // [64][OP]
  double* rowsB = rowsA + kSB * OP;                    // [64][OP]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  const int set = (int)blockIdx.x >= p.nb1 ? 1 : 0;
  const int c0 = ((int)blockIdx.x - (set ? p.nb1 : 0)) * kSB;
  const int n = set ? p.n2 : p.n1;
  __shared__ unsigned long long use_idx;
  if (p.pipe) {                                        // ticket first, then the next kernel may launch
    if (tid == 0) use_idx = atomicAdd(p.pipe + kPClaim + p.slot, 1ull) / (unsigned long long)p.k1_ctas;
    __syncthreads();
  }
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  SMALL_STAMP(0, 0);
  {
    const int nt = SH::NSP * gp;                       // 16-byte pieces of both tables
    for (int i = tid; i < nt; i += kSThreads)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n"
                   ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(Gs + 2 * i))), "l"(p.G + 2 * i) : "memory");
    const void* raw = set ? p.raw2 : p.raw1;
    const long long ld = set ? p.ld2 : p.ld1;
#pragma unroll 1
    for (int idx = tid; idx < m * kSB; idx += kSThreads) {
      const int t = idx >> 6, ch = idx & 63, c = c0 + ch;
      const bool v = c < n;
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(ys + t * kFYP + ch));
      if (p.in_f32) {
        const float* src = static_cast<const float*>(raw) + (long long)t * ld + (v ? c : 0);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 4 : 0) : "memory");
      } else {
        const double* src = static_cast<const double*>(raw) + (long long)t * ld + (v ? c : 0);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(v ? 8 : 0) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    for (int i = tid; i < (mpad - m) * kSB; i += kSThreads)   // sample rows past m stay zero
      ys[(m + (i >> 6)) * kFYP + (i & 63)] = 0.0;
    if (OP > 3 * KG)                                   // row pads
      for (int i = tid; i < 2 * kSB; i += kSThreads)
        for (int s = 3 * KG; s < OP; ++s) rowsA[i * OP + s] = 0.0;
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  __syncthreads();
  SMALL_STAMP(0, 2);
  LaneStat lst{0.0, 0.0, 0};
  const int c = c0 + tid;
  const bool valid = c < n;
  if (tid < kSB) {
    if (p.in_f32)
      for (int t = 0; t < m; ++t) ys[t * kFYP + tid] = (double)reinterpret_cast<const float*>(ys + t * kFYP + tid)[0];
    lst = lane_stats<kFYP>(p, set, c, valid, ys + tid);
  }
  __syncthreads();
  SMALL_STAMP(0, 3);
  const bool wantA = !set, wantB = set || p.homo;
  if (wantA) rows_transform<KG>(mpad, gp, ys, Gs, rowsA, p.norm, warp, lr, lk);
  if (wantB) rows_transform<KG>(mpad, gp, ys, Gs + SH::NSP * gp, rowsB, 1.0, warp, lr, lk);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic-proxy writes -> bulk copy
  __syncwarp();
  SMALL_STAMP(0, 7);
  if (p.pipe) {                                        // this slot's previous user has finished with it
    if (tid == 0) pipe_wait_value(p, p.pipe + kPGen + p.slot, use_idx);
    __syncthreads();
  } else {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");   // the previous call's contraction is done
  }
  if (blockIdx.x == 0 && tid < 3) p.stats[tid] = 0ull;
  if (tid < kSB && valid) lane_report(p, set, c, lst);
  {
    const int cw = c0 + 16 * warp;                     // the warp's 16 rows
    const int nrow = min(16, n - cw);
    if (nrow > 0 && lane == 0) {
      const unsigned bytes = (unsigned)(nrow * OP) * 8u;
      if (wantA)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                     ::"l"(p.opsA + (long long)cw * OP),
                       "r"(static_cast<unsigned>(__cvta_generic_to_shared(rowsA + 16 * warp * OP))), "r"(bytes) : "memory");
      if (wantB)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                     ::"l"(p.opsB + (long long)cw * OP),
                       "r"(static_cast<unsigned>(__cvta_generic_to_shared(rowsB + 16 * warp * OP))), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;\n" ::: "memory");
    }
  }
  if (p.pipe) {                                        // pipelined: count this CTA into ready[slot]
    if (lane == 0) asm volatile("fence.proxy.async.global;\n" ::: "memory");   // the bulk-copied rows
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(p.pipe + kPReady + p.slot, 1ull);
  }
  SMALL_STAMP(0, 5);
}

// Per-(device, m) table of the fused path: [2][nsp][gp] doubles -- role A rows
// s (slot of the Gauss segments, corr2d.h CORR2D_PACK_F64_GAUSS) hold
// pa cos(2 pi w t / m) + qa (-sin(2 pi w t / m)) for t < m (Norm is applied in
// the kernel), role B rows pb cos + qb (-sin); pads are zero.
static const double* fused_table(int m, int nsp, int gp, cudaStream_t st, int* rc) {
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
  std::vector<double> h((size_t)2 * nsp * gp, 0.0);
  const double two_pi = 6.283185307179586476925286766559;
  for (int s = 0; s < ns; ++s) {
    const int seg = s / kg, j = s - seg * kg, w = gauss_bin(seg, j, m);
    if (w < 0) continue;
    const bool edge = w == 0 || (m % 2 == 0 && w == m / 2);
    const double kk = edge ? 1.0 : 2.0, ki = edge ? 0.0 : 1.0;
    double pa, qa, pb, qb;
    if (seg == 0) { pa = kk; qa = kk * ki; pb = 1.0; qb = 0.0; }          // a + b, c
    else if (seg == 1) { pa = kk; qa = 0.0; pb = -1.0; qb = -ki; }        // a, d - c
    else if (edge) { pa = kk; qa = 0.0; pb = 1.0; qb = 0.0; }             // Nyquist: a, c
    else { pa = 0.0; qa = -kk; pb = 1.0; qb = -1.0; }                     // -b, c + d
    for (int t = 0; t < m; ++t) {
      const int q = (w * t) % m;
      const double ang = two_pi * (double)q / (double)m;
      const double c = std::cos(ang);
      const double ns_ = (q == 0 || 2 * q == m) ? 0.0 : -std::sin(ang);   // Im part of exp(-i ang): exact 0 at 0, pi
      h[(size_t)s * gp + t] = pa * c + qa * ns_;
      h[(size_t)(nsp + s) * gp + t] = pb * c + qb * ns_;
    }
  }
  double* d = nullptr;
  if (cudaMalloc(&d, h.size() * sizeof(double)) != cudaSuccess ||
      cudaMemcpy(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
    *rc = check_launch("small fused table");
    return nullptr;
  }
  tab[dev][m] = d;
  return d;
}

static int device_sms() {
  constexpr int kDev = 64;
  static int sms[kDev] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kDev) return 148;
  if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  return sms[dev] > 0 ? sms[dev] : 148;
}

static PFN_cuTensorMapEncodeTiled_v12000 fused_encode_fn() {
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

// Output plane (rows x cols fp64, leading dimension ld): 64-row x 16-column
// boxes, SWIZZLE_128B (the staging layout of swz()).
static int fused_plane_map(CUtensorMap* map, double* base, long long ld, long long rows, long long cols) {
  auto fn = fused_encode_fn();
  if (!fn) return fail(CORR2D_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {16, 64};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CORR2D_ERR_CUDA, "cuTensorMapEncodeTiled(small planes) failed (" + std::to_string((int)r) + ")");
  return CORR2D_OK;
}

// operand row pitch of the streamed contraction
static int stream_ks(int kg) { return small_ops_pitch(kg); }

// CORR2D_SMALL_STREAM=0 (read once) selects the one-CTA-per-block contraction
static bool stream_disabled() {
  static const int v = [] {
    const char* e = getenv("CORR2D_SMALL_STREAM");
    return (e && e[0] == '0') ? 1 : 0;
  }();
  return v != 0;
}

// a 0/1 switch from the environment, read once per name
static int env_flag(const char* name) {
  const char* e = getenv(name);
  return (e && e[0] == '1') ? 1 : 0;
}

// CORR2D_SMALL_STREAM_NB=2 (read once): one streamed-contraction CTA per SM
static int stream_nb() {
  static const int v = [] {
    const char* e = getenv("CORR2D_SMALL_STREAM_NB");
    return (e && e[0] == '2') ? 2 : 0;
  }();
  return v;
}

static int launch_fused(const SmallParams& q, cudaStream_t st) {
  FusedParams p{};
  p.raw1 = q.raw1; p.raw2 = q.raw2; p.ld1 = q.ld1; p.ld2 = q.ld2; p.in_f32 = q.in_f32;
  p.al1 = (reinterpret_cast<uintptr_t>(q.raw1) & 15) == 0 && q.ld1 % 2 == 0;
  p.al2 = q.raw2 && (reinterpret_cast<uintptr_t>(q.raw2) & 15) == 0 && q.ld2 % 2 == 0;
  p.m = q.m; p.mpad = q.mpad; p.gp = q.mpad + 2; p.n1 = q.n1; p.n2 = q.n2; p.homo = q.homo;
  p.ref_mode1 = q.ref_mode1; p.ref_mode2 = q.ref_mode2; p.ref_in1 = q.ref_in1; p.ref_in2 = q.ref_in2;
  p.sigma_in1 = q.sigma_in1; p.sigma_in2 = q.sigma_in2; p.alpha = q.alpha; p.substitute = q.substitute;
  p.norm = q.norm;
  p.ref_out1 = q.ref_out1; p.sigma_out1 = q.sigma_out1; p.ref_out2 = q.ref_out2; p.sigma_out2 = q.sigma_out2;
  p.kg = gauss_kg(q.m); p.ns = 3 * p.kg; p.nsp = (p.ns + 7) / 8 * 8; p.ks = p.nsp + 4;
  p.T1 = q.T1; p.T2 = q.T2;
  p.tiles = small_blocks(q.n1, q.n2, q.homo);
  const int sms = device_sms();
  p.nctas = (int)std::min<long long>(p.tiles, sms);
  p.phi = q.phi; p.psi = q.psi; p.ld_out = q.ld_out; p.vec = q.vec && q.n2 >= 2;
  p.status1 = q.status1; p.status2 = q.status2; p.stats = q.stats; p.work = q.work; p.trace = q.trace;
  int rc = CORR2D_OK;
  p.G = fused_table(p.m, p.nsp, p.gp, st, &rc);
  if (!p.G) return rc;
  CUtensorMap map_phi, map_psi;
  memset(&map_phi, 0, sizeof(map_phi));
  memset(&map_psi, 0, sizeof(map_psi));
  if (p.vec) {
    if (int e = fused_plane_map(&map_phi, p.phi, p.ld_out, p.n1, p.n2 & ~1)) return e;
    if (int e = fused_plane_map(&map_psi, p.psi, p.ld_out, p.n1, p.n2 & ~1)) return e;
  }
  size_t smem = 1024 + (8192 + 2 * (size_t)p.nsp * p.gp + 2 * (size_t)p.mpad * kFYP + 2 * 64 * (size_t)p.ks) *
                           sizeof(double);
  if (p.homo && smem + 65536 <= 226 * 1024) {
    p.mirror_buf = 1;
    smem += 65536;
  }
  static bool attr_set = false;
  if (!attr_set) {
    const int worst = 226 * 1024;   // 227 KB per block minus the static 1 KB
    cudaFuncSetAttribute(small_fused_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
    cudaFuncSetAttribute(small_fused_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
    cudaFuncSetAttribute(small_fused_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
    cudaFuncSetAttribute(small_fused_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
    attr_set = true;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kSThreads);
  cfg.gridDim = dim3((unsigned)p.nctas);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (p.kg) {
    case 4: cudaLaunchKernelEx(&cfg, small_fused_kernel<4>, p, map_phi, map_psi); break;
    case 8: cudaLaunchKernelEx(&cfg, small_fused_kernel<8>, p, map_phi, map_psi); break;
    case 12: cudaLaunchKernelEx(&cfg, small_fused_kernel<12>, p, map_phi, map_psi); break;
    default: cudaLaunchKernelEx(&cfg, small_fused_kernel<16>, p, map_phi, map_psi); break;
  }
  const int code = check_launch("small_fused_kernel");
#ifdef CORR2D_PROFILING
  if (p.trace) {
    std::vector<unsigned long long> h(16 * (size_t)p.nctas);
    cudaMemcpyAsync(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < p.nctas; ++b) t0 = std::min(t0, h[16 * b]);
    const char* nm[16] = {"start", "after wait", "samples in", "prep done", "mma done", "staged",
                          "stores issued", "end", "stats done (t0)", "stats done (t1)", "transforms done",
                          "prep done (t1)", "mma done (t1)", "stores issued (t1)", "tile 1 top", "samples in (t1)"};
    fprintf(stderr, "small fused trace (m %d, %d x %d, %s, %d CTAs, %lld tiles; first tile of each CTA):\n",
            p.m, p.n1, p.n2, p.homo ? "homo" : "hetero", p.nctas, p.tiles);
    for (int k : {0, 1, 2, 8, 10, 3, 4, 5, 6, 14, 15, 9, 11, 12, 13, 7}) {
      std::vector<double> v;
      for (int b = 0; b < p.nctas; ++b)
        if (h[16 * b + k]) v.push_back((double)(h[16 * b + k] - t0));
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      fprintf(stderr, "  %-16s min %8.0f  med %8.0f  max %8.0f ns\n", nm[k], v.front(), v[v.size() / 2], v.back());
    }
  }
#endif
  return code;
}

}  // namespace corr2d

using namespace corr2d;

extern "C" int64_t corr2d_small_block_count(int n1, int n2, int homo) {
  if (n1 < 1 || n2 < 1 || (homo && n1 != n2)) return -1;
  return small_blocks(n1, n2, homo);
}

extern "C" int corr2d_small_launches(int n1, int n2, int homo) {
  if (n1 < 1 || n2 < 1 || (homo && n1 != n2)) return -1;
#if defined(CORR2D_SMALL_FORCE_FUSED)
  return 1;
#else
  return 2;
#endif
}

extern "C" int corr2d_small_ops_depth(int m) { return (m >= 2 && m <= kSMaxM) ? small_ops_pitch(gauss_kg(m)) : -1; }

static int correlate_small(
    int in_dtype, const void* raw1, int64_t ld_raw1, const void* raw2, int64_t ld_raw2,
    int m, int n1, int n2,
    int ref_mode1, const double* ref_in1, const double* sigma_in1,
    int ref_mode2, const double* ref_in2, const double* sigma_in2,
    double alpha, int substitute_zero_var, double norm_const,
    double* ops_a, double* ops_b, int64_t ld_ops,
    double* ref_out1, double* sigma_out1, double* ref_out2, double* sigma_out2,
    double* phi, double* psi, int64_t ld_out,
    int32_t* status1, int32_t* status2, unsigned long long* stats, int32_t* work, void* stream, int slot, unsigned long long* pipe) {
  const bool homo = raw2 == nullptr;
  if (!raw1 || !phi || !psi || !status1 || !stats || !work || (!homo && !status2))
    return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: null pointer");
  if (in_dtype != CORR2D_F64 && in_dtype != CORR2D_F32) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad dtype");
  if (m < 2 || m > kSMaxM) return fail(CORR2D_ERR_UNSUPPORTED, "corr2d_correlate_small_f64: needs 2 <= m <= 32");
  if (n1 < 1 || n2 < 1) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: bad sizes");
  if (homo && n1 != n2) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: homo needs n1 == n2");
  if (ld_raw1 < n1 || (!homo && ld_raw2 < n2)) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: ld_raw < n");
  if (ld_out < n2) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: ld_out < n2");
  if ((ops_a || ops_b) && (ld_ops != corr2d_small_ops_depth(m) ||
      ((reinterpret_cast<uintptr_t>(ops_a) | reinterpret_cast<uintptr_t>(ops_b)) & 15)))
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
  p.kg = gauss_kg(m);
  p.T1 = (n1 + kSB - 1) / kSB; p.T2 = (n2 + kSB - 1) / kSB;
  p.phi = phi; p.psi = psi; p.ld_out = ld_out;
  p.vec = (ld_out % 2 == 0) && ((reinterpret_cast<uintptr_t>(phi) | reinterpret_cast<uintptr_t>(psi)) & 15) == 0;
  p.status1 = status1; p.status2 = homo ? nullptr : status2; p.stats = stats; p.work = work;
  if (pipe && (slot < 0 || slot > 1)) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64_slot: slot must be 0 or 1");
#ifdef CORR2D_PROFILING
  if (const char* e = getenv("CORR2D_DEBUG_SKIP")) p.dbg = atoi(e);
  if (const char* e = getenv("CORR2D_SMALL_TRACE"))
    if (e[0] == '1') {
      static unsigned long long* tbuf = nullptr;
      const size_t words = 16 * (size_t)(kTraceK1 + 65536);
      if (!tbuf) cudaMalloc(&tbuf, words * 8);
      cudaMemsetAsync(tbuf, 0, words * 8, st);
      p.trace = tbuf;
    }
#endif
  // K1 once per channel, then the streamed contraction (the operand rows stay
  // in L2 between the two kernels; K1 overlaps the previous call's
  // contraction): cfg1 8.4 us vs 10.4 us for the one-kernel variant, which
  // serves calls without operand scratch
#if defined(CORR2D_SMALL_FORCE_FUSED)
  const bool fused = true;
#else
  const bool fused = !ops_a || !ops_b;
#endif
  if (fused) return launch_fused(p, st);
  if (!ops_a || !ops_b) return fail(CORR2D_ERR_DATA, "corr2d_correlate_small_f64: null pointer");
  int rc = CORR2D_OK;
  const int nsp = (3 * p.kg + 7) / 8 * 8, gp = p.mpad + 2;
  p.G = fused_table(m, nsp, gp, st, &rc);
  if (!p.G) return rc;
  p.ks = (3 * p.kg + 11) / 16 * 16 + 4;
  p.nb1 = (n1 + kSB - 1) / kSB;
  p.opsA = ops_a; p.opsB = ops_b; p.ld_ops = ld_ops;
  const long long blocks = small_blocks(n1, n2, homo);
  if (blocks > 0x7fffffffLL) return fail(CORR2D_ERR_UNSUPPORTED, "corr2d_correlate_small_f64: too many blocks");
  const int prep_blocks = p.nb1 + (homo ? 0 : (n2 + kSB - 1) / kSB);
  const size_t prep_smem = (2 * (size_t)nsp * gp + (size_t)p.mpad * kFYP + 2 * (size_t)kSB * ld_ops) * sizeof(double);
  const size_t ops = 2 * (size_t)kSB * p.ks * sizeof(double);
  const size_t stage = 2 * (size_t)kSB * kCS * sizeof(double);
  const size_t smem = ops > stage ? ops : stage;
  static bool attr_set = false;
  if (!attr_set) {
    const size_t worst_ops = 2 * (size_t)kSB * 52 * sizeof(double);
    cudaFuncSetAttribute(small_contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(worst_ops > stage ? worst_ops : stage));
    const int worst_rows = (int)((2 * 48 * 34 + 32 * kFYP + 2 * kSB * 52) * sizeof(double));   // m = 32: kg = 16
    cudaFuncSetAttribute(small_rows_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst_rows);
    cudaFuncSetAttribute(small_rows_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst_rows);
    cudaFuncSetAttribute(small_rows_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst_rows);
    cudaFuncSetAttribute(small_rows_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst_rows);
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
  // streamed contraction (persistent, TMA stores) when the planes take 16-B
  // tensor stores; the one-CTA-per-block kernel otherwise.  Only the streamed
  // contraction takes part in pipelining.
  const bool streamed = p.vec && n2 >= 2 && !stream_disabled();
  if (streamed && pipe) {
    p.slot = slot;
    p.pipe = pipe;
    p.k1_ctas = prep_blocks;
  }
  // everything that can fail is settled before K1 launches (a pipelined K1
  // takes tickets that only its contraction retires)
  int nb = 1;
  size_t sops = 0;                                     // streamed: operand-buffer bytes
  CUtensorMap map_phi, map_psi;
  memset(&map_phi, 0, sizeof(map_phi));
  memset(&map_psi, 0, sizeof(map_psi));
  if (streamed) {
    p.tiles = blocks;
    // two CTAs per SM (one operand buffer and one staging slot each) when
    // both fit, else one CTA per SM with a prefetch buffer (and two slots when
    // they fit); CORR2D_SMALL_STREAM_NB=2 forces the latter
    const size_t ops1 = 128 * (size_t)stream_ks(p.kg) * sizeof(double);
    nb = (2 * (1024 + 65536 + ops1 + 1024) <= 228 * 1024 && stream_nb() != 2) ? 1 : 2;
    p.nctas = (int)std::min<long long>(blocks, (long long)(3 - nb) * device_sms());
    sops = nb * ops1;
    p.nslots = (nb == 2 && 1024 + 2 * 65536 + sops <= 226 * 1024) ? 2 : 1;
    if (int e = fused_plane_map(&map_phi, p.phi, p.ld_out, p.n1, p.n2 & ~1)) return e;
    if (int e = fused_plane_map(&map_psi, p.psi, p.ld_out, p.n1, p.n2 & ~1)) return e;
    p.tma_ops = env_flag("CORR2D_SMALL_TMA_OPS");
  }
  cfg.gridDim = dim3((unsigned)prep_blocks);
  cfg.dynamicSmemBytes = prep_smem;
  switch (p.kg) {
    case 4: cudaLaunchKernelEx(&cfg, small_rows_kernel<4>, p); break;
    case 8: cudaLaunchKernelEx(&cfg, small_rows_kernel<8>, p); break;
    case 12: cudaLaunchKernelEx(&cfg, small_rows_kernel<12>, p); break;
    default: cudaLaunchKernelEx(&cfg, small_rows_kernel<16>, p); break;
  }
  if (int e = check_launch("small_rows_kernel")) return e;
  long long k2_ctas = blocks;
  if (streamed) {
    k2_ctas = p.nctas;
    static bool sattr = false;
    if (!sattr) {
      const int worst = 226 * 1024;
      cudaFuncSetAttribute(small_stream_kernel<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
      cudaFuncSetAttribute(small_stream_kernel<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
      cudaFuncSetAttribute(small_stream_kernel<12, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
      cudaFuncSetAttribute(small_stream_kernel<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
      cudaFuncSetAttribute(small_stream_kernel<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
      cudaFuncSetAttribute(small_stream_kernel<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
      cudaFuncSetAttribute(small_stream_kernel<12, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
      cudaFuncSetAttribute(small_stream_kernel<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, worst);
      sattr = true;
    }
    cfg.gridDim = dim3((unsigned)p.nctas);
    cfg.dynamicSmemBytes = 1024 + (size_t)p.nslots * 65536 + sops;
    switch (p.kg * 4 + nb) {
      case 17: cudaLaunchKernelEx(&cfg, small_stream_kernel<4, 1>, p, map_phi, map_psi); break;
      case 33: cudaLaunchKernelEx(&cfg, small_stream_kernel<8, 1>, p, map_phi, map_psi); break;
      case 49: cudaLaunchKernelEx(&cfg, small_stream_kernel<12, 1>, p, map_phi, map_psi); break;
      case 65: cudaLaunchKernelEx(&cfg, small_stream_kernel<16, 1>, p, map_phi, map_psi); break;
      case 18: cudaLaunchKernelEx(&cfg, small_stream_kernel<4, 2>, p, map_phi, map_psi); break;
      case 34: cudaLaunchKernelEx(&cfg, small_stream_kernel<8, 2>, p, map_phi, map_psi); break;
      case 50: cudaLaunchKernelEx(&cfg, small_stream_kernel<12, 2>, p, map_phi, map_psi); break;
      default: cudaLaunchKernelEx(&cfg, small_stream_kernel<16, 2>, p, map_phi, map_psi); break;
    }
  } else {
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchKernelEx(&cfg, small_contract_kernel, p);
  }
  int code = check_launch(streamed ? "small_stream_kernel" : "small_contract_kernel");
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
    const char* k2n[8] = {"K2 start", "K2 after wait", "K2 operands in", "K2 mma done", "K2 stores issued", "K2 end",
                          "K2 block 2 top", "K2 block 2 issued"};
    const char* k2s[8] = {"K2 blk2 stage begin", "K2 after wait", "K2 blk0 operands in", "K2 blk2 mma done",
                          "K2 blk2 staged", "K2 end", "K2 blk2 top", "K2 blk2 issued"};
    for (int k : {0, 1, 2, 3, 4, 7, 5}) row(k1n[k], 0, prep_blocks, k);
    if (streamed)
      for (int k : {1, 2, 6, 3, 0, 4, 7, 5}) row(k2s[k], kTraceK1, (int)k2_ctas, k);
    else
      for (int k = 0; k < 6; ++k) row(k2n[k], kTraceK1, (int)k2_ctas, k);
  }
#endif
  return code;
}

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
  return correlate_small(in_dtype, raw1, ld_raw1, raw2, ld_raw2, m, n1, n2, ref_mode1, ref_in1, sigma_in1,
                         ref_mode2, ref_in2, sigma_in2, alpha, substitute_zero_var, norm_const, ops_a, ops_b, ld_ops,
                         ref_out1, sigma_out1, ref_out2, sigma_out2, phi, psi, ld_out, status1, status2, stats, work,
                         stream, 0, nullptr);
}

extern "C" int corr2d_correlate_small_f64_slot(
    int in_dtype, const void* raw1, int64_t ld_raw1, const void* raw2, int64_t ld_raw2,
    int m, int n1, int n2,
    int ref_mode1, const double* ref_in1, const double* sigma_in1,
    int ref_mode2, const double* ref_in2, const double* sigma_in2,
    double alpha, int substitute_zero_var, double norm_const,
    double* ops_a, double* ops_b, int64_t ld_ops,
    double* ref_out1, double* sigma_out1, double* ref_out2, double* sigma_out2,
    double* phi, double* psi, int64_t ld_out,
    int32_t* status1, int32_t* status2, unsigned long long* stats, int32_t* work, void* stream,
    int slot, unsigned long long* pipe) {
  return correlate_small(in_dtype, raw1, ld_raw1, raw2, ld_raw2, m, n1, n2, ref_mode1, ref_in1, sigma_in1,
                         ref_mode2, ref_in2, sigma_in2, alpha, substitute_zero_var, norm_const, ops_a, ops_b, ld_ops,
                         ref_out1, sigma_out1, ref_out2, sigma_out2, phi, psi, ld_out, status1, status2, stats, work,
                         stream, slot, pipe);
}
