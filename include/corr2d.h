/*
 * corr2d.h -- C ABI of libcorr2d.so, the B200 (sm_100a) implementation of the
 * corr2D Fourier-route hot path (arXiv 1808.00685; reference Python package
 * `corrtwo` 0.1.0, files cited relative to /root/reference/pkg/src/corrtwo/).
 *
 * Plain C: raw device pointers, sizes and a cudaStream_t (passed as void*).
 * No torch types.  Every entry point returns CORR2D_OK (0) or a status code;
 * corr2d_last_error() returns the message of the last failure on the calling
 * thread.  The Python drop-in (paper_1808_00685_b200/_abi.py) maps the codes
 * onto the reference's exception classes (errors.py:4-36):
 *   CORR2D_ERR_DATA -> DataError, CORR2D_ERR_NUMERIC / _OOM -> NumericError.
 *
 * Data conventions (match the reference layouts):
 *   raw intensities : m_in x n, row-major, row j = spectrum at t_j, leading
 *                     dimension ld_raw (elements)              dataset.py:54-56
 *   dynamic values  : m x n row-major, float64                 preprocess.py:90-120
 *   half spectra    : K x n complex128 interleaved (re, im), K = m/2 + 1
 *                                                              fourier.py:61-82
 *   sync / async    : n1 x n2 row-major planes (float64, or float32 for the
 *                     fp32 path), leading dimension ld_out     fourier.py:123
 *
 * Packed spectra (the intermediate between the two kernels):
 * for each spectral channel a row of mp >= m "slots" (real packing of the
 * half spectrum, depth exactly m, zero padded to mp):
 *   slot s <  K      : Re Y(w = s)
 *   slot K <= s < m  : Im Y(w = s - K + 1)
 * Operand A_phi carries Norm*weight(w)*[Re | Im], A_psi Norm*weight(w)*[Im | -Re]
 * and B the plain [Re | Im]; then sync = A_phi . B^T and async = A_psi . B^T
 * exactly reproduce  Norm * sum_w weight(w) Y1 conj(Y2)  (fourier.py:107-123).
 */
#ifndef CORR2D_H
#define CORR2D_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CORR2D_ABI_VERSION 3

enum corr2d_status {
  CORR2D_OK = 0,
  CORR2D_ERR_DATA = 1,        /* invalid argument / shape       -> DataError    */
  CORR2D_ERR_NUMERIC = 2,     /* non-finite, zero variance      -> NumericError */
  CORR2D_ERR_OOM = 3,         /* device allocation failed       -> NumericError */
  CORR2D_ERR_CUDA = 4,        /* CUDA runtime / launch failure  -> RuntimeError */
  CORR2D_ERR_UNSUPPORTED = 5  /* shape outside the kernel's range               */
};

enum corr2d_dtype { CORR2D_F64 = 0, CORR2D_F32 = 1 };

enum corr2d_resample { CORR2D_RESAMPLE_NONE = 0, CORR2D_RESAMPLE_LINEAR = 1, CORR2D_RESAMPLE_MATRIX = 2 };

enum corr2d_pack {
  CORR2D_PACK_NONE = 0,
  CORR2D_PACK_F64 = 1,       /* float64 operands (fp64 DMMA contraction)            */
  CORR2D_PACK_BF16X2 = 2,    /* bf16 hi/lo, k-block interleaved (bf16x3 tcgen05 contraction) */
  CORR2D_PACK_F64_TIME = 3,  /* float64 time-domain values, no DFT (Hilbert route, hilbert.py) */
  CORR2D_PACK_F16F8 = 4,     /* scaled fp16 hi + e4m3 hi / residual (fp16+fp8 tcgen05 contraction) */
  CORR2D_PACK_F64_GAUSS = 5  /* float64 three-product (Gauss) operands: corr2d_contract_f64_gauss */
};

enum corr2d_ref_mode { CORR2D_REF_MEAN = 0, CORR2D_REF_PROVIDED = 1, CORR2D_REF_NONE = 2 };

/* pack role bits */
#define CORR2D_ROLE_A 1      /* write A_phi and A_psi (row operand, dataset 1)  */
#define CORR2D_ROLE_B 2      /* write B (column operand, dataset 2)             */

/* status word layout written by corr2d_prep (device int32[4]) */
#define CORR2D_ST_NONFINITE 0     /* count of non-finite raw values              */
#define CORR2D_ST_ZEROVAR 1       /* count of zero-variance channels (alpha > 0)  */
#define CORR2D_ST_FIRST_ZEROVAR 2 /* INT32_MAX - smallest zero-variance channel, 0 if none */

/* ---------------------------------------------------------------- misc ---- */
const char* corr2d_last_error(void);
int corr2d_abi_version(void);
/* Number of SMs, compute capability of `device`.  Fails with CORR2D_ERR_CUDA
 * when no device is present. */
int corr2d_device_info(int device, int* sms, int* cc_major, int* cc_minor);
/* Packed depth (slots per channel) the contraction kernels need for m.  A
 * CORR2D_PACK_BF16X2 row stores every slot twice (hi and lo), i.e. 2 * depth
 * bf16 values. */
int corr2d_packed_depth(int m, int pack_kind);
/* Prime/radix factorisation used by the perturbation-axis FFT (for tests). */
int corr2d_fft_factors(int m, int* factors, int max_factors);

/* ------------------------------------------------------ K1: preprocess ---- */
/*
 * One pass over the raw intensities, one CTA per tile of spectral channels:
 *   resample (preprocess.py:155-195; linear via host-computed idx/frac exactly
 *   as _interp_linear :147-152, or a dense m x m_in matrix for the natural
 *   spline :174-175) -> reference (mean :123-125 or provided :56-64) ->
 *   sigma about it (:198-211, only when alpha > 0; sigma_out receives the
 *   sigma BEFORE zero-variance substitution so the host can name the dead
 *   channels) -> divide by sigma**alpha
 *   (:214-259) -> [optional] real DFT of length m along the perturbation axis
 *   (fourier.py:73, mixed-radix Stockham in shared memory) -> packing.
 *
 * ref_mode CORR2D_REF_NONE treats `raw` as already-dynamic values (no
 * reference subtraction): with alpha = 0 the entry used by dft_channels /
 * correlate_ft on DynamicSpectra, with sigma_in the one used by apply_scaling.
 * sigma_in (optional, n) replaces the computed sigma.
 * CORR2D_PACK_F64_TIME (Hilbert route, hilbert.py:92-115): no DFT; slot s < m of
 * a row holds the dynamic value y(t_s) -- A_phi = norm_const * y (ROLE_A), B = y
 * (ROLE_B), zero padded to mp = corr2d_packed_depth(m, ...); a_psi is unused
 * (the caller forms A_psi = -norm_const * N y with one corr2d_contract_f64 call
 * against the Hilbert-Noda matrix, since async = Y1^T N Y2 = (-N Y1)^T Y2).
 * Packing: ld_pack is the row pitch of the packed operands in elements
 * (>= mp for F64; for BF16X2 and F16F8, in 2-byte units, >= 2 * mp + 64 and a
 * multiple of 64; both layouts are described at corr2d_contract_tc).  split_plane is unused (ABI v1 kept
 * the bf16 lo values in a separate plane; v2 interleaves them).
 * CORR2D_PACK_F64_GAUSS: the complex product Y1 conj(Y2) with THREE real
 * products instead of four (Gauss).  With a = Norm w Re Y1, b = Norm w Im Y1,
 * c = Re Y2, d = -Im Y2 per bin: P1 = (a + b) c, P2 = a (d - c), P3 = b (c + d),
 * sync = P1 - P3, async = P1 + P2.  A row (a_phi, ROLE_A) and a B row (b,
 * ROLE_B) hold three segments of kg = corr2d_packed_depth(m, GAUSS) / 3 slots:
 *   seg 1  A = a + b, B = c      : DC bin at slot 0, interior bins 1..I at 1..I
 *   seg 2  A = a,     B = d - c  : the same bins
 *   seg 3  A = -b,    B = c + d  : interior bins at 0..I-1; even m: the Nyquist
 *                                  bin at slot I as A = a, B = c
 * (I = ceil(m/2) - 1 interior bins; unused slots 0; a_psi is unused).  The DC /
 * Nyquist bins are real, so the segments reproduce the exact weighted
 * half-spectrum sum with 3 kg <= 3/4 of the 2 m multiply-adds of CORR2D_PACK_F64.
 * Any output pointer may be NULL.  `status` (device int32[4]; reset on the
 * stream by this call) receives the counters above; the host raises the
 * reference's errors from them after the stream synchronises.
 */
int corr2d_prep(
    int in_dtype, const void* raw, int64_t ld_raw, int m_in, int n,
    int resample_kind, const int32_t* lin_idx, const double* lin_frac,
    const double* resample_matrix, int m,
    int ref_mode, const double* ref_in, const double* sigma_in, double alpha, int substitute_zero_var,
    double norm_const, int pack_kind, int pack_roles,
    void* a_phi, void* a_psi, void* b, int64_t ld_pack, int64_t split_plane,
    double* values_out, int64_t ld_values, double* half_out,
    double* ref_out, double* sigma_out, int32_t* status, void* stream);

/* ------------------------------------------------------- K2: contract ---- */
/*
 * sync/async = A_phi . B^T / A_psi . B^T over packed depth mp
 * (fourier.py:107-123: weighted half-spectrum cross sum x Norm, split).
 * Output rows [row0, row1) of the n1 x n2 result are written to
 * phi/psi + (i - row0) * ld_out (a rank's row shard, engine_core.py:106-112).
 * homo != 0: the row operand and the column operand are the same dataset;
 * tiles in the shard's own diagonal square are computed once and mirrored,
 * so sync is exactly symmetric and async exactly skew-symmetric with a zero
 * diagonal (dataset.py:159-170).  stats (device uint64[3], reset on the
 * stream by this call) receives
 * [0] = max|sync| and [1] = max|async| as IEEE bits (uint64), [2] = nonzero iff
 * an output is non-finite (the number of flagging threads; engine_core.py:139-140).
 */
int corr2d_contract_f64(
    const double* a_phi, const double* a_psi, const double* b, int64_t ld_pack,
    int n1, int n2, int mp, int homo, int row0, int row1, int64_t tile0, int64_t tile1,
    double* phi, double* psi, int64_t ld_out, unsigned long long* stats, void* stream);

/*
 * The same contraction from CORR2D_PACK_F64_GAUSS operands (a: A rows, b: B
 * rows, 3 kg slots each, kg a multiple of 4): one accumulator runs P1 over
 * segment 1, is copied, then segment 3 goes into the sync accumulator and
 * segment 2 into the async one -- 25 % fewer FP64 tensor-core MMAs than
 * corr2d_contract_f64 for the same map.  Tiles, shards, mirroring, stats and
 * errors as corr2d_contract_f64.  Reference: fourier.py:107-123.
 */
int corr2d_contract_f64_gauss(
    const double* a, const double* b, int64_t ld_pack, int n1, int n2, int kg, int homo,
    int row0, int row1, int64_t tile0, int64_t tile1,
    double* phi, double* psi, int64_t ld_out, unsigned long long* stats, void* stream);

/*
 * fp32 path (tcgen05 tensor cores).  Operands are K1's CORR2D_PACK_BF16X2 or
 * CORR2D_PACK_F16F8 rows: per channel three thirds [Re' | Im' | -Im'] of
 * hp = mp/3 slots (Re'[s] = Re Y(s), Im'[0] = Re Y(m/2) for even m else 0,
 * Im'[s] = Im Y(s)), every slot scaled by sqrt(Norm * weight).  Each third is
 * a run of 32-slot blocks of 128 bytes, so one 128-byte TMA box row feeds a
 * whole k-block; row pitch ld_pack (2-byte units) >= 2*mp + 64, multiple of 64.
 *   BF16X2: block = [bf16 hi of the 32 slots | bf16 lo], x = hi + lo; products
 *     hi*hi + hi*lo + lo*hi (tcgen05.mma kind::f16).  Row pad at element 2*mp:
 *     float32 (hi + lo) of Re'[0] and Im'[0].
 *   F16F8: the channel is scaled by sc = 2^s (max|x| sc in [2^7, 2^8)); block =
 *     [fp16(x sc) * 2^5 of the 32 slots (64 B) | e4m3(x sc) (32 B) |
 *     e4m3((x sc - fp16(x sc)) * 2^10) (32 B)]; products hi*hi (kind::f16) +
 *     e4m3 hi * e4m3 residual both ways (kind::f8f6f4, twice the rate), all at
 *     scale 2^10 sc_i sc_j, undone in the epilogue.  Row pad at element 2*mp:
 *     float32 Re'[0], Im'[0] (unscaled) and 2^-(s+5).
 * FP32 accumulators in TMEM; the even-m Nyquist x DC cross term is removed in
 * the epilogue.  a == b for homo.  Same row / homo / stats contract as
 * corr2d_contract_f64, shard bounds multiples of 128.
 */
int corr2d_contract_tc(
    int pack_kind, const void* a, const void* b, int64_t ld_pack,
    int n1, int n2, int mp, int m, int homo, int row0, int row1, int64_t tile0, int64_t tile1,
    float* phi, float* psi, int64_t ld_out, unsigned long long* stats, void* stream);

/* corr2d_contract_tc(CORR2D_PACK_BF16X2, ...); split_a / split_b are unused (ABI v1). */
int corr2d_contract_bf16x3(
    const void* a, const void* b, int64_t ld_pack, int64_t split_a, int64_t split_b,
    int n1, int n2, int mp, int m, int homo, int row0, int row1, int64_t tile0, int64_t tile1,
    float* phi, float* psi, int64_t ld_out, unsigned long long* stats, void* stream);

/*
 * Number of tiles in the enumeration corr2d_contract_f64 / _bf16x3 would use for
 * this call (the [tile0, tile1) range of the contract calls indexes it): the
 * unit of the multi-GPU tile-range partition.  -1 on bad arguments.  For
 * pack_kind BF16X2 / F16F8 and a whole-map call with ld_out % 4 == 0 this is the
 * 2-SM (CTA-pair) enumeration; CORR2D_BF16_1SM=1 in the environment forces the
 * 1-SM kernel.
 */
int64_t corr2d_contract_tile_count(int pack_kind, int n1, int n2, int homo, int row0, int row1,
                                   int64_t ld_out);

/* ----------------------------------- small m: the whole call, one C call ---- */
/*
 * fp64, 2 <= m <= 32, no resampling (cfg1 / cfg2 shapes): preprocess + DFT +
 * contraction of a whole map (csrc/small_path.cu).  Replaces the corr2d_prep +
 * corr2d_contract_f64_gauss sequence that preprocess_dataset / dft_channels /
 * correlate_ft (preprocess.py:262-275, fourier.py:61-125) map onto; same
 * argument meanings as those two calls.  Two kernels chained by programmatic
 * dependent launch: K1 once per channel (64 channels per CTA, the Gauss
 * operand rows of every role as one FP64 tensor-core product, into ops_a /
 * ops_b), then a persistent contraction over the 64 x 64 output blocks
 * (corr2d_small_block_count blocks; homo: the upper triangle, mirrored) with
 * TMA tensor stores of the planes (planes that are not 16-B aligned with an
 * even ld_out: one CTA per block, plain stores).  With ops_a or ops_b NULL the
 * call is ONE kernel instead: each CTA centres its blocks' channels and builds
 * their operand rows in shared memory.  Within one call no CTA waits for
 * another CTA (pipelined calls: see corr2d_correlate_small_f64_slot).
 *   ops_a / ops_b      : device operand scratch, n1 (resp. n2; homo: n1) rows
 *                       of ld_ops doubles, 16-B aligned, ld_ops ==
 *                       corr2d_small_ops_depth(m) (3 kg Gauss slots padded to
 *                       4 or 12 mod 16 doubles: a 64-row block is one
 *                       contiguous run, fragment loads conflict-free); NULL
 *                       selects the one-kernel variant
 *   ref_out* / sigma_out* : as corr2d_prep (either may be NULL)
 *   status1 / status2  : device int32[4] each, the corr2d_prep status words
 *                       (status2 unused when homo); written by the call
 *   stats              : device uint64[3], as corr2d_contract_f64; written by the call
 *   work               : device int32[16], zero-filled by the caller ONCE before
 *                       the first call on it: K1's status accumulators, left
 *                       zero by every call (the contraction grid publishes and
 *                       resets them).  One work buffer per concurrently running
 *                       call.
 * The first call for a given m on a device builds a small DFT table (must not
 * be inside a CUDA graph capture).
 */
int64_t corr2d_small_block_count(int n1, int n2, int homo);
/* Kernels one corr2d_correlate_small_f64 call WITH operand scratch launches:
 * 2 (K1 + contraction); a call with ops_a / ops_b NULL launches 1 (the fused
 * kernel); -1 on bad sizes. */
int corr2d_small_launches(int n1, int n2, int homo);
int corr2d_small_ops_depth(int m);
int corr2d_correlate_small_f64(
    int in_dtype, const void* raw1, int64_t ld_raw1, const void* raw2, int64_t ld_raw2,
    int m, int n1, int n2,
    int ref_mode1, const double* ref_in1, const double* sigma_in1,
    int ref_mode2, const double* ref_in2, const double* sigma_in2,
    double alpha, int substitute_zero_var, double norm_const,
    double* ops_a, double* ops_b, int64_t ld_ops,
    double* ref_out1, double* sigma_out1, double* ref_out2, double* sigma_out2,
    double* phi, double* psi, int64_t ld_out,
    int32_t* status1, int32_t* status2, unsigned long long* stats, int32_t* work, void* stream);
/*
 * The same call, PIPELINED with the previous call of the same plan on the
 * same stream (what corr2d() / correlate_ft() use): consecutive calls pass
 * alternate scratch sets -- ops_a / ops_b, stats, work, status1 / status2 --
 * as slot 0 / 1, and one `pipe` (device uint64[16], zero-filled once; its
 * monotonic counters order the calls).  No kernel then waits for a whole
 * earlier grid: K1 of call k runs while earlier calls' contractions do (it
 * writes its slot once that slot's previous use, call k-2, is complete), the
 * contraction starts once K1's CTAs have all written their rows, and it loads
 * and contracts before it waits for every earlier call's stores to complete
 * -- so the calls' planes are written in call order.  Calls that take the
 * one-kernel or the plain-store variant ignore the pipe (they serialise as
 * usual).
 */
int corr2d_correlate_small_f64_slot(
    int in_dtype, const void* raw1, int64_t ld_raw1, const void* raw2, int64_t ld_raw2,
    int m, int n1, int n2,
    int ref_mode1, const double* ref_in1, const double* sigma_in1,
    int ref_mode2, const double* ref_in2, const double* sigma_in2,
    double alpha, int substitute_zero_var, double norm_const,
    double* ops_a, double* ops_b, int64_t ld_ops,
    double* ref_out1, double* sigma_out1, double* ref_out2, double* sigma_out2,
    double* phi, double* psi, int64_t ld_out,
    int32_t* status1, int32_t* status2, unsigned long long* stats, int32_t* work, void* stream,
    int slot, unsigned long long* pipe);

/* ------------------------------------------ homo map: device -> host ---- */
/*
 * Device -> host copy of a homo map's planes (n x n, leading dimensions ld_dev
 * on the device, ld_host on the host) that sends part of the lower triangle as
 * its mirror image only:
 * row band [r0, r0 + band) travels as columns [split, n), split = fill_pct %
 * of r0 (rounded down to 64; 0 = a plain full copy, 100 = the upper triangle
 * only), and `threads` host threads fill the band's columns [0, split) as
 * sync(i, j) = sync(j, i), async(i, j) = -async(j, i) from rows that already
 * landed, while later bands are in flight (csrc/fetch.cu).  band: a positive multiple of 256 (diagonal
 * blocks travel whole).  Ordered after the work queued on `stream`; returns
 * once both host planes are complete; *d2h_bytes (may be NULL) = bytes moved.
 * Bit-identical to a full-plane copy of a map any homo contraction wrote.
 * Replaces the reference's host-side result hand-off of a homo map
 * (fourier.py:123 / dataset.py:133-170 assemble the full planes on the host).
 */
int corr2d_fetch_mirrored(int dtype, const void* d_sync, const void* d_async, int64_t ld_dev, int n,
                          void* h_sync, void* h_async, int64_t ld_host, int band, int fill_pct, int threads,
                          int64_t* d2h_bytes, void* stream);

/* ------------------------------------------------- K3: peak candidates ---- */
/*
 * max |x| over an n1 x n2 plane (dtype CORR2D_F64 / CORR2D_F32, leading
 * dimension ld) into *out_dev (device double, reset by this call).  Used by
 * find_peaks for maps that did not come with K2's fused statistics.
 */
int corr2d_plane_absmax(int dtype, const void* x, int64_t ld, int n1, int n2, double* out_dev, void* stream);

/*
 * Cross-peak candidates of a correlation map (analysis.py:136-201): strict
 * 8-neighbourhood local maxima of |sync| above thr_sync OR of |async| above
 * thr_async, the map padded with -inf (analysis.py:136-149); homo != 0 keeps
 * k > i only.  Each candidate's row-major linear index i * n2 + k is appended
 * to out_idx (device int64[capacity]) in no particular order; *count (device
 * uint64, reset by this call) receives the total, which may exceed capacity
 * (the caller then retries with a larger buffer).  Pass thr = +inf to exclude
 * a plane whose maximum is 0 (analysis.py:186-194).
 */
int corr2d_find_peaks(int dtype, const void* sync, const void* asyn, int64_t ld, int n1, int n2, int homo,
                      double thr_sync, double thr_async, int64_t* out_idx, int64_t capacity,
                      unsigned long long* count, void* stream);

/* ------------------------------------- result serialization (host code) ---- */
/*
 * repr(float(x)) of the reference's format_number (dataset.py:34-36): shortest
 * round-trip decimal digits laid out with CPython's repr rules.  x[0..n) are
 * formatted back to back into out (capacity cap bytes); offsets[i + 1] is the
 * end of item i (offsets has n + 1 entries).
 */
int corr2d_format_repr(const double* x, int64_t n, char* out, int64_t cap, int64_t* offsets);

/*
 * Rows [r0, r1) of a serialized correlation table (write_correlation,
 * dataset.py:303-341): matrix-pair lines "repr(nu1)<d>repr(m[i,0])<d>..." or,
 * with long_form != 0, one "nu1,nu2,sync,async" line per element (matrix =
 * sync, matrix2 = async).  Host pointers; dtype CORR2D_F64 or CORR2D_F32
 * (float32 values are written as the float64 they convert to, like
 * repr(float(np.float32))).  `threads` host threads.  *written receives the
 * byte count; if it exceeds cap the call fails and nothing is copied.
 */
int corr2d_format_rows(int dtype, const double* axis1, const double* axis2, const void* matrix,
                       const void* matrix2, int64_t ld, int n2, int r0, int r1, char delim, int long_form,
                       int threads, char* out, int64_t cap, int64_t* written);

#ifdef __cplusplus
}
#endif
#endif /* CORR2D_H */
