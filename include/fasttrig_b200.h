/*
 * fasttrig_b200.h -- C ABI of the B200-native batched fasttrig path.
 *
 * This is the drop-in boundary for the reference's hot path
 *   std::vector<double> fasttrig::proposed_{sin,cos,tan}_batch(
 *       std::span<const double> xs, SqrtMode mode = {})      R:proj/include/fasttrig/kernels.hpp:84-94
 * whose element i is bitwise the scalar proposed_{sin,cos,tan}(xs[i], mode)
 * (kernels.hpp:46-67, contract at :82-83).  The reference is header-only C++
 * with no FFI of its own; the functions below are what a ctypes / cgo / JNI
 * binding of that batch API would bind (INTEGRATION.md shows such stubs), and
 * include/fasttrig/gpu.hpp re-exposes them with the reference's C++ signatures.
 *
 * Conventions
 *   - Plain C types only; every function returns an ft_status (0 = FT_OK) and
 *     never throws.  ft_last_error_string() describes the last failure on the
 *     calling thread.
 *   - "_host" / "_batch" entry points take HOST pointers and block until the
 *     results are in host memory (the reference's semantics).  Pinned host
 *     memory (cudaHostAlloc / ft_host_alloc) is streamed at full PCIe rate;
 *     pageable memory works but is slower.
 *   - Every other entry point takes DEVICE pointers on the current CUDA device
 *     and is asynchronous on `stream` (a cudaStream_t; NULL = legacy default
 *     stream).  Reentrant per stream.
 *   - f64 results are bitwise equal to the reference: identical to
 *     proposed_*(x).  f32 inputs are compared with (float)proposed_*((double)x)
 *     (the reference is double-only): under the default policy FT_F32_ULP2 the
 *     f32 outputs are within 2 ulp of it with the identical segment choice
 *     (the north-star tolerance; all 2^32 inputs are checked in the GPU
 *     tests); under FT_F32_BITWISE they are bit-identical to it.
 *   - Non-finite x yields a quiet NaN (reduction.hpp:60-62); tan inside the
 *     pole window |red - pi/2| < 1e-3 yields a signed infinity (kernels.hpp:62-64).
 */
#ifndef FASTTRIG_B200_H_
#define FASTTRIG_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FT_ABI_VERSION 2

typedef enum ft_status {
  FT_OK = 0,
  FT_ERR_INVALID_ARG = 1, /* bad dtype / mask / n_terms / null or misaligned pointer */
  FT_ERR_CUDA = 2,        /* CUDA runtime error (see ft_last_error_string) */
  FT_ERR_OOM = 3,         /* device or pinned allocation failed */
  FT_ERR_NO_DEVICE = 4    /* no CUDA device visible */
} ft_status;

typedef enum ft_dtype { FT_F32 = 0, FT_F64 = 1 } ft_dtype;

/* Output mask bits: which of sin / cos / tan a fused call writes. */
enum { FT_OUT_SIN = 1u, FT_OUT_COS = 2u, FT_OUT_TAN = 4u };

/* Mirrors fasttrig::SqrtMode (fisr.hpp:14-24) field for field:
 *   method 0 = exact  (1.0/std::sqrt(v); tan divides),
 *   method 1 = fisr   (magic 0x5fe6eb50c7b537a9 + newton_steps Newton steps).
 * The reference default SqrtMode{} is {FT_SQRT_FISR, 1}.  newton_steps is used
 * verbatim, as a SqrtMode aggregate would be (fisr(s) clamps s<1 to 1 on the
 * C++ side before it gets here). */
typedef enum ft_sqrt_method { FT_SQRT_EXACT = 0, FT_SQRT_FISR = 1 } ft_sqrt_method;
typedef struct ft_sqrt_mode {
  int32_t method;
  int32_t newton_steps;
} ft_sqrt_mode;

/* Input distributions for ft_gen_inputs (counter-based SplitMix64). */
typedef enum ft_dist {
  FT_DIST_UNIFORM = 0,   /* x = lo + (hi - lo) * u,  u = (z >> 11) * 2^-53        */
  FT_DIST_TAN_STRESS = 1 /* x = (2k+1) pi/2 + delta, k ~ U{lo..hi} (integers),
                            delta ~ N(0, 1e-3) clipped to |delta| <= 0.05        */
} ft_dist;

/* Parity / error statistics of one checked batch (K3).  Index j: 0 sin, 1 cos,
 * 2 tan.  Maxima of non-negative doubles and all counters combine across
 * shards/GPUs by max / wrap-around sum, so any sharding gives the same totals. */
typedef struct ft_stats {
  uint64_t n_checked;
  uint64_t max_ulp[3];          /* vs the oracle, in units of the output dtype */
  uint64_t n_over_tol[3];       /* elements with ulp distance > ulp_tol        */
  uint64_t seg_mismatch[2];     /* [0] sin/cos segment, [1] tan segment       */
  uint64_t n_inf[3];
  uint64_t n_nan[3];
  uint64_t n_finite_libm[3];    /* elements entering the vs-libm statistics   */
  uint64_t checksum[3];         /* sum of output bit patterns (NaN canonical) */
  double max_abs_vs_oracle[3];  /* finite pairs only                          */
  double max_abs_vs_libm[3];    /* finite outputs only                        */
  double max_rel_vs_libm[3];    /* |libm| > 1e-12 guard    */
  double sum_abs_vs_libm[3];
  double sum_rel_vs_libm[3];
  uint64_t n_bit_mismatch[3];   /* raw bit patterns differ (NaNs canonical; sees +0 vs -0) */
} ft_stats;

/* ---- host-pointer entry points: the reference batch API (kernels.hpp:84-94) ---- */

/* proposed_{sin,cos,tan}_batch: out[i] = proposed_*(xs[i], mode). */
int ft_proposed_sin_batch(const double* xs, size_t n, ft_sqrt_mode mode, double* out);
int ft_proposed_cos_batch(const double* xs, size_t n, ft_sqrt_mode mode, double* out);
int ft_proposed_tan_batch(const double* xs, size_t n, ft_sqrt_mode mode, double* out);

/* Fused host-pointer form: reads x once, writes the outputs selected by mask
 * (unselected output pointers may be NULL).  Streams H2D / kernel / D2H in
 * chunks on the current device. */
int ft_proposed_batch_host(ft_dtype dtype, const void* x, size_t n, unsigned mask,
                           ft_sqrt_mode mode, void* sin_out, void* cos_out, void* tan_out);
int ft_taylor_batch_host(ft_dtype dtype, const void* x, size_t n, unsigned mask, int n_terms,
                         void* sin_out, void* cos_out, void* tan_out);

/* f32 evaluation policy (process-wide; default FT_F32_ULP2).
 *   FT_F32_ULP2     <= 2 ulp of (float)proposed_*((double)x), identical segment
 *                   choice; one signed reduction and FMA-contracted evaluation
 *                   for |x| < 2^16, bit-exact elsewhere.
 *   FT_F32_BITWISE  bit-identical to (float)proposed_*((double)x).
 * Taylor f32 calls follow it for n_terms 5, 7 and 9.  f64 is always bitwise. */
typedef enum ft_f32_policy { FT_F32_ULP2 = 0, FT_F32_BITWISE = 1 } ft_f32_policy;
int ft_set_f32_policy(int policy);
int ft_get_f32_policy(void);

/* Number of GPUs the host-pointer entry points spread one call over: arrays of
 * at least 4 Mi elements are split into that many contiguous shards, each
 * streamed through its own device (round robin from the current one) by its
 * own host thread.  Default 1 (the current device); n <= 0 selects every
 * visible device.  Results are identical for any setting. */
int ft_set_host_devices(int n);
int ft_get_host_devices(void);

/* ---- device-pointer entry points (asynchronous on `stream`) ---- */

/* K1: fused proposed sin/cos/tan (kernels.hpp:46-67 per element). */
int ft_proposed_eval(ft_dtype dtype, const void* x, size_t n, unsigned mask, ft_sqrt_mode mode,
                     void* sin_out, void* cos_out, void* tan_out, void* stream);

/* K1 with the per-element segment choice (segments.hpp:70-73) written out:
 * seg_sc[i] = sin/cos segment, seg_t[i] = tan segment or 255 inside the pole
 * window.  Either seg pointer may be NULL.  For parity testing. */
int ft_proposed_eval_seg(ft_dtype dtype, const void* x, size_t n, unsigned mask,
                         ft_sqrt_mode mode, void* sin_out, void* cos_out, void* tan_out,
                         uint8_t* seg_sc, uint8_t* seg_t, void* stream);

/* K2: Taylor comparator, n_terms nonzero terms in [1, 9]. */
int ft_taylor_eval(ft_dtype dtype, const void* x, size_t n, unsigned mask, int n_terms,
                   void* sin_out, void* cos_out, void* tan_out, void* stream);

/* Device restatement of the reference (plain IEEE division, no fast paths):
 * the device-side oracle used by K3 when no host oracle array is supplied.
 * kind 0 = proposed (mode), 1 = Taylor (n_terms). */
int ft_mirror_eval(ft_dtype dtype, const void* x, size_t n, unsigned mask, int kind,
                   ft_sqrt_mode mode, int n_terms, void* sin_out, void* cos_out, void* tan_out,
                   uint8_t* seg_sc, uint8_t* seg_t, void* stream);

/* K3: parity + error reduction.  Compares the outputs (sin/cos/tan, per mask)
 * with oracle arrays ref_* when given (device pointers, same dtype), else with
 * the device restatement recomputed on the fly; optionally checks segment
 * choices.  Accumulates into *stats_dev (device memory; zero it first with
 * ft_stats_reset).  Warp-shuffle reduction, one atomic per warp. */
int ft_parity_reduce(ft_dtype dtype, const void* x, size_t n, unsigned mask, int kind,
                     ft_sqrt_mode mode, int n_terms, const void* sin_out, const void* cos_out,
                     const void* tan_out, const void* ref_sin, const void* ref_cos,
                     const void* ref_tan, const uint8_t* seg_sc, const uint8_t* seg_t,
                     uint64_t ulp_tol, ft_stats* stats_dev, void* stream);
int ft_stats_reset(ft_stats* stats_dev, void* stream);

/* K4: seeded inputs generated in place.  Element i of the shard is element
 * (offset + i) of the global stream, so any sharding reproduces one array. */
int ft_gen_inputs(ft_dtype dtype, int dist, double lo, double hi, uint64_t seed, uint64_t offset,
                  size_t n, void* x, void* stream);

/* K5: write a buffer of twice the L2 size (timing hygiene between reps). */
int ft_l2_flush(void* stream);

/* ---- utilities ---- */
int ft_host_alloc(void** p, size_t bytes);  /* pinned host memory */
int ft_host_free(void* p);
/* The device-resident constant table: 6 x {a,b,c,d,X,Y,Z} then 7 knots
 * (segments.hpp:14-66), bit-identical to fasttrig::segment_table. */
int ft_segment_table(double* out49);
/* Taylor coefficients sin/cos/tan, 9 each. */
int ft_taylor_coeffs(double* sin9, double* cos9, double* tan9);
/* Monotone thresholds of the fast reduction: out8[0..3] = quad[3],
 * guard found by host bisection against IEEE division/subtraction; out8[4..7]
 * = the same constants as compiled into the kernels (must be identical). */
int ft_thresholds(double* out8);
/* The segment table as held in device constant memory, read back from the GPU
 * (same layout as ft_segment_table).  unit: 0 = the K1/K2 kernels' copy, 1 =
 * K3's, 2 = K4/K5's, 3 = the C-ABI unit's.  Synchronous. */
int ft_device_const_table(int unit, double* out49);
/* The shared-memory segment rows a K1 block stages, copied out by a kernel.
 * kind 0 = bit-exact rows: 8 x 80 bytes (a,b,c,d,X,Y,Z as doubles, the
 * bracket's two high words as int32, the exact bracket as two doubles);
 * kind 1..7 = the relaxed f32 rows for that output mask: 8 x 48 bytes in the
 * first 384 bytes (a,b,c,d as doubles, the two bracket high words, 8 bytes of
 * padding).  Synchronous. */
int ft_device_rows(int kind, void* out640);
/* Free the host-pointer pipeline (streams, device slots, pinned staging) and
 * the L2-flush buffer of `device` (-1: every device).  They are re-created on
 * demand by the next call.  Not to be called concurrently with host-pointer
 * calls on that device. */
int ft_release(int device);
/* Number of K1/K2/K3/K4/K5 launches issued by this process so far. */
uint64_t ft_launch_count(void);
const char* ft_last_error_string(void);
int ft_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FASTTRIG_B200_H_ */
