// ft_core.cuh -- constants, the segment table and the per-element device math
// for the batched piecewise sin/cos/tan path (arXiv 2502.10831).
//
// Two families of device functions live here:
//
//   mirror_*  A literal restatement of the reference scalar code
//             (R:proj/include/fasttrig/{fisr,reduction,segments,kernels}.hpp),
//             with every binary64 operation written as an explicitly rounded
//             intrinsic (__dmul_rn/__dadd_rn/__ddiv_rn/__dsqrt_rn) so that
//             nvcc can never contract a mul+add into an FMA.  Used by the
//             device-side checker (K3) and as the reference for the fast path.
//
//   fast_*    The production path used by K1/K2.  Same results bit for bit,
//             fewer FP64-pipe instructions:
//               * a/2pi via Markstein's correction instead of IEEE division
//                 (RN(1/2pi) has relative error 0.206*2^-53, so RN(a*y) is
//                 within 0.912 ulp of a/2pi, and one FMA correction returns
//                 exactly RN(a/2pi) -- Markstein 1990);
//               * a/pi = 2 * (a/2pi) exactly, so the tangent quotient is a
//                 doubling of the sine quotient (no second division);
//               * floor(RN(r/(pi/2))) by three threshold compares (RN(r/c) is
//                 monotone in r; thresholds found once on the host by
//                 bisection against IEEE division, see ft_capi.cu);
//               * the tan pole guard |red - pi/2| < 1e-3 as one threshold
//                 compare (monotone in red on [0, pi/2]);
//               * sign multiplications by +-1.0 as sign-bit XORs and 0.5*v as
//                 an exponent decrement (both exact for the values they see);
//               * the segment row from one fma.rz guess validated by a bracket
//                 compare, shared by tan; elements the bracket cannot certify
//                 (near knots, the reference's r clamps, +0, NaN) are redone
//                 by the mirror path -- so no r / red clamp and no isfinite
//                 branch on the fast path (see fast_proposed);
//               * the quadrant / tan-fold compares and the bracket on the
//                 high words only (integer pipe): an r sharing a threshold's
//                 high word may fold wrongly, but then lands in no bracket;
//               * 2*q1 as an exponent increment, the FISR Newton step as
//                 y*fma(-0.5, (v*y)*y, 1.5) (same roundings, see fisr_newton).
//             All products/sums that the reference rounds separately stay
//             separately rounded.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace ft {

// ---- constants (R:reduction.hpp:18-20, kernels.hpp:17, fisr.hpp:26) ----
constexpr double kPi = 0x1.921fb54442d18p+1;  // std::numbers::pi
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kHalfPi = 0.5 * kPi;
constexpr double kInvTwoPi = 1.0 / kTwoPi;  // RN(1/(2pi)); Markstein reciprocal
constexpr double kTanPoleGuard = 1e-3;
constexpr std::uint64_t kFisrMagic = 0x5fe6eb50c7b537a9ull;
constexpr std::uint64_t kQuietNaN = 0x7ff8000000000000ull;  // std::numeric_limits<double>::quiet_NaN()

// ---- segment table (R:segments.hpp:14-66), built by the same constexpr
// arithmetic as the reference so the bits cannot drift (checked in tests) ----
struct Coeffs {
  double a, b, c, d, X, Y, Z;
};
struct Table {
  Coeffs seg[6];
  double knots[7];
};

constexpr Table make_table() {
  // segments.hpp:33-40 integer degree-space coefficients.
  constexpr double deg[6][4] = {{11.0, 0.0, -1.0, 632.0},   {10.0, 10.0, -4.0, 657.0},
                                {6.0, 46.0, -5.0, 541.0},   {10.0, 217.0, -13.0, 1252.0},
                                {4.0, 297.0, -10.0, 910.0}, {1.0, 542.0, -11.0, 990.0}};
  Table t{};
  const double deg_per_rad = 180.0 / kPi;  // segments.hpp:42
  for (int k = 0; k < 6; ++k) {            // segments.hpp:44-50
    const double a = deg[k][0] * deg_per_rad;
    const double b = deg[k][1];
    const double c = deg[k][2] * deg_per_rad;
    const double d = deg[k][3];
    t.seg[k] = Coeffs{a, b, c, d, a * a + c * c, 2.0 * (a * b + c * d), b * b + d * d};
  }
  // segments.hpp:60
  t.knots[0] = 0.0;
  t.knots[1] = kPi / 12.0;
  t.knots[2] = kPi / 6.0;
  t.knots[3] = kPi / 4.0;
  t.knots[4] = kPi / 3.0;
  t.knots[5] = 5.0 * kPi / 12.0;
  t.knots[6] = kPi / 2.0;
  return t;
}
constexpr Table kTable = make_table();

// ---- Taylor coefficients: exact rationals, one
// rounding each; n! for n <= 17 is exact in binary64 ----
struct TaylorCoeffs {
  double sin_c[9], cos_c[9], tan_c[9];
};
constexpr TaylorCoeffs make_taylor() {
  TaylorCoeffs t{};
  double f[18]{};
  f[0] = 1.0;
  double fact = 1.0;
  for (int k = 1; k < 18; ++k) {
    fact = fact * static_cast<double>(k);
    f[k] = fact;
  }
  for (int k = 0; k < 9; ++k) {
    const double s = 1.0 / f[2 * k + 1];
    const double c = 1.0 / f[2 * k];
    t.sin_c[k] = (k & 1) ? -s : s;
    t.cos_c[k] = (k & 1) ? -c : c;
  }
  constexpr double tn[9] = {1.0, 1.0, 2.0, 17.0, 62.0, 1382.0, 21844.0, 929569.0, 6404582.0};
  constexpr double td[9] = {1.0,         3.0,         15.0,          315.0,         2835.0,
                            155925.0,    6081075.0,   638512875.0,   10854718875.0};
  for (int k = 0; k < 9; ++k) t.tan_c[k] = tn[k] / td[k];
  return t;
}
constexpr TaylorCoeffs kTaylor = make_taylor();

// Constants of the fast path, compiled into constant bank 3 so every compare
// and multiply reads them as c[][] operands.  The two derived thresholds are
// the results of the host bisection in ft_capi.cu (compute_thresholds, run
// against IEEE division / subtraction); ft_thresholds() returns both and
// tests/test_capi_host.py asserts they are identical.
struct FastConsts {
  double quad[3];  // smallest r >= 0 with floor(RN(r/(pi/2))) >= 1, 2, 3
  double guard;    // smallest red in [0,pi/2] with |RN(red - pi/2)| < 1e-3
  double knot[5];  // segment knots k*pi/12, k = 1..5 (segments.hpp:60)
  double pi, two_pi, half_pi, inv_two_pi;
  double twelve_over_pi;  // RN(12/pi): row guess floor(red * 12/pi)
  double two52;           // 2^52: fma.rz(red, 12/pi, 2^52) puts floor() in the low word
  double half;            // 0.5 (FISR Newton step, as a c[][] operand)
  double inv_pi;          // RN(1/pi) = 2 * RN(1/2pi)
};
constexpr FastConsts make_fast_consts() {
  return FastConsts{{kHalfPi, kPi, 3.0 * kHalfPi},
                    0x1.91de2c0cf70aep+0,
                    {kTable.knots[1], kTable.knots[2], kTable.knots[3], kTable.knots[4], kTable.knots[5]},
                    kPi, kTwoPi, kHalfPi, kInvTwoPi, 12.0 / kPi, 0x1p52, 0.5, 2.0 * kInvTwoPi};
}
constexpr FastConsts kFast = make_fast_consts();

// Sqrt-mode selector as a template parameter of the kernels.
enum SqrtKind : int { kExact = 0, kFisr1 = 1, kFisrN = 2, kFisr2 = 3 };  // kFisrN: runtime step count

// Output mask bits (mirrors include/fasttrig_b200.h).
enum : unsigned { kSin = 1u, kCos = 2u, kTan = 4u };

#ifdef __CUDACC__

// Device copies of the constexpr tables (per translation unit; no relocatable
// device code needed).  Uniform-index reads only.
static __constant__ Table c_table = make_table();
static __constant__ TaylorCoeffs c_taylor = make_taylor();
static __constant__ FastConsts c_fast = make_fast_consts();

// Programmatic dependent launch (the launchers set
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel may be
// scheduled while the previous kernel on its stream drains; it stages its
// constant tables, then waits here for that kernel's completion (and memory
// flush) before touching global memory.  Without the attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// This block has no more launches to wait for: the next kernel may be scheduled
// once every block has called it (or exited).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ std::uint64_t d2u(double d) {
  return static_cast<std::uint64_t>(__double_as_longlong(d));
}
__device__ __forceinline__ double u2d(std::uint64_t u) {
  return __longlong_as_double(static_cast<long long>(u));
}
// Flip the sign bit when `neg` (== multiplication by -1.0, exact for all values).
__device__ __forceinline__ double flip_sign(double v, bool neg) {
  return u2d(d2u(v) ^ (static_cast<std::uint64_t>(neg) << 63));
}

// ======================================================================
// mirror_*: literal restatement of the reference (checker path)
// ======================================================================

// fisr.hpp:31-46
__device__ __forceinline__ double mirror_fast_inverse_sqrt(double v, int method, int steps) {
  if (!(v > 0.0) || v == __longlong_as_double(0x7ff0000000000000ll)) return u2d(kQuietNaN);
  if (method == 0) return __ddiv_rn(1.0, __dsqrt_rn(v));
  double y = u2d(kFisrMagic - (d2u(v) >> 1));
  const double half_v = __dmul_rn(0.5, v);
  for (int i = 0; i < steps; ++i) {
    y = __dmul_rn(y, __dsub_rn(1.5, __dmul_rn(__dmul_rn(half_v, y), y)));
  }
  return y;
}

// reduction.hpp:26-30
__device__ __forceinline__ double mirror_mod_positive(double a, double period) {
  double r = __dsub_rn(a, __dmul_rn(period, floor(__ddiv_rn(a, period))));
  r = r < 0.0 ? 0.0 : r;
  return r < period ? r : 0.0;
}

// reduction.hpp:32-35
__device__ __forceinline__ double mirror_clamp_red(double red) {
  red = red < 0.0 ? 0.0 : red;
  return red < kHalfPi ? red : kHalfPi;
}

struct Reduced {
  double red;
  bool neg;  // sign == -1.0
};

// reduction.hpp:44-52 + :59-79.  `cos` selects the cosine sign rule.
__device__ __forceinline__ Reduced mirror_reduce_sincos(double x, bool cos_sign) {
  if (!isfinite(x)) return {u2d(kQuietNaN), false};
  const double r = mirror_mod_positive(fabs(x), kTwoPi);
  double q = floor(__ddiv_rn(r, kHalfPi));
  q = q > 3.0 ? 3.0 : q;
  const double red = q == 0.0   ? r
                     : q == 1.0 ? __dsub_rn(kPi, r)
                     : q == 2.0 ? __dsub_rn(r, kPi)
                                : __dsub_rn(kTwoPi, r);
  if (cos_sign) return {mirror_clamp_red(red), !(q == 0.0 || q == 3.0)};
  return {mirror_clamp_red(red), (q >= 2.0) != static_cast<bool>(signbit(x))};
}

// reduction.hpp:83-93
__device__ __forceinline__ Reduced mirror_reduce_tan(double x) {
  if (!isfinite(x)) return {u2d(kQuietNaN), false};
  const double r = mirror_mod_positive(fabs(x), kPi);
  const bool upper = r > kHalfPi;
  const double red = mirror_clamp_red(upper ? __dsub_rn(kPi, r) : r);
  return {red, upper != static_cast<bool>(signbit(x))};
}

// segments.hpp:70-73
__device__ __forceinline__ int mirror_segment_index(const double* knots, double red) {
  return (red >= knots[1]) + (red >= knots[2]) + (red >= knots[3]) + (red >= knots[4]) +
         (red >= knots[5]);
}

// kernels.hpp:46-67 (which: 0 sin, 1 cos, 2 tan).  Returns the value; writes the
// segment choice (255 inside the tan guard window) to *seg.
__device__ __forceinline__ double mirror_proposed(const Table& T, int which, double x, int method,
                                                  int steps, int* seg) {
  if (which == 2) {
    const Reduced ra = mirror_reduce_tan(x);
    if (fabs(__dsub_rn(ra.red, kHalfPi)) < kTanPoleGuard) {
      *seg = 255;
      return flip_sign(__longlong_as_double(0x7ff0000000000000ll), ra.neg);
    }
    const int k = mirror_segment_index(T.knots, ra.red);
    *seg = k;
    const Coeffs& s = T.seg[k];
    const double poly = __dadd_rn(__dmul_rn(s.a, ra.red), s.b);
    const double den = __dadd_rn(__dmul_rn(s.c, ra.red), s.d);
    double v;
    if (method == 0) {
      v = __ddiv_rn(poly, den);
    } else {
      const double r = mirror_fast_inverse_sqrt(den, method, steps);
      v = __dmul_rn(poly, __dmul_rn(r, r));
    }
    return ra.neg ? __dmul_rn(-1.0, v) : __dmul_rn(1.0, v);
  }
  const Reduced ra = mirror_reduce_sincos(x, which == 1);
  const int k = mirror_segment_index(T.knots, ra.red);
  *seg = k;
  const Coeffs& s = T.seg[k];
  const double poly = which == 0 ? __dadd_rn(__dmul_rn(s.a, ra.red), s.b)
                                 : __dadd_rn(__dmul_rn(s.c, ra.red), s.d);
  const double rad = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(s.X, ra.red), s.Y), ra.red), s.Z);
  const double v = __dmul_rn(poly, mirror_fast_inverse_sqrt(rad, method, steps));
  return ra.neg ? __dmul_rn(-1.0, v) : __dmul_rn(1.0, v);
}

// SPEC.md:224-247 Taylor comparator, pinned order (see oracle/ft_oracle.c).
__device__ __forceinline__ double mirror_taylor(const TaylorCoeffs& C, int which, double x, int n) {
  const Reduced ra = which == 2 ? mirror_reduce_tan(x) : mirror_reduce_sincos(x, which == 1);
  const double* c = which == 0 ? C.sin_c : which == 1 ? C.cos_c : C.tan_c;
  const double s = __dmul_rn(ra.red, ra.red);
  double p = c[n - 1];
  for (int k = n - 2; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, s), c[k]);
  const double v = which == 1 ? p : __dmul_rn(ra.red, p);
  return ra.neg ? __dmul_rn(-1.0, v) : __dmul_rn(1.0, v);
}

// ======================================================================
// fast_*: production path (bitwise equal to mirror_* for every input)
// ======================================================================
//
// Instruction count (and, at the power cap, energy) per element is the design
// constraint, so:
//   * every constant lives in constant bank 3 (c_fast) and is read as a c[][]
//     instruction operand, never re-materialised into registers in the loop;
//   * compares are DSETP (one issue slot, exact) whose predicates feed SELs
//     directly -- no integer quadrant number is formed;
//   * the quadrant fold is one DADD of a selected base and a sign-selected r
//     (reference: {r, pi-r, r-pi, 2pi-r}); the reference's final clamp of red
//     to [0, pi/2] is provably a no-op once r is in [0, 2pi)
//     (tests/test_capi_host.py::test_fold_needs_no_clamp checks the edges);
//   * the reference's r clamps are not executed either: an r outside
//     [0, period) folds to red <= 0 or NaN, which fails the row bracket of
//     fast_proposed and sends the element to the exact path -- so non-finite
//     x needs no branch of its own.

// Per-segment coefficient row in shared memory: the coefficients plus the
// bracket of reduced angles the row is valid for, as the high words of its two
// ends: a lane accepts the row iff klo_hi < hi(red) < khi_hi (signed compare).
// That implies knot_lo < red < knot_hi for any red (negative and NaN red have
// a negative or > inf high word and never pass), and it is what lets the
// quadrant compares of fast_reduce use high words only (see there).
// 80-byte stride: the 16-byte chunks of the eight rows fall in disjoint banks
// (80k/4 mod 32 = 0,20,8,28,16,4,24,12), so a warp's LDS.128 never conflicts
// whichever rows its lanes pick.
struct alignas(16) SegRow {
  double a, b, c, d, X, Y, Z;
  int klo_hi, khi_hi;  // 16-byte chunk with Z
  double klo, khi;     // exact bracket [klo, khi) (tan-only kernels)
};
constexpr unsigned kRowBytes = sizeof(SegRow);
static_assert(kRowBytes == 80, "row stride");

// High words of the bounds the hi-word compares use (checked against the
// bisection thresholds in tests/test_capi_host.py::test_hiword_constants).
constexpr int kHiHalfPi = 0x3ff921fb;    // pi/2 = quad[0]
constexpr int kHiPiQ = 0x400921fb;       // pi = quad[1]
constexpr int kHiThreeHalfPi = 0x4012d97c;  // RN(3pi/2) = quad[2]
constexpr int kHiRow0Lo = 0x3ee00000;       // 2^-17: row 0 accepts hi(red) > this

// Rows 0..5 are segments 0..5 (segments.hpp:33-66); the row is chosen by the
// guess g = floor(red * 12/pi) (0..6 for red in [0, pi/2], 7 for NaN) and then
// validated against its bracket.  Row 0 accepts only hi(red) > hi(2^-17) (red
// >= 2^-17 + 2^-37: +0, tiny and negative red go to the exact path, which also
// covers the quadrant mis-folds of fast_reduce); row 5 stops below the high
// word of pi/2 (red < pi/2 - 3.1e-7); rows 6 and 7 accept nothing.  Lanes
// outside the brackets take the exact path (fast_proposed).  Tan-only kernels
// use exact compares and the double bracket [klo, khi) instead: row 0 from
// 2^-17, rows 5 and 6 up to +inf (red == pi/2 guesses 6),
// row 7 (NaN) empty.
struct SmemTable {
  SegRow row[8];
};

__device__ __forceinline__ void stage_table(SmemTable* s) {
  for (int i = threadIdx.x; i < 8; i += blockDim.x) {
    const int k = i < 6 ? i : 5;
    const Coeffs& c = c_table.seg[k];
    const int klo = i == 0 ? kHiRow0Lo : i >= 6 ? 0 : __double2hiint(c_table.knots[k]);
    const int khi = i == 5 ? kHiHalfPi : i >= 6 ? 0 : __double2hiint(c_table.knots[k + 1]);
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    const double dlo = i == 0 ? 0x1p-17 : i == 7 ? inf : c_table.knots[k];
    const double dhi = i >= 5 ? inf : c_table.knots[k + 1];
    s->row[i] = SegRow{c.a, c.b, c.c, c.d, c.X, c.Y, c.Z, klo, khi, dlo, dhi};
  }
}

__device__ __forceinline__ void lds_f64x2(unsigned addr, double& a, double& b) {
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(addr));
}
__device__ __forceinline__ int4 lds_i32x4(unsigned addr) {
  int4 v;
  asm("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ double xor_hi(double v, unsigned bits) {
  return __hiloint2double(__double2hiint(v) ^ static_cast<int>(bits), __double2loint(v));
}

// v^(-1/2) for the evaluation domain (radicand in [1.98e5, 8.9e5]; tan
// denominator > 0.63 outside the pole window -- the only lanes whose tan value
// is kept).  fisr.hpp:31-46 without the NaN guard, which cannot fire there.
// The Newton step y*(1.5 - (0.5v*y)*y) is evaluated as y*fma(-0.5, (v*y)*y, 1.5):
// 0.5v is exact, so RN(0.5v*y) = RN(v*y)/2 and RN(RN(0.5v*y)*y) = RN(RN(v*y)*y)/2
// (no subnormals here), and the FMA of the exact product -0.5t with 1.5 rounds
// once, as the reference's subtraction does -- same bits, no 0.5v to form.
// magic - (bits >> 1) == (2*magic + 1 - bits) >> 1 for bits <= 2*magic + 1 (all
// positive doubles): with bits = 2k + e, floor((2m + 1 - 2k - e) / 2) = m - k.
// One 64-bit subtract then one 64-bit shift (4 integer instructions, vs 5 for
// shift-then-subtract, whose subtrahend needs a complement).
constexpr std::uint64_t kFisrMagic2p1 = 2 * kFisrMagic + 1;
__device__ __forceinline__ double fisr_seed(double v) {
  return u2d((kFisrMagic2p1 - d2u(v)) >> 1);
}
__device__ __forceinline__ double fisr_newton(double v, double y) {
  return __dmul_rn(y, __fma_rn(-c_fast.half, __dmul_rn(__dmul_rn(v, y), y), 1.5));
}

template <int SQ>
__device__ __forceinline__ double fast_rsqrt(double v, int steps) {
  if constexpr (SQ == kExact) {
    return __ddiv_rn(1.0, __dsqrt_rn(v));
  } else {
    double y = fisr_seed(v);
    if constexpr (SQ == kFisr1 || SQ == kFisr2) {
      y = fisr_newton(v, y);
      if constexpr (SQ == kFisr2) y = fisr_newton(v, y);
    } else {
      for (int i = 0; i < steps; ++i) y = fisr_newton(v, y);
    }
    return y;
  }
}

struct FastRed {
  // sin/cos and tan reduced angles (reduction.hpp:59-79, 83-93) up to sign:
  // the fused proposed path leaves the fold's sign in them, so every consumer
  // reads fabs(red) / fabs(redt) (free as FP64 operand modifiers)
  double red;
  double redt;
  unsigned neg_s;  // sign-bit masks (0 or 0x80000000) to XOR into the results
  unsigned neg_c;
  unsigned neg_t;
  bool guard;      // tan pole window (kernels.hpp:62)
  bool valid;      // proposed path: r within [0, 2pi]'s high words (see fast_reduce)
};

constexpr unsigned kHiPi = 0x400921fbu, kHiTwoPi = 0x401921fbu, kHiMinusPi = 0xc00921fbu;
constexpr unsigned kLoPi = 0x54442d18u;  // pi, -pi, 2pi share the low word

// CLAMP: apply the reference's r clamps (NaN-preserving form).  The proposed
// path runs without them and validates instead (fast_proposed).
template <bool NEED_SC, bool NEED_T, bool CLAMP, bool HIW_T = !CLAMP>
__device__ __forceinline__ FastRed fast_reduce(double x) {
  const FastConsts& K = c_fast;
  FastRed o{};
  o.valid = true;
  const double a = fabs(x);
  // q1 = RN(a / 2pi) exactly: y = RN(1/2pi) is within 0.206*2^-53 relative, so
  // q0 = RN(a*y) is within 0.912 ulp of a/2pi and one Markstein correction
  // (exact FMA remainder) rounds to RN(a/2pi).
  // Tan-only proposed kernels need only RN(a/pi)'s stand-in 2*q0, which is
  // RN(a * RN(1/pi)) exactly (RN(1/pi) = 2 RN(1/2pi)): one DMUL, no doubling.
  constexpr bool kTanOnly = !NEED_SC && !CLAMP;
  const double q0 = kTanOnly ? __dmul_rn(a, K.inv_pi) : __dmul_rn(a, K.inv_two_pi);
  double q1 = q0;
  if constexpr (CLAMP) {
    const double rem = __fma_rn(-q0, K.two_pi, a);
    q1 = __fma_rn(rem, K.inv_two_pi, q0);
  } else {
    // Proposed path: no correction.  q0 differs from RN(a/2pi) by at most one
    // ulp, so floor(q0) differs from the reference's floor only when an
    // integer k lies between them, i.e. a is within ~a*2^-52 of 2pi*k (or pi*k
    // for tan).  The r that follows is then off by one period: r <= 0 (+0
    // when a == RN(2pi*k)), or r within that distance of 2pi (pi), whose fold
    // is <= 0 or smaller than 2^-22 for |x| < 2^30 -- no row bracket accepts
    // either, so those elements take the exact path
    // (tests/test_capi_host.py::test_markstein_free_floor_is_caught).
    // `valid` sends |x| >= 2^24 * 2pi (q0 >= 2^24; NaN, inf) to the exact path:
    // the argument above needs |x| < 2^30, the fused kernel's shared row
    // (fast_proposed_core) |x| < 2^27.
    o.valid = __double2hiint(q0) < (kTanOnly ? 0x41800000 : 0x41700000);  // (2)q0 < 2^24 (2^25)
  }
  const unsigned xs = static_cast<unsigned>(__double2hiint(x)) & 0x80000000u;
  double k = 0.0;       // floor(q1)
  bool upper = false;   // proposed path: r >= pi by the high-word compare
  if constexpr (NEED_SC) {
    // reduction.hpp:26-30 (period 2pi) without its two clamps on the proposed
    // path: r < 0 or r >= 2pi is caught by `valid` / the row brackets and
    // takes the exact path (fast_proposed).
    k = floor(q1);
    double r = __dsub_rn(a, __dmul_rn(K.two_pi, k));
    if constexpr (CLAMP) r = (r < 0.0 || r >= K.two_pi) ? 0.0 : r;
    // reduction.hpp:44-52: q = floor(RN(r/(pi/2))) = p1 + p2 + p3
    bool p1, p2, p3;
    if constexpr (CLAMP) {
      p1 = r >= K.quad[0], p2 = r >= K.quad[1], p3 = r >= K.quad[2];
      const bool odd = p1 ^ p2 ^ p3;
      const unsigned bhi = p3 ? kHiTwoPi : (p2 ? kHiMinusPi : (p1 ? kHiPi : 0u));
      const unsigned blo = p1 ? kLoPi : 0u;
      o.red = __dadd_rn(__hiloint2double(static_cast<int>(bhi), static_cast<int>(blo)),
                        xor_hi(r, odd ? 0x80000000u : 0u));
    } else {
      // High words only, on the integer pipe: exact unless hi(r) equals a
      // threshold's high word; such an r may be given the lower quadrant.
      const int rh = __double2hiint(r);
      p1 = rh > kHiHalfPi, p2 = rh > kHiPiQ, p3 = rh > kHiThreeHalfPi;
      // Fold as red = |RN(r - c)|, c = 0, pi, pi, 2pi for q = 0..3: RN is odd,
      // so RN(pi - r) = -RN(r - pi) and RN(2pi - r) = -RN(r - 2pi).  A wrong
      // quadrant from the high-word compares puts red within 2^-19 of 0
      // (r ~ pi: same |red|, wrong sine sign) or at/above pi/2 (r ~ pi/2,
      // 3pi/2).  For |x| < 2^27 (`valid`) an r outside [0, 2pi) -- the
      // reference's clamps, or a floor off by one (above) -- is within
      // 2^-24 of 0 or 2pi (2pi's high word spans 2pi + 2.4e-6), so it folds
      // to red < 2^-17 too; NaN keeps a NaN high word.  No row bracket accepts
      // red < 2^-17 or hi(red) >= hi(pi/2) (SmemTable), so all of these take
      // the exact path.
      const unsigned chi = p3 ? kHiTwoPi : (p1 ? kHiPi : 0u);
      const unsigned clo = p1 ? kLoPi : 0u;
      const double d = __dsub_rn(r, __hiloint2double(static_cast<int>(chi), static_cast<int>(clo)));
      o.red = d;  // signed: consumers take |red| (operand modifier / integer mask)
      // cos sign: q in {1, 2} == (q >= 2) xor (q odd), and q is odd exactly
      // when r - c < 0 (q = 1, 3), so it is the sign bit of d xor p2.
      o.neg_c = (static_cast<unsigned>(__double2hiint(d)) & 0x80000000u) ^ (p2 ? 0x80000000u : 0u);
      upper = p2;
    }
    o.neg_s = (p2 ? 0x80000000u : 0u) ^ xs;  // q >= 2, odd symmetry (reduction.hpp:65-66)
    if constexpr (CLAMP) o.neg_c = (p1 != p3) ? 0x80000000u : 0u;  // q in {1, 2} (reduction.hpp:77)
  }
  if constexpr (NEED_T) {
    // RN(a/pi) == 2*RN(a/2pi) exactly (2pi is an exact doubling of pi).  The
    // clamped path doubles the corrected q1; the tan-only proposed path floors
    // q0 = RN(a*RN(1/pi)) = 2*RN(a*RN(1/2pi)) (an off-by-one floor is rejected
    // by the bracket, as for the sine).  Non-finite x fails `valid`.
    double r;
    if constexpr (NEED_SC && !CLAMP) {
      // Fused proposed path: floor(RN(a/pi)) = 2k + [r >= pi] for the sine's
      // k and r, and RN(pi * (2k + s)) = fma(k, 2pi, s ? pi : 0) (2pi = 2 * pi
      // exactly, so the FMA rounds the same real number once).  When the
      // high-word `upper` is wrong (r within 2^-19 of pi) or k is off by one,
      // the tangent's r is off by one period and folds to red_t <= 0 or below
      // 2^-17 -- rejected like the sine's (see above).
      const double s_pi = __hiloint2double(upper ? static_cast<int>(kHiPi) : 0, upper ? static_cast<int>(kLoPi) : 0);
      r = __dsub_rn(a, __fma_rn(k, K.two_pi, s_pi));
    } else {
      const double q2 = CLAMP ? __dadd_rn(q1, q1) : q0;  // tan-only: q0 = RN(a * RN(1/pi))
      r = __dsub_rn(a, __dmul_rn(K.pi, floor(q2)));
    }
    if constexpr (CLAMP) r = (r < 0.0 || r >= K.pi) ? 0.0 : r;
    // reduction.hpp:88-89 (r > pi/2).  Proposed path: high word only; an r
    // with the high word of pi/2 keeps red = r, whose high word no row accepts.
    const bool up = HIW_T ? __double2hiint(r) > kHiHalfPi : r > K.half_pi;
    const double base = __hiloint2double(up ? static_cast<int>(kHiPi) : 0, up ? static_cast<int>(kLoPi) : 0);
    if constexpr (!CLAMP) {
      // Proposed path: red_t = |RN(r - base)| (RN(pi - r) = -RN(r - pi)); the sign of
      // r - base is `up` for every r the sine's checks accept, so it is the
      // tangent's sign before the odd symmetry.  Fused kernels: the cases
      // where r is off by a period or mis-folded coincide with a sine red the
      // row brackets reject (r within 2^-19 of a multiple of pi / pi/2).
      // Tan-only (exact `up`): r outside [0, pi) is within 2^-24 of 0 or pi
      // for |x| < 2^25 pi and folds below row 0's bound 2^-17.
      const double d = __dsub_rn(r, base);
      o.redt = d;  // signed, as red
      o.neg_t = (static_cast<unsigned>(__double2hiint(d)) & 0x80000000u) ^ xs;
    } else {
      o.redt = __dadd_rn(base, xor_hi(r, up ? 0x80000000u : 0u));
      o.neg_t = (up ? 0x80000000u : 0u) ^ xs;
    }
    o.guard = fabs(o.redt) >= K.guard;
  }
  return o;
}

struct Out3 {
  double s, c, t;
  int seg_sc, seg_t;
};

// The exact path of fast_proposed: all three functions and both segment
// choices by the device restatement.  Out of line so the rarely-taken branch
// costs the hot loop neither instructions nor registers.
static __device__ __noinline__ Out3 slow_proposed(double x, int method, int steps) {
  Out3 o;
  o.s = mirror_proposed(c_table, 0, x, method, steps, &o.seg_sc);
  o.c = mirror_proposed(c_table, 1, x, method, steps, &o.seg_sc);
  o.t = mirror_proposed(c_table, 2, x, method, steps, &o.seg_t);
  return o;
}

// Fused proposed sin/cos/tan of one element (kernels.hpp:46-67).  SEG: also
// produce both segment choices even for functions not in MASK.
//
// Row choice: g = floor(red * 12/pi) from one fma.rz, validated by
// klo_hi < hi(red) < khi_hi (and the same for the tan angle, which differs from
// the sin/cos one by a few ulps at most, so it shares the row).  A lane fails the
// check only near a knot, at red == +0, within ~2e-6 of a quadrant boundary,
// for the r < 0 / r >= period cases the reference clamps, or for non-finite x -- it then recomputes the element with
// the exact device restatement (mirror_*), so every lane returns the
// reference's bits.
template <int SQ, unsigned MASK, bool SEG = false>
__device__ __forceinline__ Out3 fast_proposed_core(double x, const SmemTable& tb, int steps, bool* okp) {
  constexpr bool kSC = (MASK & (kSin | kCos)) != 0 || SEG;
  constexpr bool kT = (MASK & kTan) != 0 || SEG;
  const FastConsts& K = c_fast;
  // Tan-only kernels fold with the exact DSETP and validate with the exact
  // bracket [klo, khi): measured faster there (444 vs 414 Gelem/s, cfg3) --
  // the high-word bracket's extra LDS sits on that short kernel's critical path.
  constexpr bool kDbl = !kSC;
  const FastRed fr = fast_reduce<kSC, kT, false, !kDbl>(x);
  const double key = fabs(kSC ? fr.red : fr.redt);
  const unsigned g = static_cast<unsigned>(__double2loint(__fma_rz(key, K.twelve_over_pi, K.two52))) & 7u;
  // Row loads as ld.shared from the table's 32-bit shared address (a generic
  // pointer costs the loop a CTA-window base re-materialisation per element).
  const unsigned ra = static_cast<unsigned>(__cvta_generic_to_shared(&tb)) + g * kRowBytes;
  SegRow s;
  lds_f64x2(ra + offsetof(SegRow, a), s.a, s.b);
  lds_f64x2(ra + offsetof(SegRow, c), s.c, s.d);
  lds_f64x2(ra + offsetof(SegRow, X), s.X, s.Y);
  lds_f64x2(ra + offsetof(SegRow, klo), s.klo, s.khi);
  // Z and the high-word bracket share one 16-byte chunk: one LDS.128
  const int4 zq = lds_i32x4(ra + offsetof(SegRow, Z));
  const double sZ = __hiloint2double(zq.y, zq.x);
  bool ok = true;
  if constexpr (kSC) {
    const int h = __double2hiint(fr.red) & 0x7fffffff;
    ok = fr.valid & (h > zq.z) & (h < zq.w);
  }
  if constexpr (kT && kDbl) {
    ok = fr.valid & (fabs(fr.redt) >= s.klo) & (fabs(fr.redt) < s.khi);
  }
  // Fused kernels: the tangent shares the sine's row without a check of its
  // own.  red and red_t both round the distance from |x| to the nearest
  // multiple of pi, |red - red_t| <= 2^-52 |x| + 2^-49 < 3e-8 for |x| < 2^27
  // (`valid`), while every accepted high-word bracket lies >= 5.2e-8 inside
  // its knots (pi/12's low word 0x382d7365 ulps of 2^-54 is the closest) --
  // so red_t is in the same segment.  tests/test_capi_host.py::test_shared_row_margin.
  Out3 o{0.0, 0.0, 0.0, 0, 0};
  if constexpr (kSC) {
    const double red = fabs(fr.red);
    const double rad = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(s.X, red), s.Y), red), sZ);
    const double rs = fast_rsqrt<SQ>(rad, steps);
    if constexpr ((MASK & kSin) != 0)
      o.s = xor_hi(__dmul_rn(__dadd_rn(__dmul_rn(s.a, red), s.b), rs), fr.neg_s);
    if constexpr ((MASK & kCos) != 0)
      o.c = xor_hi(__dmul_rn(__dadd_rn(__dmul_rn(s.c, red), s.d), rs), fr.neg_c);
  }
  if constexpr (kT) {
    const double red = fabs(fr.redt);
    const double poly = __dadd_rn(__dmul_rn(s.a, red), s.b);
    const double den = __dadd_rn(__dmul_rn(s.c, red), s.d);
    double v;
    if constexpr (SQ == kExact) {
      v = __ddiv_rn(poly, den);
    } else {
      const double r = fast_rsqrt<SQ>(den, steps);
      v = __dmul_rn(poly, __dmul_rn(r, r));
    }
    v = fr.guard ? __longlong_as_double(0x7ff0000000000000ll) : v;
    o.t = xor_hi(v, fr.neg_t);
  }
  if constexpr (SEG) {  // an accepted row is segment g (rows 0..5)
    o.seg_sc = static_cast<int>(g);
    o.seg_t = fr.guard ? 255 : static_cast<int>(g);
  }
  *okp = ok;
  return o;
}

template <int SQ>
__device__ __forceinline__ Out3 slow_proposed_mode(double x, int steps) {
  return slow_proposed(x, SQ == kExact ? 0 : 1, SQ == kFisr1 ? 1 : SQ == kFisr2 ? 2 : steps);
}

template <int SQ, unsigned MASK, bool SEG = false>
__device__ __forceinline__ Out3 fast_proposed(double x, const SmemTable& tb, int steps) {
  bool ok;
  Out3 o = fast_proposed_core<SQ, MASK, SEG>(x, tb, steps, &ok);
  if (!ok) o = slow_proposed_mode<SQ>(x, steps);  // rare
  return o;
}

// Horner on s = red^2 over the first n coefficients, highest first.
// NT > 0: n == NT known at compile time (unrolled); NT == 0: runtime n.
template <int NT>
__device__ __forceinline__ double taylor_horner(const double* c, int n, double s2) {
  if constexpr (NT > 0) {
    double p = c[NT - 1];
#pragma unroll
    for (int k = NT - 2; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, s2), c[k]);
    return p;
  } else {
    double p = c[n - 1];
    for (int k = n - 2; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, s2), c[k]);
    return p;
  }
}

// Exact path of fast_taylor: the device restatement of each requested function.
template <unsigned MASK>
static __device__ __noinline__ Out3 slow_taylor(double x, int n) {
  Out3 o{0.0, 0.0, 0.0, 0, 0};
  if constexpr ((MASK & kSin) != 0) o.s = mirror_taylor(c_taylor, 0, x, n);
  if constexpr ((MASK & kCos) != 0) o.c = mirror_taylor(c_taylor, 1, x, n);
  if constexpr ((MASK & kTan) != 0) o.t = mirror_taylor(c_taylor, 2, x, n);
  return o;
}

// Fused Taylor sin/cos/tan of one element, n nonzero terms.
// With sin or cos in MASK: the proposed path's reduction (fast_reduce, no
// clamps, no Markstein step, high-word quadrant, signed folds) certified by
// red's high word -- every case where it can differ from the reference
// (off-by-one floor, quadrant mis-fold, r outside [0, 2pi), |x| >= 2^24 * 2pi,
// non-finite x) has red < 2^-17 or hi(red) >= hi(pi/2) (see fast_reduce), and
// is redone exactly; the tangent shares k and its failure cases (as in
// fast_proposed_core).  CERT = false, or tan only: the clamped exact reduction
// (f64 kernels are memory-bound and measured faster without the exact-path
// branch: 256 vs 246 Gelem/s, cfg4 f64; f32 gains 381 -> 419).
template <int NT, unsigned MASK, bool CERT = true>
__device__ __forceinline__ Out3 fast_taylor(double x, int n) {
  constexpr bool kSC = (MASK & (kSin | kCos)) != 0;
  constexpr bool kT = (MASK & kTan) != 0;
  Out3 o{0.0, 0.0, 0.0, 0, 0};
  if constexpr (kSC && !CERT) {
    const FastRed fr = fast_reduce<true, kT, true>(x);
    const double s2 = __dmul_rn(fr.red, fr.red);
    if constexpr ((MASK & kSin) != 0)
      o.s = xor_hi(__dmul_rn(fr.red, taylor_horner<NT>(c_taylor.sin_c, n, s2)), fr.neg_s);
    if constexpr ((MASK & kCos) != 0)
      o.c = xor_hi(taylor_horner<NT>(c_taylor.cos_c, n, s2), fr.neg_c);
    if constexpr (kT) {
      const double s2t = __dmul_rn(fr.redt, fr.redt);
      o.t = xor_hi(__dmul_rn(fr.redt, taylor_horner<NT>(c_taylor.tan_c, n, s2t)), fr.neg_t);
    }
  } else if constexpr (kSC) {
    const FastRed fr = fast_reduce<true, kT, false, true>(x);
    const int h = __double2hiint(fr.red) & 0x7fffffff;
    const bool ok = fr.valid & (h > kHiRow0Lo) & (h < kHiHalfPi);
    const double red = fabs(fr.red);
    const double s2 = __dmul_rn(red, red);
    if constexpr ((MASK & kSin) != 0)
      o.s = xor_hi(__dmul_rn(red, taylor_horner<NT>(c_taylor.sin_c, n, s2)), fr.neg_s);
    if constexpr ((MASK & kCos) != 0)
      o.c = xor_hi(taylor_horner<NT>(c_taylor.cos_c, n, s2), fr.neg_c);
    if constexpr (kT) {
      const double redt = fabs(fr.redt);
      const double s2t = __dmul_rn(redt, redt);
      o.t = xor_hi(__dmul_rn(redt, taylor_horner<NT>(c_taylor.tan_c, n, s2t)), fr.neg_t);
    }
    if (!ok) o = slow_taylor<MASK>(x, n);  // rare
  } else {
    const FastRed fr = fast_reduce<false, true, true>(x);
    const double s2 = __dmul_rn(fr.redt, fr.redt);
    o.t = xor_hi(__dmul_rn(fr.redt, taylor_horner<NT>(c_taylor.tan_c, n, s2)), fr.neg_t);
  }
  return o;
}

// ======================================================================
// relaxed_*: f32 inputs at the north-star tolerance (<= 2 ulp of the
// float-rounded reference, identical segment choice)
// ======================================================================
//
// The reference result for an f32 element is (float)proposed((double)x), so the
// binary64 value is only needed to ~2^-26 relative: any evaluation within that
// of the reference's own binary64 result rounds to the same float or to a
// neighbour (<= 1 ulp).  That frees the reduction and the evaluation:
//
//   * one signed reduction for all three functions: m = rint(|x|/pi) from one
//     FMA with 1.5*2^52 (m in the low word), d = RN(|x| - pi*m) by one FMA.
//     |d| is the distance from |x| to the nearest multiple of pi, which is
//     what reduce_sin / reduce_cos / reduce_tan all compute (the quadrant fold
//     of reduction.hpp:44-52 and the tangent's r > pi/2 fold of :88-89 both
//     pick the nearest multiple of pi), so red = red_t = |d| and the signs are
//     bits: sin (d<0) ^ (m odd) ^ (x<0), cos (m odd), tan (d<0) ^ (x<0).  The
//     tan-only kernels reduce the signed x instead (relaxed_x<true>): m and d
//     are then the exact negatives, and the tangent's sign is d's alone.
//     The reference's red differs from |d| only by the rounding of RN(2pi*k)
//     (resp. RN(pi*k)) -- its other subtractions are exact (Sterbenz) -- so
//     |red_ref - |d|| <= 2^-38 for |x| < 2^16 (2^-37.9 with d's own rounding);
//   * the evaluation from the four linear coefficients only: Ns = a*red + b
//     and Nc = c*red + d (one FMA each) are the sine and cosine numerators,
//     the radicand is Ns^2 + Nc^2 (= X red^2 + Y red + Z identically: X, Y, Z
//     are a^2+c^2, 2(ab+cd), b^2+d^2, segments.hpp:44-50), and with red_t = red
//     the tangent's numerator and denominator are Ns and Nc as well
//     (kernels.hpp:33-41).  Relative to the reference's rounded X, Y, Z and
//     Horner steps this moves the radicand by ~2^-50 relative; the FISR seed is
//     a continuous function of it, so the output moves by the same order.
//     Rows shrink from 80 to 48 bytes (3 shared-memory loads, 10 wavefronts
//     per warp instead of 16 -- cfg1 was L1-throughput bound at 84%) and the
//     tangent needs no FMAs of its own.
//
// Certification (else the lane takes the bit-exact path, relaxed_slow):
//   * |x| < 2^16;
//   * the segment row's high-word bracket (as fast_proposed_core): every
//     accepted bracket lies >= 5.2e-8 inside its knots, >> 2^-37.9, so the
//     reference's red is in the same segment;
//   * the output's relative sensitivity to red is 1/red for sin and tan near
//     0 (segment 0: b = 0), 1/(pi/2 - red) for cos near pi/2 (c*pi/2 + d = 0
//     for segment 5), <= ~1000 for tan up to the pole guard and O(1)
//     elsewhere, so red >= 2^-11 (masks with sin or tan) and red <= pi/2 -
//     2^-11 (masks with cos) keep it below 2^-37.9 * 2^11 = 2^-26.9;
//   * the tangent's guard decision |red_t - pi/2| < 1e-3 and its sign are
//     certain when hi(red) != hi(guard) (the guard sits >= 2.3e-7 inside its
//     high-word bucket) and hi(red) < hi(pi/2) (row 5's bracket; m's parity
//     can flip only within ~2^-38 of pi/2).
// Segment choice is g, the certified row.  tests/test_f32_exhaustive_gpu.py
// checks all 2^32 float inputs against the bit-exact kernels and the
// reference library (<= 1 ulp observed, segments identical).
constexpr float kRelaxMaxAbs = 65536.0f;  // 2^16
constexpr int kHiRelaxLo = 0x3f400000;    // hi(2^-11)
constexpr int kHiRelaxCos = 0x3ff91ffb;   // hi(pi/2 - 2^-11)
constexpr int kHiGuard = 0x3ff91de2;      // hi(kFast.guard)
constexpr double kRintMagic = 0x1.8p52;   // 1.5 * 2^52: RN(v + magic) - magic = rint(v), |v| < 2^51

// Relaxed rows: the linear coefficients and the high-word bracket narrowed by
// the sensitivity bounds above for the functions MASK evaluates.  48-byte
// stride: a warp's LDS.128 (8 lanes per phase) and LDS.64 (16 lanes) of any
// row mix fall in disjoint banks (row k starts at word 12k: 0,12,24,4,16,28,8,20).
struct alignas(16) RelaxRow {
  double a, b, c, d;
  int klo_hi, khi_hi;  // accept iff klo_hi < hi(red) < khi_hi
  int pad[2];
};
static_assert(sizeof(RelaxRow) == 48, "relaxed row stride");
struct RelaxTable {
  RelaxRow row[8];
};

template <unsigned MASK, bool SEG>
__device__ __forceinline__ void stage_table_relaxed(RelaxTable* s) {
  constexpr bool kLo = (MASK & (kSin | kTan)) != 0 || SEG;
  constexpr bool kHi = (MASK & kCos) != 0;
  for (int i = threadIdx.x; i < 8; i += blockDim.x) {
    const int k = i < 6 ? i : 5;
    const Coeffs& c = c_table.seg[k];
    const int klo = i >= 6 ? 0x7fffffff : i == 0 ? (kLo ? kHiRelaxLo : -1) : __double2hiint(c_table.knots[k]);
    const int khi = i >= 6 ? 0 : i == 5 ? (kHi ? kHiRelaxCos : kHiHalfPi) : __double2hiint(c_table.knots[k + 1]);
    s->row[i] = RelaxRow{c.a, c.b, c.c, c.d, klo, khi, {0, 0}};
  }
}

__device__ __forceinline__ int2 lds_i32x2(unsigned addr) {
  int2 v;
  asm("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

struct Out3f {
  float s, c, t;
  int seg_sc, seg_t;
};

__device__ __forceinline__ float xor_f(float v, unsigned bits) { return __uint_as_float(__float_as_uint(v) ^ bits); }

// The reduction's argument and the sign word of the folded angle.  SIGNED
// reduces the signed x: m = rint(x/pi) and d = x - m pi are the exact negatives
// of the |x| reduction's (RN is odd-symmetric, and x/pi never falls on a
// rounding tie for |x| < 2^52), so red = |d| is unchanged and the sign of x is
// already in d.  Used by the tan-only kernels (one LOP3 fewer per element);
// the fused kernels reduce |x| (the abs is a free F2F modifier, and their sine
// sign then needs one LOP3 fewer; r02bc, r02bk).  (F2F on the XU pipe; an
// integer re-bias measured slower, r02l.)
template <bool SIGNED>
__device__ __forceinline__ double relaxed_x(float xf) {
  if constexpr (SIGNED) return static_cast<double>(xf);
  else return fabs(static_cast<double>(xf));
}
// Bit 31: (d < 0) ^ (x < 0) of the |x| reduction.
template <bool SIGNED>
__device__ __forceinline__ unsigned relaxed_dx(double d, float xf) {
  if constexpr (SIGNED) return static_cast<unsigned>(__double2hiint(d));
  else return static_cast<unsigned>(__double2hiint(d)) ^ __float_as_uint(xf);
}
// v to float with `sign` (bit 31) applied (a truncating funnel-shift
// conversion measured slower, r02l).
__device__ __forceinline__ float relaxed_to_float(double v, unsigned sign) {
  return xor_f(__double2float_rn(v), sign);
}

template <int SQ, unsigned MASK, bool SEG>
__device__ __forceinline__ Out3f relaxed_proposed_core(float xf, const RelaxTable& tb, int steps, bool* okp) {
  constexpr bool kS = (MASK & kSin) != 0, kC = (MASK & kCos) != 0, kT = (MASK & kTan) != 0;
  const FastConsts& K = c_fast;
  const double a = relaxed_x<MASK == kTan>(xf);
  const double t = __fma_rn(a, K.inv_pi, kRintMagic);
  const double d = __fma_rn(-K.pi, __dadd_rn(t, -kRintMagic), a);
  const double red = fabs(d);
  const unsigned g = static_cast<unsigned>(__double2loint(__fma_rz(red, K.twelve_over_pi, K.two52))) & 7u;
  const unsigned ra = static_cast<unsigned>(__cvta_generic_to_shared(&tb)) + g * sizeof(RelaxRow);
  const int2 br = lds_i32x2(ra + offsetof(RelaxRow, klo_hi));
  const int h = __double2hiint(d) & 0x7fffffff;
  bool ok = (fabsf(xf) < kRelaxMaxAbs) & (h > br.x) & (h < br.y);
  if constexpr (kT || SEG) ok = ok & (h != kHiGuard);
  const unsigned modd = static_cast<unsigned>(__double2loint(t)) << 31;  // m odd
  const unsigned dx = relaxed_dx<MASK == kTan>(d, xf);
  double ca, cb, cc, cd;
  lds_f64x2(ra + offsetof(RelaxRow, a), ca, cb);
  lds_f64x2(ra + offsetof(RelaxRow, c), cc, cd);
  const double ns = __fma_rn(ca, red, cb);  // sine numerator == tangent numerator
  const double nc = __fma_rn(cc, red, cd);  // cosine numerator == tangent denominator
  Out3f o{0.0f, 0.0f, 0.0f, 0, 0};
  const unsigned sd = dx & 0x80000000u;  // sign of the folded angle: sin, tan and the guard's infinity
  if constexpr (kS || kC) {
    const double rad = __fma_rn(ns, ns, __dmul_rn(nc, nc));
    const double rs = fast_rsqrt<SQ>(rad, steps);
    if constexpr (kS) o.s = xor_f(xor_f(__double2float_rn(__dmul_rn(ns, rs)), modd), sd);  // one 3-input LOP3
    if constexpr (kC) o.c = relaxed_to_float(__dmul_rn(nc, rs), modd);
  }
  const bool guard = h > kHiGuard;
  if constexpr (kT) {
    double v;
    if constexpr (SQ == kExact) {
      v = __ddiv_rn(ns, nc);
    } else if constexpr (SQ == kFisr1) {
      // ns * (y0 h)^2 with h = 1.5 - 0.5 nc y0^2 (one Newton step), as
      // (ns y0^2) h h: the same six FP64 operations, one dependent step fewer.
      const double y0 = fisr_seed(nc);
      const double p = __dmul_rn(y0, y0);
      const double h = __fma_rn(-c_fast.half, __dmul_rn(nc, p), 1.5);
      v = __dmul_rn(__dmul_rn(__dmul_rn(ns, p), h), h);
    } else {
      const double r = fast_rsqrt<SQ>(nc, steps);
      v = __dmul_rn(__dmul_rn(ns, r), r);
    }
    const float vf = relaxed_to_float(v, sd);
    o.t = guard ? __uint_as_float(0x7f800000u | sd) : vf;
  }
  if constexpr (SEG) {
    o.seg_sc = static_cast<int>(g);
    o.seg_t = guard ? 255 : static_cast<int>(g);
  }
  *okp = ok;
  return o;
}

// The relaxed kernels' exact path: the bit-exact fused evaluation (its own
// rows `tbx`, its own mirror fallback), rounded to float.  Out of line.
template <int SQ, unsigned MASK, bool SEG>
static __device__ __noinline__ Out3f relaxed_slow(float xf, const SmemTable* tbx, int steps) {
  const Out3 o = fast_proposed<SQ, MASK, SEG>(static_cast<double>(xf), *tbx, steps);
  return Out3f{__double2float_rn(o.s), __double2float_rn(o.c), __double2float_rn(o.t), o.seg_sc, o.seg_t};
}

// Relaxed Taylor sin/cos/tan (NT = 5, 7 or 9 terms): the relaxed reduction and
// Horner contracted to FMAs.  Brackets: red >= 2^-11 for sin and tan (zero at
// 0), red <= pi/2 - 2^-11 for cos (the truncated cosine's zero lies within
// 2.5e-5 of pi/2 for these NT: Taylor-5 cos(pi/2) = -2.47e-5).
template <int NT, unsigned MASK>
__device__ __forceinline__ Out3f relaxed_taylor_core(float xf, bool* okp) {
  constexpr bool kS = (MASK & kSin) != 0, kC = (MASK & kCos) != 0, kT = (MASK & kTan) != 0;
  const FastConsts& K = c_fast;
  const double a = relaxed_x<MASK == kTan>(xf);
  const double t = __fma_rn(a, K.inv_pi, kRintMagic);
  const double d = __fma_rn(-K.pi, __dadd_rn(t, -kRintMagic), a);
  const double red = fabs(d);
  const int h = __double2hiint(d) & 0x7fffffff;
  bool ok = fabsf(xf) < kRelaxMaxAbs;
  if constexpr (kS || kT) ok = ok & (h > kHiRelaxLo);
  ok = ok & (h < (kC ? kHiRelaxCos : kHiHalfPi));
  const unsigned modd = static_cast<unsigned>(__double2loint(t)) << 31;
  const unsigned dx = relaxed_dx<MASK == kTan>(d, xf);
  const double s2 = __dmul_rn(red, red);
  auto horner = [&](const double* c) {
    double p = c[NT - 1];
#pragma unroll
    for (int k = NT - 2; k >= 0; --k) p = __fma_rn(p, s2, c[k]);
    return p;
  };
  Out3f o{0.0f, 0.0f, 0.0f, 0, 0};
  if constexpr (kS) o.s = xor_f(__double2float_rn(__dmul_rn(red, horner(c_taylor.sin_c))), (dx ^ modd) & 0x80000000u);
  if constexpr (kC) o.c = xor_f(__double2float_rn(horner(c_taylor.cos_c)), modd);
  if constexpr (kT) o.t = xor_f(__double2float_rn(__dmul_rn(red, horner(c_taylor.tan_c))), dx & 0x80000000u);
  *okp = ok;
  return o;
}

template <int NT, unsigned MASK>
static __device__ __noinline__ Out3f relaxed_taylor_slow(float xf) {
  const Out3 o = fast_taylor<NT, MASK, true>(static_cast<double>(xf), NT);
  return Out3f{__double2float_rn(o.s), __double2float_rn(o.c), __double2float_rn(o.t), 0, 0};
}

#endif  // __CUDACC__

}  // namespace ft
