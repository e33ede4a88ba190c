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
//                 an exponent decrement (both exact for the values they see).
//             All products/sums that the reference rounds separately stay
//             separately rounded.
#pragma once

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

// Host-computed monotone thresholds (see ft_capi.cu: compute_thresholds).
struct Thresholds {
  double quad[3];  // smallest r >= 0 with floor(RN(r/(pi/2))) >= 1, 2, 3
  double guard;    // smallest red in [0,pi/2] with |RN(red - pi/2)| < 1e-3
};

// Sqrt-mode selector as a template parameter of the kernels.
enum SqrtKind : int { kExact = 0, kFisr1 = 1, kFisrN = 2 };

// Output mask bits (mirrors include/fasttrig_b200.h).
enum : unsigned { kSin = 1u, kCos = 2u, kTan = 4u };

#ifdef __CUDACC__

// Device copies of the constexpr tables (per translation unit; no relocatable
// device code needed).  Uniform-index reads only.
static __constant__ Table c_table = make_table();
static __constant__ TaylorCoeffs c_taylor = make_taylor();

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

// Coefficients staged in shared memory as pairs so one LDS.128 fetches two
// (lanes that land in the same segment broadcast; six segments span 96 B, so
// a warp's request never bank-conflicts).
struct SmemTable {
  double2 ab[6];
  double2 cd[6];
  double2 xy[6];
  double z[6];
};

__device__ __forceinline__ void stage_table(SmemTable* s) {
  for (int i = threadIdx.x; i < 6; i += blockDim.x) {
    const Coeffs& c = c_table.seg[i];
    s->ab[i] = make_double2(c.a, c.b);
    s->cd[i] = make_double2(c.c, c.d);
    s->xy[i] = make_double2(c.X, c.Y);
    s->z[i] = c.Z;
  }
}

template <int SQ>
__device__ __forceinline__ double fast_rsqrt(double v, int steps) {
  // Domain: v is a radicand in [1.98e5, 8.9e5] or a tan denominator > 0.63
  // for every finite x outside the pole guard (the only lanes whose value is
  // kept), so the NaN guard of fisr.hpp:32-34 never fires and 0.5*v is an
  // exact exponent decrement.
  if constexpr (SQ == kExact) {
    return __ddiv_rn(1.0, __dsqrt_rn(v));
  } else {
    double y = u2d(kFisrMagic - (d2u(v) >> 1));
    const double half_v = u2d(d2u(v) - (1ull << 52));
    if constexpr (SQ == kFisr1) {
      y = __dmul_rn(y, __dsub_rn(1.5, __dmul_rn(__dmul_rn(half_v, y), y)));
    } else {
      for (int i = 0; i < steps; ++i)
        y = __dmul_rn(y, __dsub_rn(1.5, __dmul_rn(__dmul_rn(half_v, y), y)));
    }
    return y;
  }
}

struct FastRed {
  double red;    // sin/cos reduced angle
  double redt;   // tan reduced angle
  bool neg_s, neg_c, neg_t;
  bool guard;    // tan inside the pole window
  bool finite;
};

template <bool NEED_SC, bool NEED_T>
__device__ __forceinline__ FastRed fast_reduce(double x, const Thresholds& th) {
  FastRed o;
  o.finite = isfinite(x);
  const double a = fabs(x);
  // q1 = RN(a / 2pi) exactly (Markstein): y = RN(1/2pi), q0 faithful.
  const double q0 = __dmul_rn(a, kInvTwoPi);
  const double rem = __fma_rn(-q0, kTwoPi, a);
  const double q1 = __fma_rn(rem, kInvTwoPi, q0);
  const bool xneg = signbit(x);
  if constexpr (NEED_SC) {
    // reduction.hpp:26-30 with period 2pi
    double r = __dsub_rn(a, __dmul_rn(kTwoPi, floor(q1)));
    r = r < 0.0 ? 0.0 : r;
    r = r < kTwoPi ? r : 0.0;
    // reduction.hpp:44-52: q = min(floor(RN(r/(pi/2))), 3) via thresholds
    const int q = (r >= th.quad[0]) + (r >= th.quad[1]) + (r >= th.quad[2]);
    // red = {r, pi - r, r - pi, 2pi - r}[q] as one rounded add
    const double base = q == 0 ? 0.0 : q == 1 ? kPi : q == 2 ? -kPi : kTwoPi;
    const double red = __dadd_rn(base, flip_sign(r, q & 1));
    o.red = red < 0.0 ? 0.0 : (red < kHalfPi ? red : kHalfPi);
    o.neg_s = (q >= 2) != xneg;
    o.neg_c = (q == 1) || (q == 2);
  }
  if constexpr (NEED_T) {
    // RN(a/pi) == 2*RN(a/2pi) exactly (2pi is an exact doubling of pi).
    double r = __dsub_rn(a, __dmul_rn(kPi, floor(__dadd_rn(q1, q1))));
    r = r < 0.0 ? 0.0 : r;
    r = r < kPi ? r : 0.0;
    const bool upper = r > kHalfPi;
    const double red = __dadd_rn(upper ? kPi : 0.0, flip_sign(r, upper));
    o.redt = red < 0.0 ? 0.0 : (red < kHalfPi ? red : kHalfPi);
    o.neg_t = upper != xneg;
    o.guard = o.redt >= th.guard;
  }
  return o;
}

__device__ __forceinline__ int fast_segment(double red) {
  constexpr double k1 = kTable.knots[1], k2 = kTable.knots[2], k3 = kTable.knots[3],
                   k4 = kTable.knots[4], k5 = kTable.knots[5];
  return (red >= k1) + (red >= k2) + (red >= k3) + (red >= k4) + (red >= k5);
}

struct Out3 {
  double s, c, t;
  int seg_sc, seg_t;
};

// Fused proposed sin/cos/tan of one element (kernels.hpp:46-67).  SEG: also
// produce both segment choices even for functions not in MASK.
template <int SQ, unsigned MASK, bool SEG = false>
__device__ __forceinline__ Out3 fast_proposed(double x, const SmemTable& tb, const Thresholds& th,
                                              int steps) {
  constexpr bool kSC = (MASK & (kSin | kCos)) != 0 || SEG;
  constexpr bool kT = (MASK & kTan) != 0 || SEG;
  const FastRed fr = fast_reduce<kSC, kT>(x, th);
  Out3 o{0.0, 0.0, 0.0, 0, 0};
  if constexpr (kSC) {
    const int k = fast_segment(fr.red);
    o.seg_sc = fr.finite ? k : 0;
    const double red = fr.red;
    const double2 xy = tb.xy[k];
    const double rad = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(xy.x, red), xy.y), red), tb.z[k]);
    const double rs = fast_rsqrt<SQ>(rad, steps);
    if constexpr (MASK & kSin) {
      const double2 ab = tb.ab[k];
      const double v = __dmul_rn(__dadd_rn(__dmul_rn(ab.x, red), ab.y), rs);
      o.s = fr.finite ? flip_sign(v, fr.neg_s) : u2d(kQuietNaN);
    }
    if constexpr (MASK & kCos) {
      const double2 cd = tb.cd[k];
      const double v = __dmul_rn(__dadd_rn(__dmul_rn(cd.x, red), cd.y), rs);
      o.c = fr.finite ? flip_sign(v, fr.neg_c) : u2d(kQuietNaN);
    }
  }
  if constexpr (kT) {
    const int k = fast_segment(fr.redt);
    o.seg_t = !fr.finite ? 0 : fr.guard ? 255 : k;
    const double red = fr.redt;
    const double2 ab = tb.ab[k];
    const double2 cd = tb.cd[k];
    const double poly = __dadd_rn(__dmul_rn(ab.x, red), ab.y);
    const double den = __dadd_rn(__dmul_rn(cd.x, red), cd.y);
    double v;
    if constexpr (SQ == kExact) {
      v = __ddiv_rn(poly, den);
    } else {
      const double r = fast_rsqrt<SQ>(den, steps);
      v = __dmul_rn(poly, __dmul_rn(r, r));
    }
    v = fr.guard ? __longlong_as_double(0x7ff0000000000000ll) : v;
    o.t = fr.finite ? flip_sign(v, fr.neg_t) : u2d(kQuietNaN);
  }
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

// Fused Taylor sin/cos/tan of one element, n nonzero terms.
template <int NT, unsigned MASK>
__device__ __forceinline__ Out3 fast_taylor(double x, const Thresholds& th, int n) {
  constexpr bool kSC = (MASK & (kSin | kCos)) != 0;
  constexpr bool kT = (MASK & kTan) != 0;
  const FastRed fr = fast_reduce<kSC, kT>(x, th);
  Out3 o{0.0, 0.0, 0.0, 0, 0};
  if constexpr (kSC) {
    const double s2 = __dmul_rn(fr.red, fr.red);
    if constexpr (MASK & kSin) {
      const double p = taylor_horner<NT>(c_taylor.sin_c, n, s2);
      o.s = fr.finite ? flip_sign(__dmul_rn(fr.red, p), fr.neg_s) : u2d(kQuietNaN);
    }
    if constexpr (MASK & kCos) {
      const double p = taylor_horner<NT>(c_taylor.cos_c, n, s2);
      o.c = fr.finite ? flip_sign(p, fr.neg_c) : u2d(kQuietNaN);
    }
  }
  if constexpr (kT) {
    const double s2 = __dmul_rn(fr.redt, fr.redt);
    const double p = taylor_horner<NT>(c_taylor.tan_c, n, s2);
    o.t = fr.finite ? flip_sign(__dmul_rn(fr.redt, p), fr.neg_t) : u2d(kQuietNaN);
  }
  return o;
}

#endif  // __CUDACC__

}  // namespace ft
