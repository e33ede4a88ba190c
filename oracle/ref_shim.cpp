// oracle/ref_shim.cpp -- C-ABI wrapper around the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  This file contains no reference source: it
// #includes R:proj/include/fasttrig/kernels.hpp from /root/reference at build
// time (oracle/Makefile) and exports plain-C entry points so that
//   * tests/ can pin the C restatement (ft_oracle.c) bit-for-bit against the
//     real reference, and generate tests/golden/ fixtures;
//   * bench.py can time the reference's own CPU path as the baseline
//     ("cpu_baseline.kind": "reference").
// The output lands in oracle/_ref/ (git-ignored, travels to the GPU box).
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <span>
#include <thread>
#include <vector>

#include "fasttrig/kernels.hpp"

namespace {

fasttrig::SqrtMode make_mode(int method, int steps) {
  // Field-for-field construction (fisr.hpp:14-18), NOT SqrtMode::fisr(), so a
  // caller-provided steps value is honoured verbatim exactly like a struct
  // literal in C++ would be.
  fasttrig::SqrtMode m;
  m.method = method == 0 ? fasttrig::SqrtMode::Method::exact : fasttrig::SqrtMode::Method::fisr;
  m.newton_steps = steps;
  return m;
}

template <class T>
void run_range(const T* x, std::size_t lo, std::size_t hi, unsigned mask, fasttrig::SqrtMode mode,
               T* s, T* c, T* t, std::uint8_t* seg_sc, std::uint8_t* seg_t) {
  for (std::size_t i = lo; i < hi; ++i) {
    const double xd = static_cast<double>(x[i]);
    if (mask & 1u) s[i] = static_cast<T>(fasttrig::proposed_sin(xd, mode));
    if (mask & 2u) c[i] = static_cast<T>(fasttrig::proposed_cos(xd, mode));
    if (mask & 4u) t[i] = static_cast<T>(fasttrig::proposed_tan(xd, mode));
    if (seg_sc) seg_sc[i] = static_cast<std::uint8_t>(fasttrig::segment_index(fasttrig::reduce_sin(xd).red));
    if (seg_t) {
      const fasttrig::ReducedAngle ra = fasttrig::reduce_tan(xd);
      seg_t[i] = std::fabs(ra.red - fasttrig::detail::half_pi) < fasttrig::tan_pole_guard
                     ? 255
                     : static_cast<std::uint8_t>(fasttrig::segment_index(ra.red));
    }
  }
}

template <class T>
void run_threads(const T* x, std::size_t n, unsigned mask, fasttrig::SqrtMode mode, T* s, T* c,
                 T* t, std::uint8_t* seg_sc, std::uint8_t* seg_t, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (static_cast<std::size_t>(nthreads) > n) nthreads = n ? static_cast<int>(n) : 1;
  std::vector<std::thread> pool;
  for (int k = 1; k < nthreads; ++k) {
    pool.emplace_back(run_range<T>, x, n * k / nthreads, n * (k + 1) / nthreads, mask, mode, s, c,
                      t, seg_sc, seg_t);
  }
  run_range<T>(x, 0, n / nthreads, mask, mode, s, c, t, seg_sc, seg_t);
  for (auto& th : pool) th.join();
}

// float ulp distance on the ordered integer line (+0 and -0 coincide; NaN vs
// NaN is 0, NaN vs number is "infinite").
std::uint64_t ulp_f32(float a, float b) {
  const bool na = a != a, nb = b != b;
  if (na || nb) return (na && nb) ? 0 : ~0ull;
  std::int32_t ia, ib;
  std::memcpy(&ia, &a, 4);
  std::memcpy(&ib, &b, 4);
  const std::int64_t oa = ia < 0 ? -static_cast<std::int64_t>(ia & 0x7fffffff) : ia;
  const std::int64_t ob = ib < 0 ? -static_cast<std::int64_t>(ib & 0x7fffffff) : ib;
  return static_cast<std::uint64_t>(oa > ob ? oa - ob : ob - oa);
}

std::uint32_t canon_bits(float v) {
  std::uint32_t u;
  std::memcpy(&u, &v, 4);
  return v != v ? 0x7fc00000u : u;
}

}  // namespace

extern "C" {

// Exhaustive-range checker: for the float inputs whose bit patterns are
// start, start+1, ..., start+n-1 (mod 2^32), evaluates the reference
// (float)proposed_*((double)x) and compares it with got_{sin,cos,tan} (any may
// be NULL) and, when given, the segment choices seg_sc / seg_t.
// out[0..2] max ulp, out[3..5] raw-bit mismatches (NaNs canonical), out[6..8]
// elements over 2 ulp, out[9..10] segment mismatches (sin/cos, tan).
int ref_check_f32_range(std::uint32_t start, std::size_t n, int method, int steps,
                        const float* got_s, const float* got_c, const float* got_t,
                        const std::uint8_t* seg_sc, const std::uint8_t* seg_t, std::uint64_t* out,
                        int nthreads) {
  const auto mode = make_mode(method, steps);
  if (nthreads < 1) nthreads = 1;
  std::vector<std::array<std::uint64_t, 11>> acc(static_cast<std::size_t>(nthreads));
  auto work = [&](int k) {
    std::array<std::uint64_t, 11> a{};
    const std::size_t lo = n * k / nthreads, hi = n * (k + 1) / nthreads;
    const float* got[3] = {got_s, got_c, got_t};
    for (std::size_t i = lo; i < hi; ++i) {
      const std::uint32_t b = start + static_cast<std::uint32_t>(i);
      float xf;
      std::memcpy(&xf, &b, 4);
      const double x = static_cast<double>(xf);
      for (int j = 0; j < 3; ++j) {
        if (!got[j]) continue;
        const double r = j == 0 ? fasttrig::proposed_sin(x, mode)
                         : j == 1 ? fasttrig::proposed_cos(x, mode)
                                  : fasttrig::proposed_tan(x, mode);
        const float rf = static_cast<float>(r), g = got[j][i];
        const std::uint64_t u = ulp_f32(g, rf);
        a[j] = u > a[j] ? u : a[j];
        a[3 + j] += canon_bits(g) != canon_bits(rf);
        a[6 + j] += u > 2;
      }
      if (seg_sc) a[9] += seg_sc[i] != static_cast<std::uint8_t>(fasttrig::segment_index(fasttrig::reduce_sin(x).red));
      if (seg_t) {
        const fasttrig::ReducedAngle ra = fasttrig::reduce_tan(x);
        const std::uint8_t want = std::fabs(ra.red - fasttrig::detail::half_pi) < fasttrig::tan_pole_guard
                                      ? 255
                                      : static_cast<std::uint8_t>(fasttrig::segment_index(ra.red));
        a[10] += seg_t[i] != want;
      }
    }
    acc[static_cast<std::size_t>(k)] = a;
  };
  std::vector<std::thread> pool;
  for (int k = 1; k < nthreads; ++k) pool.emplace_back(work, k);
  work(0);
  for (auto& th : pool) th.join();
  for (int j = 0; j < 11; ++j) out[j] = 0;
  for (const auto& a : acc) {
    for (int j = 0; j < 3; ++j) out[j] = a[j] > out[j] ? a[j] : out[j];
    for (int j = 3; j < 11; ++j) out[j] += a[j];
  }
  return 0;
}


// Scalar reference calls (kernels.hpp:46-67) on pre-allocated outputs,
// partitioned contiguously over `nthreads` host threads.
int ref_proposed_batch(int dtype, const void* x, std::size_t n, unsigned mask, int method,
                       int steps, void* s, void* c, void* t, std::uint8_t* seg_sc,
                       std::uint8_t* seg_t, int nthreads) {
  const auto mode = make_mode(method, steps);
  if (dtype == 0) {
    run_threads(static_cast<const float*>(x), n, mask, mode, static_cast<float*>(s),
                static_cast<float*>(c), static_cast<float*>(t), seg_sc, seg_t, nthreads);
  } else {
    run_threads(static_cast<const double*>(x), n, mask, mode, static_cast<double*>(s),
                static_cast<double*>(c), static_cast<double*>(t), seg_sc, seg_t, nthreads);
  }
  return 0;
}

// API-faithful single-thread batch call (kernels.hpp:84-94): allocates the
// std::vector exactly as the reference does, then copies it out.
int ref_api_batch(int which, const double* x, std::size_t n, int method, int steps, double* out) {
  const auto mode = make_mode(method, steps);
  std::span<const double> xs(x, n);
  std::vector<double> v = which == 0   ? fasttrig::proposed_sin_batch(xs, mode)
                          : which == 1 ? fasttrig::proposed_cos_batch(xs, mode)
                                       : fasttrig::proposed_tan_batch(xs, mode);
  if (n) std::memcpy(out, v.data(), n * sizeof(double));
  return 0;
}

void ref_segment_table(double* out49) {
  const auto& t = fasttrig::segment_table;
  for (int k = 0; k < 6; ++k) {
    const auto& s = t.segments[static_cast<std::size_t>(k)];
    const double v[7] = {s.a, s.b, s.c, s.d, s.X, s.Y, s.Z};
    for (int j = 0; j < 7; ++j) out49[k * 7 + j] = v[j];
  }
  for (int j = 0; j < 7; ++j) out49[42 + j] = t.knots[static_cast<std::size_t>(j)];
}

int ref_segment_index(double red) { return fasttrig::segment_index(red); }

double ref_fast_inverse_sqrt(double v, int method, int steps) {
  return fasttrig::fast_inverse_sqrt(v, make_mode(method, steps));
}

void ref_reduce(int which, double x, double* red, double* sign) {
  const fasttrig::ReducedAngle ra = which == 0   ? fasttrig::reduce_sin(x)
                                    : which == 1 ? fasttrig::reduce_cos(x)
                                                 : fasttrig::reduce_tan(x);
  *red = ra.red;
  *sign = ra.sign;
}

double ref_scalar(int which, double x, int method, int steps) {
  const auto mode = make_mode(method, steps);
  return which == 0 ? fasttrig::proposed_sin(x, mode)
         : which == 1 ? fasttrig::proposed_cos(x, mode)
                      : fasttrig::proposed_tan(x, mode);
}

}  // extern "C"
