// fasttrig/gpu.hpp -- the reference's batch API, evaluated on B200.
//
// Drop-in for R:proj/include/fasttrig/kernels.hpp:84-94:
//
//   std::vector<double> fasttrig::proposed_sin_batch(std::span<const double>, SqrtMode = {});
//   -> std::vector<double> fasttrig::gpu::proposed_sin_batch(std::span<const double>, SqrtMode = {});
//
// Same argument meaning (SqrtMode is the reference's own type when its headers
// are on the include path), same per-element bits (element i equals the
// scalar proposed_sin(xs[i], mode), kernels.hpp:82-83), same error convention
// (the batch form may throw; here std::runtime_error carries the C-ABI error
// text, where the reference could only throw std::bad_alloc).  Everything is
// a thin inline layer over the C ABI in fasttrig_b200.h; link with
// -lfasttrig_b200.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#if __has_include("fasttrig/fisr.hpp")
#include "fasttrig/fisr.hpp"  // the reference's SqrtMode (fisr.hpp:14-24)
#define FASTTRIG_B200_REFERENCE_TYPES 1
#else
namespace fasttrig {
// Layout- and value-compatible stand-in for fasttrig::SqrtMode (fisr.hpp:14-24),
// used only when the reference headers are not on the include path.
struct SqrtMode {
  enum class Method : std::uint8_t { exact, fisr };
  Method method = Method::fisr;
  int newton_steps = 1;
  static constexpr SqrtMode exact() noexcept { return {Method::exact, 0}; }
  static constexpr SqrtMode fisr(int steps = 1) noexcept { return {Method::fisr, steps < 1 ? 1 : steps}; }
};
}  // namespace fasttrig
#define FASTTRIG_B200_REFERENCE_TYPES 0
#endif

#include "fasttrig_b200.h"

namespace fasttrig::gpu {

inline constexpr unsigned kSin = FT_OUT_SIN, kCos = FT_OUT_COS, kTan = FT_OUT_TAN;

inline ft_sqrt_mode to_c(SqrtMode m) noexcept {
  return ft_sqrt_mode{m.method == SqrtMode::Method::exact ? FT_SQRT_EXACT : FT_SQRT_FISR,
                      m.newton_steps};
}

inline void check(int rc) {
  if (rc != FT_OK) throw std::runtime_error(std::string("fasttrig_b200: ") + ft_last_error_string());
}

template <class T>
constexpr ft_dtype dtype_of() {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "float or double");
  return std::is_same_v<T, float> ? FT_F32 : FT_F64;
}

// How many GPUs one host-memory call spreads over (default 1; n <= 0: all
// visible).  Arrays of >= 4 Mi elements are split into contiguous shards, one
// device and host thread each; results do not depend on the setting.
inline void set_devices(int n) { check(ft_set_host_devices(n)); }

// Free the host-pointer pipeline and staging buffers of `device` (-1: all);
// they are re-created on demand.
inline void release(int device = -1) { check(ft_release(device)); }

// ---- reference-shaped batch calls (host memory in, host memory out) ----
inline std::vector<double> proposed_sin_batch(std::span<const double> xs, SqrtMode mode = {}) {
  std::vector<double> out(xs.size());
  check(ft_proposed_sin_batch(xs.data(), xs.size(), to_c(mode), out.data()));
  return out;
}
inline std::vector<double> proposed_cos_batch(std::span<const double> xs, SqrtMode mode = {}) {
  std::vector<double> out(xs.size());
  check(ft_proposed_cos_batch(xs.data(), xs.size(), to_c(mode), out.data()));
  return out;
}
inline std::vector<double> proposed_tan_batch(std::span<const double> xs, SqrtMode mode = {}) {
  std::vector<double> out(xs.size());
  check(ft_proposed_tan_batch(xs.data(), xs.size(), to_c(mode), out.data()));
  return out;
}

// f32 evaluation policy (process-wide).  Default F32Policy::ulp2: within 2 ulp
// of (float)proposed_*((double)x) with the identical segment choice (checked on
// all 2^32 floats); F32Policy::bitwise: bit-identical to it.
enum class F32Policy : int { ulp2 = FT_F32_ULP2, bitwise = FT_F32_BITWISE };
inline void set_f32_policy(F32Policy p) { check(ft_set_f32_policy(static_cast<int>(p))); }
inline F32Policy f32_policy() { return static_cast<F32Policy>(ft_get_f32_policy()); }

// f32 overloads: (float)proposed_*((double)x) per element, at the f32 policy.
inline std::vector<float> proposed_sin_batch(std::span<const float> xs, SqrtMode mode = {}) {
  std::vector<float> out(xs.size());
  check(ft_proposed_batch_host(FT_F32, xs.data(), xs.size(), kSin, to_c(mode), out.data(), nullptr, nullptr));
  return out;
}
inline std::vector<float> proposed_cos_batch(std::span<const float> xs, SqrtMode mode = {}) {
  std::vector<float> out(xs.size());
  check(ft_proposed_batch_host(FT_F32, xs.data(), xs.size(), kCos, to_c(mode), nullptr, out.data(), nullptr));
  return out;
}
inline std::vector<float> proposed_tan_batch(std::span<const float> xs, SqrtMode mode = {}) {
  std::vector<float> out(xs.size());
  check(ft_proposed_batch_host(FT_F32, xs.data(), xs.size(), kTan, to_c(mode), nullptr, nullptr, out.data()));
  return out;
}

// ---- fused forms: read x once, write any subset of {sin, cos, tan} ----
template <class T>
struct SinCosTan {
  std::vector<T> sin, cos, tan;
};

template <class T>
SinCosTan<T> proposed_sincostan_batch(std::span<const T> xs, SqrtMode mode = {}, unsigned mask = 7) {
  SinCosTan<T> r;
  if (mask & kSin) r.sin.resize(xs.size());
  if (mask & kCos) r.cos.resize(xs.size());
  if (mask & kTan) r.tan.resize(xs.size());
  check(ft_proposed_batch_host(dtype_of<T>(), xs.data(), xs.size(), mask, to_c(mode),
                               (mask & kSin) ? r.sin.data() : nullptr,
                               (mask & kCos) ? r.cos.data() : nullptr,
                               (mask & kTan) ? r.tan.data() : nullptr));
  return r;
}

// Span-out form (no allocation; pinned buffers stream at full PCIe rate).
template <class T>
void proposed_batch(std::span<const T> xs, std::span<T> sin_out, std::span<T> cos_out,
                    std::span<T> tan_out, SqrtMode mode = {}) {
  unsigned mask = 0;
  if (!sin_out.empty()) mask |= kSin;
  if (!cos_out.empty()) mask |= kCos;
  if (!tan_out.empty()) mask |= kTan;
  for (auto s : {sin_out.size(), cos_out.size(), tan_out.size()})
    if (s != 0 && s != xs.size()) throw std::invalid_argument("fasttrig_b200: output span size mismatch");
  if (mask == 0 || xs.empty()) return;
  check(ft_proposed_batch_host(dtype_of<T>(), xs.data(), xs.size(), mask, to_c(mode),
                               sin_out.empty() ? nullptr : sin_out.data(),
                               cos_out.empty() ? nullptr : cos_out.data(),
                               tan_out.empty() ? nullptr : tan_out.data()));
}

// Taylor comparator, n_terms nonzero terms.
template <class T>
SinCosTan<T> taylor_batch(std::span<const T> xs, int n_terms = 5, unsigned mask = kSin | kCos) {
  SinCosTan<T> r;
  if (mask & kSin) r.sin.resize(xs.size());
  if (mask & kCos) r.cos.resize(xs.size());
  if (mask & kTan) r.tan.resize(xs.size());
  check(ft_taylor_batch_host(dtype_of<T>(), xs.data(), xs.size(), mask, n_terms,
                             (mask & kSin) ? r.sin.data() : nullptr,
                             (mask & kCos) ? r.cos.data() : nullptr,
                             (mask & kTan) ? r.tan.data() : nullptr));
  return r;
}

// ---- device-resident form: pointers in GPU memory, async on `stream` ----
template <class T>
void proposed_eval_device(const T* x, std::size_t n, unsigned mask, SqrtMode mode, T* sin_out,
                          T* cos_out, T* tan_out, void* stream = nullptr) {
  check(ft_proposed_eval(dtype_of<T>(), x, n, mask, to_c(mode), sin_out, cos_out, tan_out, stream));
}

}  // namespace fasttrig::gpu
