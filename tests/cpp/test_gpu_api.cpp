// C++ drop-in test: the reference-shaped batch API (include/fasttrig/gpu.hpp)
// against known answers and the batch/scalar contract.  Built and run by
// tests/test_parity_gpu.py::test_cpp_dropin_program on the GPU box, where the
// reference headers are absent (the stand-in SqrtMode is used); compiled
// (-fsyntax-only) against the real reference headers by tests/test_cpp_header.py.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <vector>

#include "fasttrig/gpu.hpp"

static int failures = 0;
#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                   \
    }                                                               \
  } while (0)

int main() {
  using fasttrig::SqrtMode;
  namespace g = fasttrig::gpu;
  constexpr double pi = std::numbers::pi;
  std::vector<double> xs = {0.0, pi / 2, -pi / 2, pi / 4, pi, 1.5707, -0.0};

  auto s = g::proposed_sin_batch(xs);
  auto c = g::proposed_cos_batch(xs, SqrtMode::exact());
  auto t = g::proposed_tan_batch(xs);
  EXPECT(s.size() == xs.size());
  EXPECT(s[0] == 0.0);
  EXPECT(std::fabs(s[1] - 0.99853611925345331) < 1e-15);  // fisr(1) value at pi/2
  EXPECT(s[2] == -s[1]);
  EXPECT(std::fabs(c[4] + 1.0) <= 1e-9);
  EXPECT(std::isinf(t[5]) && t[5] > 0);                     // pole guard, kernels.hpp:62-64
  EXPECT(std::signbit(s[6]));                               // -0.0 -> -0.0
  EXPECT(std::fabs(t[3] - 0.99651) < 1e-5);                 // fisr tan(pi/4)

  // empty span -> empty vector
  EXPECT(g::proposed_sin_batch(std::span<const double>{}).empty());

  // fused == separate, bitwise
  auto f = g::proposed_sincostan_batch<double>(xs);
  EXPECT(std::memcmp(f.sin.data(), s.data(), xs.size() * 8) == 0);
  EXPECT(std::memcmp(f.tan.data(), t.data(), xs.size() * 8) == 0);

  // f32 overload: bitwise policy == (float) of the f64 result; default policy
  // within 2 ulp of it
  std::vector<float> xf(xs.begin(), xs.end());
  for (int k = 0; k < 2000; ++k) xf.push_back(-300.0f + 0.3f * static_cast<float>(k));
  auto sd = g::proposed_sin_batch(std::vector<double>(xf.begin(), xf.end()));
  EXPECT(g::f32_policy() == g::F32Policy::ulp2);
  auto sf = g::proposed_sin_batch(std::span<const float>(xf));
  for (std::size_t i = 0; i < xf.size(); ++i) {
    const float want = static_cast<float>(sd[i]);
    std::int32_t a, b;
    std::memcpy(&a, &sf[i], 4);
    std::memcpy(&b, &want, 4);
    EXPECT(std::abs(static_cast<long long>(a) - b) <= 2 && (a < 0) == (b < 0));
  }
  g::set_f32_policy(g::F32Policy::bitwise);
  auto sb = g::proposed_sin_batch(std::span<const float>(xf));
  for (std::size_t i = 0; i < xf.size(); ++i) EXPECT(sb[i] == static_cast<float>(sd[i]));
  g::set_f32_policy(g::F32Policy::ulp2);

  // larger batch: element i == element i of a one-element batch (kernels.hpp:82-83)
  std::vector<double> big(100003);
  for (std::size_t i = 0; i < big.size(); ++i) big[i] = -1e4 + 2e4 * (static_cast<double>(i) / big.size());
  auto bs = g::proposed_sin_batch(big);
  for (std::size_t i = 0; i < big.size(); i += 9973) {
    auto one = g::proposed_sin_batch(std::span<const double>(&big[i], 1));
    EXPECT(std::memcmp(&one[0], &bs[i], 8) == 0);
  }

  // Taylor
  auto ty = g::taylor_batch<double>(std::vector<double>{pi / 2}, 5);
  EXPECT(std::fabs(ty.sin[0] - (1 + 3.6e-6)) <= 1e-7);

  // invalid argument -> exception with the C-ABI message
  bool threw = false;
  try {
    g::taylor_batch<double>(xs, 42);
  } catch (const std::runtime_error& e) {
    threw = std::strstr(e.what(), "n_terms") != nullptr;
  }
  EXPECT(threw);

  // release the pipeline buffers; the next call re-creates them
  g::release();
  auto again = g::proposed_sin_batch(xs);
  EXPECT(std::memcmp(again.data(), s.data(), xs.size() * 8) == 0);

  std::printf("gpu.hpp drop-in: %s (%d failures)\n", failures ? "FAIL" : "OK", failures);
  return failures ? 1 : 0;
}
