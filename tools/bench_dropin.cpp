// bench_dropin -- the reference-shaped C++ API (include/fasttrig/gpu.hpp) timed
// exactly as a C++ caller of R:proj/include/fasttrig/kernels.hpp:84-94 uses it:
// std::span<const double> in, a freshly allocated std::vector<double> out per
// call.  Built by paper_2502_10831_b200/Makefile into lib/bench_dropin; run by
// bench.py for its e2e_variants.
//
//   bench_dropin <n> <steps>     -> one JSON line
//
// Inputs are the configs[1] recipe (U[-1000pi, 1000pi], SplitMix64 counter
// stream, seed 2024873 + 2) generated on the host, identical to K4.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numbers>
#include <vector>

#include "fasttrig/gpu.hpp"

namespace {

std::uint64_t splitmix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

int main(int argc, char** argv) {
  const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : (std::size_t(1) << 26);
  const int steps = argc > 2 ? std::atoi(argv[2]) : 3;
  constexpr double pi = std::numbers::pi;
  const double lo = -1000.0 * pi, hi = 1000.0 * pi;
  const std::uint64_t seed = 2024873 + 2, gamma = 0x9e3779b97f4a7c15ull;
  std::vector<double> xs(n);
  for (std::size_t g = 0; g < n; ++g)
    xs[g] = lo + (hi - lo) * (static_cast<double>(splitmix64(seed + (g + 1) * gamma) >> 11) * 0x1p-53);

  namespace G = fasttrig::gpu;
  // warm: device pipeline and staging buffers
  (void)G::proposed_sin_batch(std::span<const double>(xs.data(), std::min<std::size_t>(n, 1 << 20)));

  double t3 = 0.0, tf = 0.0, checksum = 0.0;
  for (int k = 0; k < steps; ++k) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<double> s = G::proposed_sin_batch(xs);
    std::vector<double> c = G::proposed_cos_batch(xs);
    std::vector<double> t = G::proposed_tan_batch(xs);
    t3 += seconds_since(t0);
    checksum += s[n / 2] + c[n / 3];
    t0 = std::chrono::steady_clock::now();
    auto f = G::proposed_sincostan_batch<double>(xs);
    tf += seconds_since(t0);
    checksum += f.sin[n / 2] - s[n / 2];
  }
  // what a fresh std::vector<double>(n) costs by itself (allocation, value
  // initialisation, first-touch page faults) -- the part of the drop-in's time
  // that is not the library's
  double ta = 0.0;
  for (int k = 0; k < steps; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<double> v(n);
    ta += seconds_since(t0);
    checksum += v[n / 2];
  }
  // the span-out form into caller-owned (pageable, already touched) vectors
  std::vector<double> s(n), c(n), t(n);
  (void)G::proposed_batch<double>(xs, s, c, t);
  double ts = 0.0;
  for (int k = 0; k < steps; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    G::proposed_batch<double>(xs, s, c, t);
    ts += seconds_since(t0);
  }
  std::printf(
      "{\"elements\": %zu, \"steps\": %d, \"api_x3_std_vector_gelem_s\": %.6f, "
      "\"fused_std_vector_gelem_s\": %.6f, \"span_out_preallocated_gelem_s\": %.6f, "
      "\"new_std_vector_seconds\": %.4f, \"checksum\": %.17g}\n",
      n, steps, n * steps / t3 / 1e9, n * steps / tf / 1e9, n * steps / ts / 1e9, ta / steps, checksum);
  return 0;
}
