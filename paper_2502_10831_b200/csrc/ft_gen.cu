// ft_gen.cu -- K4 (seeded input generation in place) and K5 (L2 flush fill).
//
// K4 is counter-based SplitMix64: element g of the global stream
// is mix(seed + (g+1)*gamma), identical to the g-th output of the sequential
// generator, so every GPU writes its own shard [offset, offset+n) with no host
// staging, and the CPU oracle (oracle/ft_oracle.c: ora_gen_uniform) reproduces
// the uniform distributions bit for bit (IEEE mul/add only).
#include "ft_internal.h"

namespace ft {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ std::uint64_t splitmix64(std::uint64_t seed, std::uint64_t i) {
  std::uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double unit(std::uint64_t z) {  // [0, 1), 53 bits
  return __dmul_rn(static_cast<double>(z >> 11), 0x1p-53);
}

template <typename T>
__device__ __forceinline__ T narrow(double v) {
  if constexpr (sizeof(T) == 4) return __double2float_rn(v);
  else return v;
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    k_gen_uniform(T* __restrict__ out, std::size_t n, double lo, double span, std::uint64_t seed,
                  std::uint64_t offset) {
  const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const double u = unit(splitmix64(seed, offset + i));
    out[i] = narrow<T>(__dadd_rn(lo, __dmul_rn(span, u)));
  }
}

// x = (2k+1)*pi/2 + delta, k ~ U{kmin..kmax}, delta ~ N(0, 1e-3) clipped to
// +-0.05 (BASELINE.json configs[2]).  Box-Muller uses device log/sqrt/cos, so
// these bits are generated here only and copied to the host oracle.
template <typename T>
__global__ void __launch_bounds__(kThreads)
    k_gen_tan_stress(T* __restrict__ out, std::size_t n, std::int64_t kmin, std::int64_t kmax,
                     std::uint64_t seed, std::uint64_t offset) {
  const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  const double count = static_cast<double>(kmax - kmin + 1);
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const std::uint64_t g = 3 * (offset + i);
    const double u1 = unit(splitmix64(seed, g));
    const double u2 = __dmul_rn(static_cast<double>((splitmix64(seed, g + 1) >> 11) + 1), 0x1p-53);
    const double u3 = unit(splitmix64(seed, g + 2));
    std::int64_t k = kmin + static_cast<std::int64_t>(floor(__dmul_rn(u1, count)));
    k = k > kmax ? kmax : k;
    double delta = 1e-3 * sqrt(-2.0 * log(u2)) * cospi(2.0 * u3);
    delta = delta > 0.05 ? 0.05 : (delta < -0.05 ? -0.05 : delta);
    const double x = __dadd_rn(__dmul_rn(static_cast<double>(2 * k + 1), kHalfPi), delta);
    out[i] = narrow<T>(x);
  }
}

__global__ void __launch_bounds__(kThreads) k_fill(uint4* __restrict__ buf, std::size_t n16, unsigned v) {
  const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < n16;
       i += stride)
    buf[i] = make_uint4(v, v + 1, v + 2, v + 3);
}

template <typename T>
cudaError_t gen_go(int dist, double lo, double hi, std::uint64_t seed, std::uint64_t offset,
                   std::size_t n, void* x, cudaStream_t s) {
  unsigned blocks = 0;
  if (dist == FT_DIST_UNIFORM) {
    if (const cudaError_t e = persistent_blocks(reinterpret_cast<const void*>(k_gen_uniform<T>), kThreads, n, &blocks))
      return e;
    k_gen_uniform<T><<<blocks, kThreads, 0, s>>>(static_cast<T*>(x), n, lo, hi - lo, seed, offset);
  } else {
    if (const cudaError_t e = persistent_blocks(reinterpret_cast<const void*>(k_gen_tan_stress<T>), kThreads, n, &blocks))
      return e;
    k_gen_tan_stress<T><<<blocks, kThreads, 0, s>>>(static_cast<T*>(x), n,
                                                    static_cast<std::int64_t>(lo),
                                                    static_cast<std::int64_t>(hi), seed, offset);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gen(ft_dtype dt, int dist, double lo, double hi, std::uint64_t seed,
                       std::uint64_t offset, std::size_t n, void* x, cudaStream_t s) {
  return dt == FT_F32 ? gen_go<float>(dist, lo, hi, seed, offset, n, x, s)
                      : gen_go<double>(dist, lo, hi, seed, offset, n, x, s);
}

cudaError_t read_const_table_gen(Table* out) { return cudaMemcpyFromSymbol(out, c_table, sizeof(Table)); }

cudaError_t launch_fill(void* buf, std::size_t bytes, unsigned v, cudaStream_t s) {
  const std::size_t n16 = bytes / 16;
  unsigned blocks = 0;
  if (const cudaError_t e = persistent_blocks(reinterpret_cast<const void*>(k_fill), kThreads, n16, &blocks))
    return e;
  k_fill<<<blocks, kThreads, 0, s>>>(static_cast<uint4*>(buf), n16, v);
  count_launch();
  return cudaGetLastError();
}

}  // namespace ft
