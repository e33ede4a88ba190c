// ft_check.cu -- K3: parity + error reduction.
//
// For every element: ulp distance of each requested output against the oracle
// (a host-oracle array copied to the device, or the device restatement
// mirror_* recomputed on the fly), segment-choice agreement, +-inf / NaN
// counts, an order-independent checksum of the output bit patterns, and the
// error against CUDA's double-precision libm (abs, and rel with the paper's
// |ref| > 1e-12 guard).  Per-thread accumulators are folded
// with warp shuffles and committed with one atomic per statistic per warp.
// Each element's inputs are loaded one iteration ahead; the ulp arithmetic runs
// only for outputs whose bits differ from the oracle's; libm's sine and cosine
// come from one sincos (bitwise sin, cos: tools/sincos_identity.cu).  A checker,
// outside every timed region: ~27 Gelem/s on configs[1] (profiles/README.md).
#include "ft_internal.h"

namespace ft {
namespace {

constexpr int kThreads = 256;

template <typename T>
struct Bits;
template <>
struct Bits<float> {
  static __device__ std::uint64_t raw(float v) { return static_cast<std::uint32_t>(__float_as_uint(v)); }
  static __device__ std::int64_t ordered(float v) {
    const std::int32_t b = __float_as_int(v);
    return b < 0 ? -static_cast<std::int64_t>(b & 0x7fffffff) : static_cast<std::int64_t>(b);
  }
  static constexpr std::uint64_t kNaN = 0x7fc00000u;
};
template <>
struct Bits<double> {
  static __device__ std::uint64_t raw(double v) { return d2u(v); }
  static __device__ std::int64_t ordered(double v) {
    const std::int64_t b = __double_as_longlong(v);
    return b < 0 ? -(b & 0x7fffffffffffffffll) : b;
  }
  static constexpr std::uint64_t kNaN = kQuietNaN;
};

template <typename T>
__device__ __forceinline__ std::uint64_t ulp_dist(T a, T b) {
  const bool na = isnan(a), nb = isnan(b);
  if (na || nb) return (na && nb) ? 0ull : ~0ull;
  const std::int64_t ia = Bits<T>::ordered(a), ib = Bits<T>::ordered(b);
  return ia >= ib ? static_cast<std::uint64_t>(ia) - static_cast<std::uint64_t>(ib)
                  : static_cast<std::uint64_t>(ib) - static_cast<std::uint64_t>(ia);
}

__device__ __forceinline__ std::uint64_t warp_max(std::uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const std::uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}
__device__ __forceinline__ std::uint64_t warp_sum(std::uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sumd(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct Acc {
  // per-thread counters fit 32 bits (a launch gives a thread < 2^32 elements);
  // they are widened in the warp fold
  unsigned n = 0;
  unsigned over[3] = {0, 0, 0}, seg_mm[2] = {0, 0};
  unsigned inf[3] = {0, 0, 0}, nan[3] = {0, 0, 0}, nfin[3] = {0, 0, 0};
  unsigned bits[3] = {0, 0, 0};  // raw-bit mismatches (ulp_dist treats +0 and -0 as equal)
  std::uint64_t max_ulp[3] = {0, 0, 0}, cks[3] = {0, 0, 0};
  // non-negative doubles kept as bit patterns (ordered like the values)
  std::uint64_t max_or[3] = {0, 0, 0}, max_abs[3] = {0, 0, 0}, max_rel[3] = {0, 0, 0};
  double sum_abs[3] = {0, 0, 0}, sum_rel[3] = {0, 0, 0};
};

__device__ __forceinline__ std::uint64_t umax(std::uint64_t a, std::uint64_t b) { return a > b ? a : b; }

// One element's inputs, loaded one iteration ahead of their use (K3 runs at 2-3
// blocks/SM: without the prefetch a third of its stall samples were the loads).
template <typename T>
struct Elem {
  T x;
  T got[3];
  T ref[3];
};

template <typename T>
__device__ __forceinline__ Elem<T> load_elem(const CheckArgs& a, std::size_t i) {
  Elem<T> e;
  e.x = static_cast<const T*>(a.x)[i];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    e.got[j] = T(0);
    e.ref[j] = T(0);
    if (a.mask & (1u << j)) {
      e.got[j] = static_cast<const T*>(a.got[j])[i];
      if (a.ref[j]) e.ref[j] = static_cast<const T*>(a.ref[j])[i];
    }
  }
  return e;
}

// SPEC 1: the common call -- proposed functions in the default SqrtMode
// (fisr, one Newton step) against the device restatement -- with the mode
// folded into the code; SPEC 0: everything else (runtime mode, Taylor, host
// oracle arrays).
template <typename T, int SPEC>
__device__ __forceinline__ T oracle_value(const CheckArgs& a, int j, const Elem<T>& e, double x) {
  if (SPEC == 0 && a.ref[j]) return e.ref[j];
  int seg = 0;
  double v;
  if (SPEC == 1) v = mirror_proposed(c_table, j, x, 1, 1, &seg);
  else if (a.kind == 0) v = mirror_proposed(c_table, j, x, a.method, a.steps, &seg);
  else v = mirror_taylor(c_taylor, j, x, a.n_terms);
  if constexpr (sizeof(T) == 4) return __double2float_rn(v);
  else return v;
}

#ifndef FT_MINB_K3
#define FT_MINB_K3 2
#endif
template <typename T, int SPEC>
__global__ void __launch_bounds__(kThreads, FT_MINB_K3) k_check(const CheckArgs a) {
  Acc acc;
  const std::size_t tid = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x;
  const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  Elem<T> cur{};
  if (tid < a.n) cur = load_elem<T>(a, tid);
  for (std::size_t i = tid; i < a.n; i += stride) {
    Elem<T> nxt{};
    if (i + stride < a.n) nxt = load_elem<T>(a, i + stride);
    const double xd = static_cast<double>(cur.x);
    acc.n += 1;
    // CUDA libm in binary64 (the error reference); sincos(x) is bitwise sin(x),
    // cos(x) (tools/sincos_identity.cu: 0 mismatches in 2^32 arguments) and
    // shares their argument reduction.
    double lib[3] = {0.0, 0.0, 0.0};
    if ((a.mask & 3u) == 3u) sincos(xd, &lib[0], &lib[1]);
    else if (a.mask & 1u) lib[0] = sin(xd);
    else if (a.mask & 2u) lib[1] = cos(xd);
    if (a.mask & 4u) lib[2] = tan(xd);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      if (!(a.mask & (1u << j))) continue;
      const T got = cur.got[j];
      const T want = oracle_value<T, SPEC>(a, j, cur, xd);
      const std::uint64_t bg = isnan(got) ? Bits<T>::kNaN : Bits<T>::raw(got);
      const std::uint64_t bw = isnan(want) ? Bits<T>::kNaN : Bits<T>::raw(want);
      const double g = static_cast<double>(got);
      if (bg != bw) {  // identical bits (the usual case): 0 ulp, no mismatch, |g - w| = 0
        const std::uint64_t u = ulp_dist<T>(got, want);
        acc.max_ulp[j] = umax(acc.max_ulp[j], u);
        acc.over[j] += u > a.ulp_tol;
        acc.bits[j] += 1;
        const double w = static_cast<double>(want);
        if (isfinite(g) && isfinite(w)) acc.max_or[j] = umax(acc.max_or[j], d2u(fabs(g - w)));
      }
      acc.inf[j] += isinf(g);
      acc.nan[j] += isnan(g);
      acc.cks[j] += bg;
      if (isfinite(g) && isfinite(lib[j])) {
        const double e = fabs(g - lib[j]);
        const double r = fabs(lib[j]) > 1e-12 ? e / fabs(lib[j]) : 0.0;
        acc.nfin[j] += 1;
        acc.max_abs[j] = umax(acc.max_abs[j], d2u(e));
        acc.max_rel[j] = umax(acc.max_rel[j], d2u(r));
        acc.sum_abs[j] += e;
        acc.sum_rel[j] += r;
      }
    }
    if (a.kind == 0 && (a.seg_sc || a.seg_t)) {
      int s0 = 0, s1 = 0;
      if (a.seg_sc) {
        (void)mirror_proposed(c_table, 0, xd, a.method, a.steps, &s0);
        acc.seg_mm[0] += a.seg_sc[i] != static_cast<std::uint8_t>(s0);
      }
      if (a.seg_t) {
        (void)mirror_proposed(c_table, 2, xd, a.method, a.steps, &s1);
        acc.seg_mm[1] += a.seg_t[i] != static_cast<std::uint8_t>(s1);
      }
    }
    cur = nxt;
  }
  // warp fold, one atomic per statistic per warp
  ft_stats* st = a.stats;
  const bool lead = (threadIdx.x & 31) == 0;
  std::uint64_t v = warp_sum(acc.n);
  if (lead && v) atomicAdd(reinterpret_cast<unsigned long long*>(&st->n_checked), v);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
#define FT_MAX(field, src)                                                              \
  v = warp_max(src);                                                                    \
  if (lead && v) atomicMax(reinterpret_cast<unsigned long long*>(&st->field), v);
#define FT_SUM(field, src)                                                              \
  v = warp_sum(src);                                                                    \
  if (lead && v) atomicAdd(reinterpret_cast<unsigned long long*>(&st->field), v);
    FT_MAX(max_ulp[j], acc.max_ulp[j])
    FT_SUM(n_over_tol[j], acc.over[j])
    FT_SUM(n_bit_mismatch[j], acc.bits[j])
    FT_SUM(n_inf[j], acc.inf[j])
    FT_SUM(n_nan[j], acc.nan[j])
    FT_SUM(n_finite_libm[j], acc.nfin[j])
    FT_SUM(checksum[j], acc.cks[j])
    FT_MAX(max_abs_vs_oracle[j], acc.max_or[j])
    FT_MAX(max_abs_vs_libm[j], acc.max_abs[j])
    FT_MAX(max_rel_vs_libm[j], acc.max_rel[j])
    double d = warp_sumd(acc.sum_abs[j]);
    if (lead && d != 0.0) atomicAdd(&st->sum_abs_vs_libm[j], d);
    d = warp_sumd(acc.sum_rel[j]);
    if (lead && d != 0.0) atomicAdd(&st->sum_rel_vs_libm[j], d);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    FT_SUM(seg_mismatch[j], acc.seg_mm[j])
  }
#undef FT_MAX
#undef FT_SUM
}

template <typename T, int SPEC>
cudaError_t check_launch(const CheckArgs& a, cudaStream_t s) {
  unsigned blocks = 0;
  if (const cudaError_t eg =
          persistent_blocks(reinterpret_cast<const void*>(k_check<T, SPEC>), kThreads, a.n, &blocks))
    return eg;
  k_check<T, SPEC><<<blocks, kThreads, 0, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <typename T>
cudaError_t check_go(const CheckArgs& a, cudaStream_t s) {
  const bool spec = a.kind == 0 && a.method == 1 && a.steps == 1 && !a.ref[0] && !a.ref[1] && !a.ref[2];
  return spec ? check_launch<T, 1>(a, s) : check_launch<T, 0>(a, s);
}

}  // namespace

cudaError_t read_const_table_check(Table* out) { return cudaMemcpyFromSymbol(out, c_table, sizeof(Table)); }

cudaError_t launch_check(ft_dtype dt, const CheckArgs& a, cudaStream_t s) {
  return dt == FT_F32 ? check_go<float>(a, s) : check_go<double>(a, s);
}

}  // namespace ft
