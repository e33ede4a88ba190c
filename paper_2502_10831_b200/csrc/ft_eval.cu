// ft_eval.cu -- K1 (fused proposed sin/cos/tan), K2 (Taylor) and the device
// restatement kernel, all streaming elementwise maps over HBM.
//
// Layout: x is one contiguous array (f32 or f64); each requested output is its
// own contiguous array of the same dtype (three separate arrays, as the
// reference returns three vectors from proposed_*_batch, kernels.hpp:84-94).
// Each thread moves 16 B per access (float4 / double2) with streaming cache
// hints; the grid is persistent (#SM x resident blocks) and grid-strides.
#include <cstdlib>

#include "ft_internal.h"

namespace ft {
namespace {

constexpr int kThreads = 256;
// Output path per dtype.  f64 (32 B/elem at cfg2, memory-bound): block tiles
// written by TMA bulk stores, compiled for >= 3 blocks/SM (60 registers: 4 are
// resident) -- 12% faster per launch than per-thread stores (6.16 vs 5.51 TB/s).
// f32 (16 B/elem, instruction-bound): per-thread streaming stores at 4 blocks/SM
// (the TMA path costs it 3-5%).  profiles/r01_k1_variants.json.
#ifndef FT_TMA_F64
#define FT_TMA_F64 1
#endif
#ifndef FT_TMA_TAYLOR_F32
#define FT_TMA_TAYLOR_F32 0
#endif
// TMA-store kernels: threads per block and vectors per thread per tile.
#ifndef FT_TMA_THREADS
#define FT_TMA_THREADS 256
#endif
#ifndef FT_TMA_VPT
#define FT_TMA_VPT 1
#endif
constexpr unsigned kTmaThreads = FT_TMA_THREADS;
constexpr int kTmaVpt = FT_TMA_VPT;
template <typename T>
constexpr bool kTmaK1 = sizeof(T) == 8 && FT_TMA_F64;
template <typename T>
constexpr bool kTmaK2 = (sizeof(T) == 8 && FT_TMA_F64) || (sizeof(T) == 4 && FT_TMA_TAYLOR_F32);
#ifndef FT_MINB_F32
#define FT_MINB_F32 4  // resident blocks/SM the f32 kernels are compiled for (register cap)
#endif
template <typename T>
constexpr int kMinBlocks = kTmaK1<T> ? 3 * 256 / kTmaThreads : FT_MINB_F32;
// Block size per kernel family (TMA-store kernels may differ, FT_TMA_THREADS).
template <typename T>
constexpr unsigned kBlockK1 = kTmaK1<T> ? kTmaThreads : kThreads;
// K2 f32 (Taylor, 40 registers suffice): 6 resident blocks/SM measured +4.8%
// over 4 (cfg4 f32: 4 -> 5 -> 6 blocks 434 -> 449 -> 454 Gelem/s; 8 spills);
// K1 f32 loses 2-6% at 5.
#ifndef FT_MINB_K2_F32
#define FT_MINB_K2_F32 6
#endif
// The 40-register cap spills in the tan-including instantiations (76 B at NT=0),
// so those keep K1's 4 blocks/SM.
template <typename T, unsigned MASK>
constexpr int kMinBlocksK2 =
    kTmaK2<T> ? 3 * 256 / kTmaThreads : (sizeof(T) == 4 && (MASK & kTan) == 0 ? FT_MINB_K2_F32 : FT_MINB_F32);
template <typename T>
constexpr unsigned kBlockK2 = kTmaK2<T> ? kTmaThreads : kThreads;
// Where the exact-path branch sits: 0 one per element; 1 one per vector for
// tan-only kernels (cfg3 +5%; the fused kernels lose 10% to the extra live
// registers at the 64-register cap); 2 one per vector everywhere.
#ifndef FT_BATCH_SLOW
#define FT_BATCH_SLOW 1
#endif
#ifndef FT_GROUP_RECHECK
#define FT_GROUP_RECHECK 1  // relaxed kernels: the rare exact-path block re-derives which elements of the group failed
#endif
#ifndef FT_RPF
#define FT_RPF 1  // 1: register prefetch of the next x (0: load at use)
#endif

template <typename T>
struct Vec;
template <>
struct Vec<float> {
  using type = float4;
  static constexpr int N = 4;
  __device__ static void unpack(const float4& v, float* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
  __device__ static float4 pack(const float* o) { return make_float4(o[0], o[1], o[2], o[3]); }
};
template <>
struct Vec<double> {
  using type = double2;
  static constexpr int N = 2;
  __device__ static void unpack(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
  __device__ static double2 pack(const double* o) { return make_double2(o[0], o[1]); }
};

template <typename T>
__device__ __forceinline__ T to_out(double v);
template <>
__device__ __forceinline__ float to_out<float>(double v) { return __double2float_rn(v); }
template <>
__device__ __forceinline__ double to_out<double>(double v) { return v; }
// Relaxed f32 ops already return floats.
template <typename T>
__device__ __forceinline__ T to_out(float v) { return v; }

// TMA bulk store smem -> global (SASS UBLKCP) and its bulk-group completion.
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(ssrc));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Cache hints of the per-thread streaming accesses (experiments: FT_LD_CS=0
// plain loads, FT_ST_CS=0 plain write-back stores).
#ifndef FT_LD_CS
#define FT_LD_CS 1
#endif
#ifndef FT_ST_CS
#define FT_ST_CS 1
#endif
template <typename V>
__device__ __forceinline__ V ld_x(const V* p) {
  if constexpr (FT_LD_CS) return __ldcs(p);
  else return __ldg(p);
}
template <typename V>
__device__ __forceinline__ void st_out(V* p, const V& v) {
  if constexpr (FT_ST_CS) __stcs(p, v);
  else *p = v;
}

// The streaming map shared by every evaluation kernel.  `op(T) -> Out3` (or
// Out3f for the relaxed f32 ops).
template <typename T, unsigned MASK, bool SEG, class Op, bool TMA = false>
__device__ __forceinline__ void stream_map(const EvalArgs& a, const Op& op) {
  using V = Vec<T>;
  using VT = typename V::type;
  constexpr int VN = V::N;
  // 32-bit indices: each launch covers < 2^31 elements (launch_* split larger
  // arrays), so addresses are one IMAD.WIDE.U32 each instead of 64-bit math.
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned stride = gridDim.x * blockDim.x;
  const unsigned n = static_cast<unsigned>(a.n);
  const T* __restrict__ x = static_cast<const T*>(a.x);
  T* __restrict__ o0 = static_cast<T*>(a.out[0]);
  T* __restrict__ o1 = static_cast<T*>(a.out[1]);
  T* __restrict__ o2 = static_cast<T*>(a.out[2]);
  unsigned done = 0;
  if (a.vec_ok) {
    const unsigned nv = n / VN;
    const VT* __restrict__ xv = reinterpret_cast<const VT*>(x);
    // Evaluate + store one vector.
    // Evaluate one vector into res[] (+ segment bytes in the SEG variant).
    auto compute = [&](const VT& xin, unsigned v, VT res[3]) {
      T xs[VN], rs[VN], rc[VN], rt[VN];
      std::uint8_t g0[VN], g1[VN];
      V::unpack(xin, xs);
      auto put = [&](int j, const auto& o) {
        rs[j] = to_out<T>(o.s);
        rc[j] = to_out<T>(o.c);
        rt[j] = to_out<T>(o.t);
        g0[j] = static_cast<std::uint8_t>(o.seg_sc);
        g1[j] = static_cast<std::uint8_t>(o.seg_t);
      };
      constexpr int G = Op::template kGroup<T> < VN ? Op::template kGroup<T> : VN;
      if constexpr (G > 1) {
        // Groups of G elements: the fast path of every element of the group
        // first (no branch between them, so the compiler can interleave their
        // dependency chains), then one rarely-taken branch that redoes the
        // failing ones exactly.
#pragma unroll
        for (int j0 = 0; j0 < VN; j0 += G) {
          using OutT = decltype(op.core(xs[0], nullptr));
          OutT ov[G];
          bool okv[G];
          bool all = true;
#pragma unroll
          for (int j = 0; j < G; ++j) {
            ov[j] = op.core(xs[j0 + j], &okv[j]);
            all = all && okv[j];
          }
          if (!all) {
            if constexpr (Op::kRecheck) {
              // Rare block: find the failing elements again from x itself (the
              // opaque copy stops the compiler from keeping G pass/fail
              // predicates alive across the branch, which it does by packing
              // them into a register with ~5 extra instructions per element).
#pragma unroll
              for (int j = 0; j < G; ++j) {
                T xj = xs[j0 + j];
                if constexpr (sizeof(T) == 4) asm volatile("" : "+f"(xj));
                else asm volatile("" : "+d"(xj));
                bool okj;
                (void)op.core(xj, &okj);
                if (!okj) ov[j] = op.slow(xj);
              }
            } else {
#pragma unroll
              for (int j = 0; j < G; ++j)
                if (!okv[j]) ov[j] = op.slow(xs[j0 + j]);
            }
          }
#pragma unroll
          for (int j = 0; j < G; ++j) put(j0 + j, ov[j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < VN; ++j) put(j, op(xs[j]));
      }
      res[0] = V::pack(rs);
      res[1] = V::pack(rc);
      res[2] = V::pack(rt);
      if constexpr (SEG) {
#pragma unroll
        for (int j = 0; j < VN; ++j) {
          if (a.seg_sc) a.seg_sc[v * VN + j] = g0[j];
          if (a.seg_t) a.seg_t[v * VN + j] = g1[j];
        }
      }
    };
    // Evaluate + store one vector with per-thread 16-byte streaming stores.
    auto body = [&](const VT& xin, unsigned v) {
      VT res[3];
      compute(xin, v, res);
      if constexpr ((MASK & kSin) != 0) st_out(reinterpret_cast<VT*>(o0) + v, res[0]);
      if constexpr ((MASK & kCos) != 0) st_out(reinterpret_cast<VT*>(o1) + v, res[1]);
      if constexpr ((MASK & kTan) != 0) st_out(reinterpret_cast<VT*>(o2) + v, res[2]);
    };
    if constexpr (TMA && !SEG) {
      // Block tiles of kTmaVpt x kTmaThreads vectors (each thread kTmaVpt
      // vectors, kTmaThreads apart); x register-prefetched one tile ahead;
      // outputs staged in a 3-slot shared-memory ring and written by one
      // thread as one TMA bulk store per output array per tile.  One barrier
      // per tile: after issuing tile i, thread 0 waits until the bulk store of
      // tile i-1 has read its slot; the next barrier publishes that to every
      // thread before the slot is refilled (tile i+2).
      constexpr unsigned kTile = kTmaVpt * kTmaThreads;
      __shared__ __align__(128) VT stage[3][3][kTile];
      const unsigned nt = nv / kTile;
      unsigned t = blockIdx.x;
      VT cur[kTmaVpt];
#pragma unroll
      for (int k = 0; k < kTmaVpt; ++k) cur[k] = VT{};
      if (t < nt) {
#pragma unroll
        for (int k = 0; k < kTmaVpt; ++k) cur[k] = __ldcs(xv + (t * kTile + k * kTmaThreads + threadIdx.x));
      }
      unsigned slot = 0;
      for (; t < nt; t += gridDim.x, slot = slot == 2 ? 0 : slot + 1) {
        VT nxt[kTmaVpt];
#pragma unroll
        for (int k = 0; k < kTmaVpt; ++k) nxt[k] = VT{};
        if (t + gridDim.x < nt) {
#pragma unroll
          for (int k = 0; k < kTmaVpt; ++k)  // 32-bit element index: one IMAD.WIDE.U32 per address
            nxt[k] = __ldcs(xv + ((t + gridDim.x) * kTile + k * kTmaThreads + threadIdx.x));
        }
#pragma unroll
        for (int k = 0; k < kTmaVpt; ++k) {
          VT res[3];
          compute(cur[k], t * kTile + k * kTmaThreads + threadIdx.x, res);
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (MASK & (1u << j)) stage[slot][j][k * kTmaThreads + threadIdx.x] = res[j];
        }
#pragma unroll
        for (int k = 0; k < kTmaVpt; ++k) cur[k] = nxt[k];
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (MASK & (1u << j))
              bulk_store(reinterpret_cast<VT*>(j == 0 ? o0 : j == 1 ? o1 : o2) + t * kTile,
                         &stage[slot][j][0], kTile * sizeof(VT));
          bulk_commit();
          bulk_wait_read_1();  // tile i-1's slot is free once the next barrier passes
        }
      }
      for (unsigned v = nt * kTile + tid; v < nv; v += stride) body(__ldcs(xv + v), v);
      if (threadIdx.x == 0) bulk_wait_all();
    } else {
#if FT_RPF
    // Register prefetch: the next iteration's x is loaded before this one is
    // evaluated, so its DRAM latency (reads queue behind the write stream)
    // overlaps the arithmetic.  With 4 blocks/SM (<= 64 registers) this beat
    // direct loads, cp.async / TMA staging, L2 prefetch hints and prefetching
    // two iterations ahead (profiles/r01_k1_variants.json).
#if FT_RPF == 2
    VT cur{}, nx1{};
    if (tid < nv) cur = ld_x(xv + tid);
    if (tid + stride < nv) nx1 = ld_x(xv + tid + stride);
    for (unsigned v = tid; v < nv; v += stride) {
      VT nx2{};
      if (v + 2 * stride < nv) nx2 = ld_x(xv + v + 2 * stride);
      body(cur, v);
      cur = nx1;
      nx1 = nx2;
    }
#else
    VT cur{};
    if (tid < nv) cur = ld_x(xv + tid);
    for (unsigned v = tid; v < nv; v += stride) {
      VT nxt{};
      const unsigned vn = v + stride;  // 32-bit index: one IMAD.WIDE.U32 per address
      if (vn < nv) nxt = ld_x(xv + vn);
      body(cur, v);
      cur = nxt;
    }
#endif
#else
    for (unsigned v = tid; v < nv; v += stride) body(__ldcs(xv + v), v);
#endif
    }

    done = nv * VN;
  }
  pdl_trigger();
  for (unsigned i = done + tid; i < n; i += stride) {
    const auto o = op(x[i]);
    if constexpr ((MASK & kSin) != 0) o0[i] = to_out<T>(o.s);
    if constexpr ((MASK & kCos) != 0) o1[i] = to_out<T>(o.c);
    if constexpr ((MASK & kTan) != 0) o2[i] = to_out<T>(o.t);
    if constexpr (SEG) {
      if (a.seg_sc) a.seg_sc[i] = static_cast<std::uint8_t>(o.seg_sc);
      if (a.seg_t) a.seg_t[i] = static_cast<std::uint8_t>(o.seg_t);
    }
  }
}


template <int SQ, unsigned MASK, bool SEG>
struct ProposedOp {
  // Elements per exact-path branch (see stream_map).
  template <typename T>
  static constexpr int kGroup =
      FT_BATCH_SLOW == 2 ? 4 : (FT_BATCH_SLOW == 1 && MASK == kTan) ? 4 : 1;
  static constexpr bool kRecheck = false;
  const SmemTable* tb;
  int steps;
  __device__ __forceinline__ Out3 operator()(double x) const {
    return fast_proposed<SQ, MASK, SEG>(x, *tb, steps);
  }
  __device__ __forceinline__ Out3 core(double x, bool* ok) const {
    return fast_proposed_core<SQ, MASK, SEG>(x, *tb, steps, ok);
  }
  __device__ __forceinline__ Out3 slow(double x) const { return slow_proposed_mode<SQ>(x, steps); }
};

template <int NT, unsigned MASK, bool CERT>
struct TaylorOp {
  template <typename T>
  static constexpr int kGroup = 1;
  static constexpr bool kRecheck = false;
  int n;
  __device__ __forceinline__ Out3 operator()(double x) const { return fast_taylor<NT, MASK, CERT>(x, n); }
};

// Relaxed f32 proposed path (ft_core.cuh: relaxed_proposed_core): certified
// lanes within 2 ulp of the reference, the rest redone bit-exactly.
#ifndef FT_NULL_EVAL
#define FT_NULL_EVAL 0  // 1: tools-only build whose relaxed kernels copy x (roofline of the loop itself)
#endif
#ifndef FT_RELAX_GROUP
#define FT_RELAX_GROUP 1  // elements per exact-path branch in the relaxed kernels
#endif
#ifndef FT_RELAX_GROUP_TAN
#define FT_RELAX_GROUP_TAN 2  // the same for the tan-only relaxed kernels (cfg3 +1.2% over 1, r02bb/bc; 4: -1.5%)
#endif
template <int SQ, unsigned MASK, bool SEG>
struct RelaxedOp {
  template <typename T>
  static constexpr int kGroup = MASK == kTan ? FT_RELAX_GROUP_TAN : FT_RELAX_GROUP;
  static constexpr bool kRecheck = FT_GROUP_RECHECK != 0;
  const RelaxTable* tb;  // relaxed rows
  const SmemTable* tbx;  // bit-exact rows (fallback)
  int steps;
  __device__ __forceinline__ Out3f operator()(float x) const {
#if FT_NULL_EVAL
    return Out3f{x, x, x, 0, 0};  // measurement-only build: the kernel's traffic without its math
#endif
    bool ok;
    Out3f o = relaxed_proposed_core<SQ, MASK, SEG>(x, *tb, steps, &ok);
    if (!ok) o = relaxed_slow<SQ, MASK, SEG>(x, tbx, steps);  // rare
    return o;
  }
  __device__ __forceinline__ Out3f core(float x, bool* ok) const {
    return relaxed_proposed_core<SQ, MASK, SEG>(x, *tb, steps, ok);
  }
  __device__ __forceinline__ Out3f slow(float x) const { return relaxed_slow<SQ, MASK, SEG>(x, tbx, steps); }
};

template <int NT, unsigned MASK>
struct RelaxedTaylorOp {
  template <typename T>
  static constexpr int kGroup = FT_RELAX_GROUP;
  static constexpr bool kRecheck = FT_GROUP_RECHECK != 0;
  __device__ __forceinline__ Out3f operator()(float x) const {
    bool ok;
    Out3f o = relaxed_taylor_core<NT, MASK>(x, &ok);
    if (!ok) o = relaxed_taylor_slow<NT, MASK>(x);  // rare
    return o;
  }
  __device__ __forceinline__ Out3f core(float x, bool* ok) const { return relaxed_taylor_core<NT, MASK>(x, ok); }
  __device__ __forceinline__ Out3f slow(float x) const { return relaxed_taylor_slow<NT, MASK>(x); }
};

// Device restatement: each function evaluated separately, exactly as the
// reference scalar code does (kernels.hpp:46-67 / SPEC.md:224-247).
template <unsigned MASK>
struct MirrorOp {
  template <typename T>
  static constexpr int kGroup = 1;
  static constexpr bool kRecheck = false;
  int kind, method, steps, n;
  __device__ __forceinline__ Out3 operator()(double x) const {
    Out3 o{0.0, 0.0, 0.0, 0, 0};
    if (kind == 0) {
      int seg_cos = 0;
      const double s = mirror_proposed(c_table, 0, x, method, steps, &o.seg_sc);
      if (MASK & kSin) o.s = s;
      if (MASK & kCos) o.c = mirror_proposed(c_table, 1, x, method, steps, &seg_cos);
      const double t = mirror_proposed(c_table, 2, x, method, steps, &o.seg_t);
      if (MASK & kTan) o.t = t;
    } else {
      if (MASK & kSin) o.s = mirror_taylor(c_taylor, 0, x, n);
      if (MASK & kCos) o.c = mirror_taylor(c_taylor, 1, x, n);
      if (MASK & kTan) o.t = mirror_taylor(c_taylor, 2, x, n);
    }
    return o;
  }
};

// ---------------- K1 ----------------
template <typename T, int SQ, unsigned MASK, bool SEG>
__global__ void __launch_bounds__(kBlockK1<T>, kMinBlocks<T>) k_proposed(const EvalArgs a) {
  __shared__ SmemTable tb;
  stage_table(&tb);
  pdl_wait();
  __syncthreads();
  stream_map<T, MASK, SEG, ProposedOp<SQ, MASK, SEG>, kTmaK1<T>>(a, ProposedOp<SQ, MASK, SEG>{&tb, a.steps});
}

// ---------------- K2 ----------------
template <typename T, int NT, unsigned MASK>
__global__ void __launch_bounds__(kBlockK2<T>, (kMinBlocksK2<T, MASK>)) k_taylor(const EvalArgs a) {
  using Op = TaylorOp<NT, MASK, sizeof(T) == 4>;  // certify-or-redo for the instruction-bound f32 kernels
  pdl_wait();
  stream_map<T, MASK, false, Op, kTmaK2<T>>(a, Op{a.steps});
}

// ---------------- relaxed f32 K1 / K2 ----------------
#ifndef FT_MINB_RELAX
#define FT_MINB_RELAX 4
#endif
#ifndef FT_TMA_RELAX
#define FT_TMA_RELAX 0
#endif
// Relaxed Taylor f32: 5 blocks/SM (48 registers) measured 496 vs 462 Gelem/s
// at 4 (cfg4 f32, r02c); tan-including masks keep 4.
#ifndef FT_MINB_RELAX_TAYLOR
#define FT_MINB_RELAX_TAYLOR 5
#endif
#ifndef FT_MINB_RELAX_TAN
#define FT_MINB_RELAX_TAN 4  // tan-only relaxed kernels (52 registers at 4)
#endif
template <int SQ, unsigned MASK, bool SEG>
__global__ void __launch_bounds__(kThreads, MASK == kTan ? FT_MINB_RELAX_TAN : FT_MINB_RELAX)
    k_proposed_relaxed(const EvalArgs a) {
  __shared__ RelaxTable tb;
  __shared__ SmemTable tbx;
  stage_table_relaxed<MASK, SEG>(&tb);
  stage_table(&tbx);
  pdl_wait();
  __syncthreads();
  using Op = RelaxedOp<SQ, MASK, SEG>;
  stream_map<float, MASK, SEG, Op, FT_TMA_RELAX != 0>(a, Op{&tb, &tbx, a.steps});
}

template <int NT, unsigned MASK>
__global__ void __launch_bounds__(kThreads, (MASK & kTan) ? FT_MINB_RELAX : FT_MINB_RELAX_TAYLOR)
    k_taylor_relaxed(const EvalArgs a) {
  using Op = RelaxedTaylorOp<NT, MASK>;
  pdl_wait();
  stream_map<float, MASK, false, Op, FT_TMA_RELAX != 0>(a, Op{});
}

// ---------------- device restatement ----------------
template <typename T, unsigned MASK>
__global__ void __launch_bounds__(kThreads) k_mirror(const EvalArgs a, int kind, int method) {
  stream_map<T, MASK, true>(a, MirrorOp<MASK>{kind, method, a.steps, a.steps});
}

// Grid waves of resident blocks: the relaxed f32 kernels run one wave (they
// stage two row tables per block, and with PDL the next launch's staging hides
// under this one's tail: cfg1 306 vs 294 Gelem/s at 4 waves); the others use
// persistent_blocks' default (4, tail backfill).
#ifndef FT_RELAX_WAVES
#define FT_RELAX_WAVES 1
#endif
// FT_PDL=0 in the environment launches without programmatic dependent launch.
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class K>
cudaError_t go(K kernel, const EvalArgs& a, cudaStream_t s, int waves = 0, unsigned threads = kThreads) {
  unsigned blocks = 0;
  if (const cudaError_t eg = persistent_blocks(reinterpret_cast<const void*>(kernel), static_cast<int>(threads), a.n,
                                               &blocks, waves))
    return eg;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, a);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

#define FT_MASK_SWITCH(MASK_VAR, EXPR_OF_M)   \
  switch (MASK_VAR) {                         \
    case 1: { constexpr unsigned M = 1; return EXPR_OF_M; } \
    case 2: { constexpr unsigned M = 2; return EXPR_OF_M; } \
    case 3: { constexpr unsigned M = 3; return EXPR_OF_M; } \
    case 4: { constexpr unsigned M = 4; return EXPR_OF_M; } \
    case 5: { constexpr unsigned M = 5; return EXPR_OF_M; } \
    case 6: { constexpr unsigned M = 6; return EXPR_OF_M; } \
    case 7: { constexpr unsigned M = 7; return EXPR_OF_M; } \
    default: return cudaErrorInvalidValue;    \
  }

template <typename T, int SQ, bool SEG>
cudaError_t proposed_t(unsigned mask, const EvalArgs& a, cudaStream_t s) {
  FT_MASK_SWITCH(mask, (go(k_proposed<T, SQ, M, SEG>, a, s, 0, kBlockK1<T>)))
}

template <typename T, int NT>
cudaError_t taylor_t(unsigned mask, const EvalArgs& a, cudaStream_t s) {
  FT_MASK_SWITCH(mask, (go(k_taylor<T, NT, M>, a, s, 0, kBlockK2<T>)))
}

template <int SQ, bool SEG>
cudaError_t relaxed_t(unsigned mask, const EvalArgs& a, cudaStream_t s) {
  FT_MASK_SWITCH(mask, (go(k_proposed_relaxed<SQ, M, SEG>, a, s, FT_RELAX_WAVES)))
}

template <int NT>
cudaError_t taylor_relaxed_t(unsigned mask, const EvalArgs& a, cudaStream_t s) {
  FT_MASK_SWITCH(mask, (go(k_taylor_relaxed<NT, M>, a, s, FT_RELAX_WAVES)))
}

template <bool SEG>
cudaError_t relaxed_dt(unsigned mask, int sq, const EvalArgs& a, cudaStream_t s) {
  switch (sq) {
    case kExact: return relaxed_t<kExact, SEG>(mask, a, s);
    case kFisr1: return relaxed_t<kFisr1, SEG>(mask, a, s);
    case kFisr2: return relaxed_t<kFisr2, SEG>(mask, a, s);
    default: return relaxed_t<kFisrN, SEG>(mask, a, s);
  }
}

template <typename T, unsigned M>
cudaError_t mirror_go(const EvalArgs& a, int kind, int method, cudaStream_t s) {
  unsigned blocks = 0;
  if (const cudaError_t eg = persistent_blocks(reinterpret_cast<const void*>(k_mirror<T, M>), kThreads, a.n, &blocks))
    return eg;
  k_mirror<T, M><<<blocks, kThreads, 0, s>>>(a, kind, method);
  count_launch();
  return cudaGetLastError();
}

template <typename T>
cudaError_t mirror_t(unsigned mask, const EvalArgs& a, int kind, int method, cudaStream_t s) {
  FT_MASK_SWITCH(mask, (mirror_go<T, M>(a, kind, method, s)))
}

template <typename T>
cudaError_t proposed_dt(unsigned mask, int sq, bool seg, const EvalArgs& a, cudaStream_t s) {
  if (seg) {
    switch (sq) {
      case kExact: return proposed_t<T, kExact, true>(mask, a, s);
      case kFisr1: return proposed_t<T, kFisr1, true>(mask, a, s);
      case kFisr2: return proposed_t<T, kFisr2, true>(mask, a, s);
      default: return proposed_t<T, kFisrN, true>(mask, a, s);
    }
  }
  switch (sq) {
    case kExact: return proposed_t<T, kExact, false>(mask, a, s);
    case kFisr1: return proposed_t<T, kFisr1, false>(mask, a, s);
    case kFisr2: return proposed_t<T, kFisr2, false>(mask, a, s);
    default: return proposed_t<T, kFisrN, false>(mask, a, s);
  }
}

template <typename T>
cudaError_t taylor_dt(unsigned mask, int n_terms, const EvalArgs& a, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    if (f32_policy() == FT_F32_ULP2) {
      switch (n_terms) {
        case 5: return taylor_relaxed_t<5>(mask, a, s);
        case 7: return taylor_relaxed_t<7>(mask, a, s);
        case 9: return taylor_relaxed_t<9>(mask, a, s);
        default: break;  // other term counts: the truncated cosine's zero is not near pi/2
      }
    }
  }
  switch (n_terms) {
    case 5: return taylor_t<T, 5>(mask, a, s);
    case 7: return taylor_t<T, 7>(mask, a, s);
    case 9: return taylor_t<T, 9>(mask, a, s);
    default: return taylor_t<T, 0>(mask, a, s);
  }
}

// Split launches so every kernel sees < 2^31 elements (32-bit indexing); the
// offsets keep 16-byte alignment.
constexpr std::size_t kMaxLaunch = std::size_t(1) << 30;

template <class F>
cudaError_t chunked(ft_dtype dt, const EvalArgs& a, F&& launch_one) {
  if (a.n <= kMaxLaunch) return launch_one(a);
  const std::size_t es = dt == FT_F32 ? 4 : 8;
  for (std::size_t off = 0; off < a.n; off += kMaxLaunch) {
    EvalArgs b = a;
    b.n = std::min(kMaxLaunch, a.n - off);
    b.x = static_cast<const char*>(a.x) + off * es;
    for (int j = 0; j < 3; ++j)
      if (a.out[j]) b.out[j] = static_cast<char*>(a.out[j]) + off * es;
    if (a.seg_sc) b.seg_sc = a.seg_sc + off;
    if (a.seg_t) b.seg_t = a.seg_t + off;
    const cudaError_t e = launch_one(b);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// The shared-memory rows exactly as the kernels stage them, copied out
// (kind 0: bit-exact K1 rows; kind 1..7: relaxed f32 rows for that mask).
__global__ void k_dump_rows(int kind, SmemTable* out) {
  __shared__ SmemTable tb;
  __shared__ RelaxTable tr;
  switch (kind) {
    case 1: stage_table_relaxed<1, false>(&tr); break;
    case 2: stage_table_relaxed<2, false>(&tr); break;
    case 3: stage_table_relaxed<3, false>(&tr); break;
    case 4: stage_table_relaxed<4, false>(&tr); break;
    case 5: stage_table_relaxed<5, false>(&tr); break;
    case 6: stage_table_relaxed<6, false>(&tr); break;
    case 7: stage_table_relaxed<7, false>(&tr); break;
    default: stage_table(&tb); break;
  }
  __syncthreads();
  const int4* src = kind == 0 ? reinterpret_cast<const int4*>(&tb) : reinterpret_cast<const int4*>(&tr);
  const unsigned n16 = (kind == 0 ? sizeof(SmemTable) : sizeof(RelaxTable)) / 16;
  int4* dst = reinterpret_cast<int4*>(out);
  for (unsigned i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
}

}  // namespace

cudaError_t read_const_table_eval(Table* out) { return cudaMemcpyFromSymbol(out, c_table, sizeof(Table)); }

cudaError_t launch_dump_rows(int kind, void* out640, cudaStream_t s) {
  static_assert(sizeof(SmemTable) == 640, "8 rows x 80 bytes");
  k_dump_rows<<<1, 32, 0, s>>>(kind, static_cast<SmemTable*>(out640));
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_proposed(ft_dtype dt, unsigned mask, int sq, bool seg, const EvalArgs& a,
                            cudaStream_t s) {
  const bool relaxed = dt == FT_F32 && f32_policy() == FT_F32_ULP2;
  return chunked(dt, a, [&](const EvalArgs& b) {
    if (relaxed) return seg ? relaxed_dt<true>(mask, sq, b, s) : relaxed_dt<false>(mask, sq, b, s);
    return dt == FT_F32 ? proposed_dt<float>(mask, sq, seg, b, s) : proposed_dt<double>(mask, sq, seg, b, s);
  });
}

cudaError_t launch_taylor(ft_dtype dt, unsigned mask, int n_terms, const EvalArgs& a,
                          cudaStream_t s) {
  EvalArgs b = a;
  b.steps = n_terms;  // Taylor kernels read the term count from `steps`
  return chunked(dt, b, [&](const EvalArgs& c) {
    return dt == FT_F32 ? taylor_dt<float>(mask, n_terms, c, s) : taylor_dt<double>(mask, n_terms, c, s);
  });
}

cudaError_t launch_mirror(ft_dtype dt, unsigned mask, int kind, int method, int n_terms,
                          const EvalArgs& a, cudaStream_t s) {
  EvalArgs b = a;
  if (kind == 1) b.steps = n_terms;
  return chunked(dt, b, [&](const EvalArgs& c) {
    return dt == FT_F32 ? mirror_t<float>(mask, c, kind, method, s) : mirror_t<double>(mask, c, kind, method, s);
  });
}

}  // namespace ft
