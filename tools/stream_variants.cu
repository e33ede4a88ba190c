// tools/stream_variants.cu -- how to issue a 1-read : 3-write HBM stream on
// B200 (the traffic shape of K1 on cfg2: 8 B in, 24 B out per element), with
// no arithmetic.  Variants differ only in how loads/stores are issued.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return; } } while (0)

// V0: grid-stride, one 16 B vector per thread per iteration, .cs hints
__global__ void __launch_bounds__(256) v0(const double2* __restrict__ x, double2* __restrict__ a, double2* __restrict__ b,
                                          double2* __restrict__ c, size_t nv) {
  const size_t s = size_t(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nv; i += s) {
    double2 v = __ldcs(x + i);
    __stcs(a + i, v); __stcs(b + i, v); __stcs(c + i, v);
  }
}
// V1: plain loads/stores (default caching)
__global__ void __launch_bounds__(256) v1(const double2* __restrict__ x, double2* __restrict__ a, double2* __restrict__ b,
                                          double2* __restrict__ c, size_t nv) {
  const size_t s = size_t(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nv; i += s) {
    double2 v = x[i];
    a[i] = v; b[i] = v; c[i] = v;
  }
}
// V2: unroll U=4 loads first (more bytes in flight per thread)
template <int U>
__global__ void __launch_bounds__(256) v2(const double2* __restrict__ x, double2* __restrict__ a, double2* __restrict__ b,
                                          double2* __restrict__ c, size_t nv) {
  const size_t s = size_t(gridDim.x) * blockDim.x;
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  for (; i + (U - 1) * s < nv; i += U * s) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(x + i + u * s);
#pragma unroll
    for (int u = 0; u < U; ++u) { __stcs(a + i + u * s, v[u]); __stcs(b + i + u * s, v[u]); __stcs(c + i + u * s, v[u]); }
  }
  for (; i < nv; i += s) { double2 v = __ldcs(x + i); __stcs(a + i, v); __stcs(b + i, v); __stcs(c + i, v); }
}
// V3: block-contiguous chunks of CH vectors (each block walks its own region)
template <int CH>
__global__ void __launch_bounds__(256) v3(const double2* __restrict__ x, double2* __restrict__ a, double2* __restrict__ b,
                                          double2* __restrict__ c, size_t nv) {
  const size_t nchunks = (nv + CH - 1) / CH;
  for (size_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const size_t base = ch * CH;
    for (int j = threadIdx.x; j < CH; j += blockDim.x) {
      const size_t i = base + j;
      if (i < nv) { double2 v = __ldcs(x + i); __stcs(a + i, v); __stcs(b + i, v); __stcs(c + i, v); }
    }
  }
}
// V4: stores through shared memory + TMA bulk store (cp.async.bulk.global.shared::cta)
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(ssrc));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__global__ void __launch_bounds__(256) v4(const double2* __restrict__ x, double2* __restrict__ a, double2* __restrict__ b,
                                          double2* __restrict__ c, size_t nv) {
  __shared__ __align__(128) double2 sa[256], sb[256], sc[256];  // 4 KB per output tile
  const size_t ntiles = nv / 256;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    double2 v = __ldcs(x + t * 256 + threadIdx.x);
    if (threadIdx.x == 0) bulk_wait_read0();  // previous tile's smem reads done
    __syncthreads();
    sa[threadIdx.x] = v; sb[threadIdx.x] = v; sc[threadIdx.x] = v;
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_store(a + t * 256, sa, 4096); bulk_store(b + t * 256, sb, 4096); bulk_store(c + t * 256, sc, 4096);
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// V5: st.global.L1::no_allocate with L2 evict_first via createpolicy
__global__ void __launch_bounds__(256) v5(const double2* __restrict__ x, double2* __restrict__ a, double2* __restrict__ b,
                                          double2* __restrict__ c, size_t nv) {
  const size_t s = size_t(gridDim.x) * blockDim.x;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nv; i += s) {
    double2 v = __ldcs(x + i);
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a + i), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(b + i), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(c + i), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
  }
}

// V4b: block tile, double-buffered smem, wait only for the older group
__global__ void __launch_bounds__(256) v4b(const double2* __restrict__ x, double2* __restrict__ a, double2* __restrict__ b,
                                           double2* __restrict__ c, size_t nv) {
  __shared__ __align__(128) double2 st[2][3][256];
  const size_t ntiles = nv / 256;
  int buf = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, buf ^= 1) {
    double2 v = __ldcs(x + t * 256 + threadIdx.x);
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    st[buf][0][threadIdx.x] = v; st[buf][1][threadIdx.x] = v; st[buf][2][threadIdx.x] = v;
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_store(a + t * 256, st[buf][0], 4096); bulk_store(b + t * 256, st[buf][1], 4096); bulk_store(c + t * 256, st[buf][2], 4096);
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// V6: per-warp 512 B bulk stores, double-buffered, no block barrier
__global__ void __launch_bounds__(256) v6(const double2* __restrict__ x, double2* __restrict__ a, double2* __restrict__ b,
                                          double2* __restrict__ c, size_t nv) {
  __shared__ __align__(128) double2 st[8][2][3][32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const size_t nw = nv / 32, gw = size_t(gridDim.x) * 8;
  int buf = 0;
  for (size_t t = blockIdx.x * 8 + w; t < nw; t += gw, buf ^= 1) {
    double2 v = __ldcs(x + t * 32 + l);
    if (l == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    st[w][buf][0][l] = v; st[w][buf][1][l] = v; st[w][buf][2][l] = v;
    fence_async_smem();
    __syncwarp();
    if (l == 0) {
      bulk_store(a + t * 32, st[w][buf][0], 512); bulk_store(b + t * 32, st[w][buf][1], 512); bulk_store(c + t * 32, st[w][buf][2], 512);
      bulk_commit();
    }
  }
  if (l == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef void (*KF)(const double2*, double2*, double2*, double2*, size_t);

void run(const char* name, KF f, int blocks_per_sm, double2* x, double2* o[3], size_t nv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, 256, 0);
  int bps = blocks_per_sm > 0 ? blocks_per_sm : occ;
  dim3 grid(sms * bps);
  for (int w = 0; w < 3; ++w) f<<<grid, 256>>>(x, o[0], o[1], o[2], nv);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 40;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) f<<<grid, 256>>>(x, o[0], o[1], o[2], nv);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double t = ms / reps * 1e-3, bytes = double(nv) * 16 * 4;
  printf("{\"variant\": \"%s\", \"blocks_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", name, bps, t * 1e3, bytes / t / 1e9);
}

void sustained(const char* name, KF f, int bps, double2* x, double2* o[3], size_t nv, float seconds) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  dim3 grid(sms * bps);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f<<<grid, 256>>>(x, o[0], o[1], o[2], nv);
  cudaDeviceSynchronize();
  int reps = 0;
  float ms = 0;
  cudaEventRecord(e0);
  while (ms < seconds * 1000) {
    for (int r = 0; r < 50; ++r) f<<<grid, 256>>>(x, o[0], o[1], o[2], nv);
    reps += 50;
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double t = ms / reps * 1e-3, bytes = double(nv) * 16 * 4;
  printf("{\"variant\": \"%s sustained %.1fs\", \"blocks_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", name, seconds, bps,
         t * 1e3, bytes / t / 1e9);
}

int main(int argc, char** argv) {
  if (argc > 1) {  // sustained mode: ~3 s per kernel (nvidia-smi samples power/clocks alongside)
    const size_t bytes = size_t(2) << 30, nv = bytes / 16;
    double2 *x, *o[3];
    cudaMalloc(&x, bytes);
    for (auto& p : o) cudaMalloc(&p, bytes);
    cudaMemset(x, 0, bytes);
    sustained("v0 grid-stride .cs", v0, 5, x, o, nv, 3.0f);
    sustained("v4 tma bulk store", v4, 5, x, o, nv, 3.0f);
    return 0;
  }

  const size_t bytes = size_t(2) << 30, nv = bytes / 16;
  double2 *x, *o[3];
  cudaMalloc(&x, bytes);
  for (auto& p : o) cudaMalloc(&p, bytes);
  cudaMemset(x, 0, bytes);
  for (int bps : {3, 4, 5, 6}) run("v0 grid-stride .cs", v0, bps, x, o, nv);
  for (int bps : {2, 3, 4, 5, 6, 8}) run("v4 tma bulk store", v4, bps, x, o, nv);
  for (int bps : {2, 3, 4, 5, 6, 8}) run("v4b tma bulk store 2buf", v4b, bps, x, o, nv);
  for (int bps : {2, 3, 4, 5, 6, 8}) run("v6 per-warp bulk 512B", v6, bps, x, o, nv);
  return 0;
}
