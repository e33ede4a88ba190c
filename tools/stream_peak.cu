// tools/stream_peak.cu -- achievable HBM rate for this path's traffic shapes,
// with no arithmetic: x read once, each output written once, same 16-byte
// vector accesses, streaming hints, persistent grid as K1.  Compares against
// the 1:1 copy that MEASURED_PEAKS.json's hbm_gbs is quoted on.
#include <cstdio>
#include <cuda_runtime.h>

template <typename V, int NOUT>
__global__ void __launch_bounds__(256) k(const V* __restrict__ x, V* __restrict__ o0, V* __restrict__ o1,
                                         V* __restrict__ o2, size_t nv) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nv; i += stride) {
    V v = __ldcs(x + i);
    __stcs(o0 + i, v);
    if (NOUT > 1) __stcs(o1 + i, v);
    if (NOUT > 2) __stcs(o2 + i, v);
  }
}

template <int NOUT>
void run(const char* name, size_t bytes_in) {
  size_t nv = bytes_in / 16;
  double2 *x, *o[3] = {nullptr, nullptr, nullptr};
  cudaMalloc(&x, bytes_in);
  for (int j = 0; j < NOUT; ++j) cudaMalloc(&o[j], bytes_in);
  cudaMemset(x, 0, bytes_in);
  int dev = 0, sms = 0, occ = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<double2, NOUT>, 256, 0);
  dim3 grid(sms * occ);
  for (int w = 0; w < 3; ++w) k<double2, NOUT><<<grid, 256>>>(x, o[0], o[1], o[2], nv);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 50;
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) k<double2, NOUT><<<grid, 256>>>(x, o[0], o[1], o[2], nv);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double t = ms / reps * 1e-3, tot = double(bytes_in) * (1 + NOUT);
  printf("{\"shape\": \"%s\", \"bytes_per_launch\": %.0f, \"ms\": %.4f, \"gbs\": %.1f}\n", name, tot, t * 1e3,
         tot / t / 1e9);
  cudaFree(x);
  for (int j = 0; j < NOUT; ++j) cudaFree(o[j]);
}

int main() {
  run<1>("copy 1:1 (2 GiB in)", size_t(2) << 30);
  run<3>("1 read : 3 writes, cfg2 shape (2 GiB in, 6 GiB out)", size_t(2) << 30);
  run<3>("1 read : 3 writes, cfg1 shape (64 MiB in)", size_t(64) << 20);
  run<1>("1 read : 1 write, cfg3 shape (256 MiB in)", size_t(256) << 20);
  run<2>("1 read : 2 writes, cfg4 shape (1 GiB in)", size_t(1) << 30);
  return 0;
}
