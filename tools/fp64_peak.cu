// tools/fp64_peak.cu -- FP64-pipe throughput microbenchmark (the FP64 roof is
// not in MEASURED_PEAKS.json).  Each thread runs 8 independent DFMA / DMUL /
// DADD / DSETP chains; reports warp-instructions per cycle per SM and TFLOP/s
// (DFMA = 2 flops).  Timed with CUDA events after warm-up.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, int iters, double s) {
  double a[8];
  for (int j = 0; j < 8; ++j) a[j] = s * (threadIdx.x + j + 1);
  const double m = 1.0000001, c = 1e-9;
  int cnt = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) a[j] = __fma_rn(a[j], m, c);
      if (OP == 1) a[j] = __dmul_rn(a[j], m);
      if (OP == 2) a[j] = __dadd_rn(a[j], c);
      if (OP == 3) { cnt += a[j] >= c; a[j] = __longlong_as_double(__double_as_longlong(a[j]) ^ 1); }
    }
  }
  double t = cnt;
  for (int j = 0; j < 8; ++j) t += a[j];
  if (t == 12345.678) out[0] = t;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 8);
  int sms = p.multiProcessorCount, iters = 1 << 14;
  dim3 grid(sms * 8), block(256);
  const char* names[4] = {"DFMA", "DMUL", "DADD", "DSETP"};
  for (int op = 0; op < 4; ++op) {
    void (*f)(double*, int, double) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : k<3>;
    f<<<grid, block>>>(out, 64, 1.0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    f<<<grid, block>>>(out, iters, 1.0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = double(grid.x) * block.x * iters * 8;  // lane-ops
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"op\": \"%s\", \"lane_ops_per_s\": %.4e, \"tflops_if_fma\": %.2f, \"ms\": %.3f, "
           "\"lanes_per_clk_per_sm_at_max_clock\": %.1f}\n", names[op], ops / (ms * 1e-3),
           2 * ops / (ms * 1e-3) / 1e12, ms, ops / (ms * 1e-3) / (sms * clk * 1e3));
  }
  return 0;
}
