// tools/op_energy.cu -- sustained power of single-instruction-type loops, to
// rank instruction classes by energy (the sustained K1 loop is power-capped).
// Each kernel runs ~4 s; an nvidia-smi trace taken alongside (tools/op_energy.sh)
// gives watts, the printout gives lane-ops/s; energy/op = (W - idle) / rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <ctime>

template <int OP>
__global__ void __launch_bounds__(256) k(double* out, int iters, double s) {
  double a[8];
  unsigned u[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    a[j] = s * (threadIdx.x + j + 1);
    u[j] = threadIdx.x * 2654435761u + j;
  }
  const double m = 1.0000001, c = 1e-9;
  unsigned cnt = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) a[j] = __fma_rn(a[j], m, c);
      if (OP == 1) a[j] = __dmul_rn(a[j], m);
      if (OP == 2) a[j] = __dadd_rn(a[j], c);
      if (OP == 3) {  // DSETP + dependent select on the result (kept live)
        const bool p = a[j] >= c * (i & 7);
        cnt += p;
        asm volatile("" : "+d"(a[j]));
      }
      if (OP == 4) u[j] = u[j] * 0x9E3779B1u + (u[j] >> 7);  // integer IMAD/SHF
      if (OP == 5) u[j] = (u[j] ^ (u[j] >> 3)) + 0x7f4a7c15u;  // ALU LOP3/IADD3
    }
  }
  double t = cnt;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += a[j] + u[j];
  if (t == 12345.678) out[0] = t;
}

typedef void (*KF)(double*, int, double);

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const char* names[6] = {"DFMA", "DMUL", "DADD", "DSETP", "IMAD+SHF", "LOP3+IADD3"};
  KF fs[6] = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>};
  dim3 grid(sms * 8), block(256);
  for (int op = 0; op < 6; ++op) {
    fs[op]<<<grid, block>>>(out, 256, 1.0);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    long long launches = 0;
    const int iters = 1 << 14;
    cudaEventRecord(e0);
    while (ms < 4000.0f) {
      for (int r = 0; r < 4; ++r) fs[op]<<<grid, block>>>(out, iters, 1.0);
      launches += 4;
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    const double ops = double(grid.x) * block.x * iters * 8 * launches;
    printf("{\"op\": \"%s\", \"lane_ops_per_s\": %.4e, \"seconds\": %.2f}\n", names[op], ops / (ms * 1e-3), ms / 1e3);
    fflush(stdout);
    // idle gap so the power trace separates the phases
    cudaDeviceSynchronize();
    struct timespec ts = {1, 500000000};
    nanosleep(&ts, nullptr);
  }
  return 0;
}
