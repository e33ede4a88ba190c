// tools/latency.cu -- dependent-issue latency (cycles) of the instruction
// classes on K1's critical path, one warp, clock64 around 1024-long chains.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, double s) {
  double a = s + threadIdx.x;
  unsigned u = threadIdx.x;
  float f = static_cast<float>(s);
  __shared__ double sm[64];
  sm[threadIdx.x] = a;
  __syncwarp();
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (OP == 0) a = __dmul_rn(a, 1.0000001);
    if (OP == 1) a = __dadd_rn(a, 1e-9);
    if (OP == 2) a = __fma_rn(a, 1.0000001, 1e-9);
    if (OP == 3) a = floor(a) + 0.5;                       // FRND + DADD
    if (OP == 4) { a = (a >= 1.0) ? a * 0.5 : a + 1.0; }   // DSETP -> select -> DMUL/DADD
    if (OP == 5) { f = static_cast<float>(a); a = static_cast<double>(f) + 1e-9; }  // F2F x2 + DADD
    if (OP == 6) { a = sm[(__double2loint(a) & 31)]; }      // LDS (dependent address)
    if (OP == 7) { u = u * 2654435761u + 1u; }              // IMAD
  }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[OP] = t1 - t0;
  out[threadIdx.x] = a + u + f;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 * sizeof(double));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  const char* names[8] = {"DMUL", "DADD", "DFMA", "FRND+DADD", "DSETP+SEL+DMUL/DADD", "F2F.F32.F64+F2F.F64.F32+DADD", "LDS(dep addr)", "IMAD"};
  void (*fs[8])(double*, long long*, double) = {chain<0>, chain<1>, chain<2>, chain<3>, chain<4>, chain<5>, chain<6>, chain<7>};
  for (int k = 0; k < 8; ++k) {
    fs[k]<<<1, 32>>>(out, cyc, 1.0);
    fs[k]<<<1, 32>>>(out, cyc, 1.0);
    cudaDeviceSynchronize();
    printf("{\"chain\": \"%s\", \"cycles_per_step\": %.1f}\n", names[k], cyc[k] / 1024.0);
  }
  return 0;
}
