// Is CUDA's sincos(x) bitwise sin(x), cos(x)?  (K3 uses libm as the error
// reference; this decides whether it may share the argument reduction.)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sincos_identity tools/sincos_identity.cu
#include <cstdio>
#include <cstdint>
__device__ unsigned long long g_bad;
__device__ inline unsigned long long mix(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k(unsigned long long n, int mode) {
  unsigned long long bad = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long r = mix(i * 0x9E3779B97F4A7C15ull + mode);
    double x;
    if (mode == 0) x = __longlong_as_double(r);                               // every bit pattern
    else if (mode == 1) x = ((double)(r >> 11) * 0x1p-53 - 0.5) * 6283.185307179586;  // +-1000 pi
    else if (mode == 2) x = (double)__uint_as_float((unsigned)r);             // float inputs
    else x = ((double)(r >> 11) * 0x1p-53) * 6.283185307179586;               // [0, 2pi)
    double s, c;
    sincos(x, &s, &c);
    const double s1 = sin(x), c1 = cos(x);
    bad += (__double_as_longlong(s) != __double_as_longlong(s1)) + (__double_as_longlong(c) != __double_as_longlong(c1));
  }
  if (bad) atomicAdd(&g_bad, bad);
}
int main() {
  for (int mode = 0; mode < 4; ++mode) {
    unsigned long long zero = 0, bad = 0;
    cudaMemcpyToSymbol(g_bad, &zero, sizeof zero);
    k<<<148 * 8, 256>>>(1ull << 30, mode);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&bad, g_bad, sizeof bad);
    printf("{\"mode\": %d, \"n\": %llu, \"sincos_vs_sin_cos_bit_mismatches\": %llu}\n", mode, 1ull << 30, bad);
  }
  return 0;
}
