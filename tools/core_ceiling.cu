// SM-only ceiling of the relaxed f32 cores: the same per-element code as the
// production kernels (relaxed_proposed_core + the rare exact path, shared-memory
// rows, 4 blocks/SM of 256 threads, 4 elements per thread in a row) evaluated
// `reps` times on register-resident inputs that step by one ulp per pass -- no
// global loads or stores inside the loop.  Gelem/s here is what the SMs alone
// sustain for this instruction mix; compare with the kernels' measured rates
// and with the HBM roof (817 Gelem/s tan-only, 409 fused).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -fmad=false \
//        -Iinclude -Ipaper_2502_10831_b200/csrc -o tools/core_ceiling tools/core_ceiling.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ft_core.cuh"

using namespace ft;

template <unsigned MASK>
__global__ void __launch_bounds__(256, 4) k_core(const float* __restrict__ x, unsigned* __restrict__ out, int reps) {
  __shared__ RelaxTable tb;
  __shared__ SmemTable tbx;
  stage_table_relaxed<MASK, false>(&tb);
  stage_table(&tbx);
  __syncthreads();
  const unsigned gid = blockIdx.x * blockDim.x + threadIdx.x;
  const float4 v = reinterpret_cast<const float4*>(x)[gid];
  float xs[4] = {v.x, v.y, v.z, v.w};
  // tan-only: each slot stays within +-2e-3 of its own pole; otherwise [0, 2 pi)
  const float width = MASK == kTan ? 4e-3f : 6.2831853f;
  const float step = MASK == kTan ? 7.3e-4f : 1.2345f;
  float hi[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) hi[j] = MASK == kTan ? xs[j] + 2e-3f : 6.2831853f;
  unsigned acc = 0;
  Out3f prev[4] = {};
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // consume the result this slot produced one pass ago (the production
      // kernels' results wait in registers for the vector's store, so a
      // result's conversion latency overlaps the next element's reduction)
      if (MASK & kSin) acc ^= __float_as_uint(prev[j].s);
      if (MASK & kCos) acc ^= __float_as_uint(prev[j].c);
      if (MASK & kTan) acc ^= __float_as_uint(prev[j].t);
      bool ok;
      Out3f o = relaxed_proposed_core<kFisr1, MASK, false>(xs[j], tb, 1, &ok);
      if (!ok) o = relaxed_slow<kFisr1, MASK, false>(xs[j], &tbx, 1);
      prev[j] = o;
      // next input: walk through the window [lo, lo + width) in steps that are
      // incommensurate with it, so the lanes that need the exact path change
      // from pass to pass as they do along a real array (3 extra instructions)
      float xn = xs[j] + step;
      if (xn >= hi[j]) xn -= width;
      xs[j] = xn;
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) acc ^= __float_as_uint(prev[j].s) ^ __float_as_uint(prev[j].c) ^ __float_as_uint(prev[j].t);
  out[gid] = acc;
}

template <unsigned MASK>
double run(const std::vector<float>& h, int reps, int blocks) {
  float* dx;
  unsigned* dout;
  cudaMalloc(&dx, h.size() * sizeof(float));
  cudaMalloc(&dout, h.size() / 4 * sizeof(unsigned));
  cudaMemcpy(dx, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice);
  k_core<MASK><<<blocks, 256>>>(dx, dout, 10);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int t = 0; t < 3; ++t) {
    cudaEventRecord(e0);
    k_core<MASK><<<blocks, 256>>>(dx, dout, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaFree(dx);
  cudaFree(dout);
  return double(h.size()) * reps / (best * 1e-3) / 1e9;
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? std::atoi(argv[1]) : 400;  // ~20 ms: inside the pre-limiter window
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4;
  const size_t n = size_t(blocks) * 256 * 4;
  std::vector<float> tanx(n), uni(n);
  unsigned long long s = 2024873;
  auto u01 = [&] {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return double(s >> 11) * 0x1p-53;
  };
  for (size_t i = 0; i < n; ++i) {
    const int k = int(u01() * 2001) - 1000;
    // ~N(0, 1e-3) by the sum of 12 uniforms, clipped like configs[2]
    double g = -6.0;
    for (int q = 0; q < 12; ++q) g += u01();
    double d = g * 1e-3;
    d = d > 0.05 ? 0.05 : d < -0.05 ? -0.05 : d;
    tanx[i] = float((2 * k + 1) * 1.5707963267948966 + d * 0.5);
    uni[i] = float(u01() * 6.283185307179586);
  }
  printf("{\"kernel\": \"tan-only core, configs[2]-like inputs\", \"reps\": %d, \"gelem_s\": %.1f}\n", reps, run<kTan>(tanx, reps, blocks));
  printf("{\"kernel\": \"fused S/C/T core, U[0,2pi)\", \"reps\": %d, \"gelem_s\": %.1f}\n", reps, run<7u>(uni, reps, blocks));
  printf("{\"kernel\": \"sin+cos core, U[0,2pi)\", \"reps\": %d, \"gelem_s\": %.1f}\n", reps, run<3u>(uni, reps, blocks));
  return 0;
}
