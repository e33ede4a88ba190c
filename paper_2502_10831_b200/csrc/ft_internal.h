// ft_internal.h -- launcher interface shared by the CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "fasttrig_b200.h"
#include "ft_core.cuh"

namespace ft {

struct EvalArgs {
  const void* x;
  void* out[3];  // sin, cos, tan
  std::uint8_t* seg_sc;
  std::uint8_t* seg_t;
  std::size_t n;
  int steps;
  int vec_ok;  // all pointers aligned for 128-bit access
};

struct CheckArgs {
  const void* x;
  const void* got[3];
  const void* ref[3];
  const std::uint8_t* seg_sc;
  const std::uint8_t* seg_t;
  std::size_t n;
  unsigned mask;
  int kind;  // 0 proposed, 1 taylor
  int method, steps, n_terms;
  std::uint64_t ulp_tol;
  ft_stats* stats;
};

// Launchers: return cudaError_t of the launch.  `kind`: 0 proposed, 1 taylor.
cudaError_t launch_proposed(ft_dtype dt, unsigned mask, int sq, bool seg, const EvalArgs& a,
                            cudaStream_t s);
cudaError_t launch_taylor(ft_dtype dt, unsigned mask, int n_terms, const EvalArgs& a,
                          cudaStream_t s);
cudaError_t launch_mirror(ft_dtype dt, unsigned mask, int kind, int method, int n_terms,
                          const EvalArgs& a, cudaStream_t s);
cudaError_t launch_check(ft_dtype dt, const CheckArgs& a, cudaStream_t s);
cudaError_t launch_gen(ft_dtype dt, int dist, double lo, double hi, std::uint64_t seed,
                       std::uint64_t offset, std::size_t n, void* x, cudaStream_t s);
cudaError_t launch_fill(void* buf, std::size_t bytes, unsigned v, cudaStream_t s);

// Grid sizing: waves x (#SM x resident blocks of `fn` at `threads` per block),
// capped by the work available (work_items / threads blocks).  `waves` > 0
// overrides the default (4).  Fails (and sets no grid) if the device or
// occupancy queries fail.
cudaError_t persistent_blocks(const void* fn, int threads, std::size_t work_items, unsigned* blocks,
                              int waves = 0);
// Read-back of the device-resident tables (ft_device_const_table /
// ft_device_rows): the __constant__ segment table of each translation unit
// that evaluates the path, and the shared-memory rows K1 stages.
cudaError_t read_const_table_eval(Table* out);
cudaError_t read_const_table_check(Table* out);
cudaError_t read_const_table_gen(Table* out);
cudaError_t launch_dump_rows(int kind, void* out640, cudaStream_t s);

// Process-wide f32 policy (ft_set_f32_policy): FT_F32_ULP2 or FT_F32_BITWISE.
int f32_policy();
void count_launch();

}  // namespace ft
