// spmx_probe.cuh — in-run measurement of the L2 -> SM ceiling (spmx_probe_l2_to_sm).
//
// The SpMM kernel gathers one X row (4*d bytes) per nonzero; once X is L2-resident the chip
// cannot deliver those rows faster than the L2 -> SM path allows, whatever the kernel does.
// bench.py reports the kernel's gather rate against that ceiling (roofline.gather), so the
// ceiling is measured on the GPU and at the clocks of the very run that reports it: every
// 8-lane group reads a different random 256-byte row of an L2-resident buffer per step (the
// SpMM's own access shape at d = 64), two LDG.128 per lane, 8 loads in flight per lane, 32 warps
// per SM. Same experiment as tools/microbench/l2_fill.cu ("row" mode).
#pragma once

namespace spmx_dev {

__global__ void __launch_bounds__(128)
l2_rows_probe_kernel(const float4* __restrict__ buf, size_t n_rows, int steps, unsigned rot,
                     float* sink) {
  constexpr int kU = 8;
  const int lane = threadIdx.x & 31;
  const size_t warp = (size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  unsigned long long s = (warp * 4 + lane / 8 + 1) * 0x9E3779B97F4A7C15ull + rot;
  float acc = 0.f;
  for (int it = 0; it < steps; it += kU) {
    float4 v[kU];
#pragma unroll
    for (int u = 0; u < kU / 2; ++u) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      const size_t row = (size_t)(s >> 24) & (n_rows - 1);  // n_rows is a power of two
      const float4* p = buf + row * 16 + (lane & 7);
      v[2 * u] = __ldg(p);
      v[2 * u + 1] = __ldg(p + 8);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 12345.678f) *sink = acc;  // keeps the loads alive
}

}  // namespace spmx_dev
