// gather_one.cu — one configuration of the rotating-pipeline gather (for ncu):
// 256-byte rows, R-MAT-skewed indices over 2^20 rows, U=16, 16 resident warps/SM.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)
template <int G, int U>
__global__ void __launch_bounds__(256, 2) gather_pipe(const float4* __restrict__ table, const uint32_t* __restrict__ idx,
                            size_t n_idx, float4* __restrict__ out) {
  const int lane = threadIdx.x & 31, lg = lane % G;
  const size_t group = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const size_t n_groups = ((size_t)gridDim.x * blockDim.x) / G;
  size_t per = (n_idx + n_groups - 1) / n_groups; per = (per + G - 1) / G * G;
  const size_t lo = group * per;
  const uint32_t L = lo < n_idx ? (uint32_t)((lo + per < n_idx ? lo + per : n_idx) - lo) : 0;
  const uint32_t Lmax = __reduce_max_sync(0xffffffffu, L);
  const uint32_t* ip = idx + lo;
  const float4* tb = table + lg;
  float4 acc = make_float4(0, 0, 0, 0);
  uint32_t c0 = 0, c1 = 0;
  if ((uint32_t)lg < L) c0 = __ldcs(ip + lg);
  if ((uint32_t)(G + lg) < L) c1 = __ldcs(ip + G + lg);
  float4 xv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { uint32_t k = __shfl_sync(0xffffffffu, c0, u, G); if ((uint32_t)u < L) xv[u] = __ldg(tb + (size_t)k * G); }
#pragma unroll 1
  for (uint32_t nb = 0; nb < Lmax; nb += G) {
    uint32_t c2 = 0;
    if (nb + 2 * G + lg < L) c2 = __ldcs(ip + nb + 2 * G + lg);
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const int u = t % U; const uint32_t n = nb + t;
      const uint32_t k = (t + U < G) ? __shfl_sync(0xffffffffu, c0, t + U, G) : __shfl_sync(0xffffffffu, c1, t + U - G, G);
      if (n < L) { acc.x += xv[u].x; acc.y += xv[u].y; acc.z += xv[u].z; acc.w += xv[u].w; }
      if (n + U < L) xv[u] = __ldg(tb + (size_t)k * G);
    }
    c0 = c1; c1 = c2;
  }
  if (acc.x == 123.456f) out[group] = acc;
}
int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n_idx = 1u << 24, rows = 1u << 20;
  std::mt19937_64 rng(1);
  std::vector<uint32_t> h(n_idx);
  for (auto& v : h) { uint32_t k = 0; for (int b = 0; b < 20; ++b) k = (k << 1) | ((rng() >> 40) % 100 >= 76); v = k; }
  float4* table; uint32_t* idx; float4* out;
  CK(cudaMalloc(&table, rows * 256)); CK(cudaMemset(table, 0, rows * 256));
  CK(cudaMalloc(&idx, n_idx * 4)); CK(cudaMalloc(&out, (size_t)sms * 64 * 32 * 16));
  CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(gather_pipe<16, 16>, cudaFuncAttributePreferredSharedMemoryCarveout, 25));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int it = 0; it < 6; ++it) {
    CK(cudaEventRecord(a));
    gather_pipe<16, 16><<<sms * 2, 256>>>(table, idx, n_idx, out);
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    printf("pure gather U=16, 16 warps/SM: %.1f us  %.0f GB/s\n", ms * 1e3, (double)n_idx * 256 / ms / 1e6);
  }
  return 0;
}
