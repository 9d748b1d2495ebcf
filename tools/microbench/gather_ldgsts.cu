// gather_ldgsts.cu — the pure gather of gather_one.cu with per-thread async copies
// (cp.async.cg 16 B, global -> shared, L1 bypassed) instead of LDG.128 into registers.
// Question: with the in-flight rows parked in shared memory (up to ~200 KB/SM) instead of
// registers (131 KB/SM at 16 warps x 16 LDG.128), does the gather get past 20.5 TB/s?
// 256-byte rows, R-MAT-skewed indices over 2^20 rows, a group of 16 lanes per row.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)
constexpr int G = 16;
__device__ __forceinline__ void cp16(void* smem, const void* g) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
template <int S>
__global__ void gather_async(const float4* __restrict__ table, const uint32_t* __restrict__ idx,
                             size_t n_idx, float4* __restrict__ out) {
  extern __shared__ float4 ring[];  // [warp][S][32]
  const int lane = threadIdx.x & 31, lg = lane % G, w = threadIdx.x >> 5;
  float4* my = ring + (size_t)w * S * 32 + lane;
  const size_t group = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const size_t n_groups = ((size_t)gridDim.x * blockDim.x) / G;
  const size_t per = (n_idx + n_groups - 1) / n_groups;
  const size_t lo = group * per;
  const uint32_t L = lo < n_idx ? (uint32_t)((lo + per < n_idx ? lo + per : n_idx) - lo) : 0;
  const uint32_t Lmax = __reduce_max_sync(0xffffffffu, L);
  const uint32_t* ip = idx + lo;
  const float4* tb = table + lg;
  float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll
  for (int u = 0; u < S; ++u) {
    if ((uint32_t)u < L) cp16(my + u * 32, tb + (size_t)__ldg(ip + u) * G);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
#pragma unroll 1
  for (uint32_t nb = 0; nb < Lmax; nb += S) {
#pragma unroll
    for (int u = 0; u < S; ++u) {
      const uint32_t n = nb + u;
      asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
      if (n < L) { const float4 v = my[u * 32]; acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
      if (n + S < L) cp16(my + u * 32, tb + (size_t)__ldg(ip + n + S) * G);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  }
  if (acc.x == 123.456f) out[group] = acc;
}
template <int S>
void run(int sms, int warps_per_sm, const float4* table, const uint32_t* idx, size_t n_idx, float4* out) {
  const int wpb = 4, blocks_per_sm = warps_per_sm / wpb;
  const size_t smem = (size_t)wpb * S * 32 * 16;
  if (smem * blocks_per_sm > 220 * 1024) return;
  CK(cudaFuncSetAttribute(gather_async<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(gather_async<S>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_async<S>, wpb * 32, smem));
  if (occ < blocks_per_sm) { printf("S=%d warps/SM=%d: occupancy %d blocks only\n", S, warps_per_sm, occ); return; }
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float best = 1e9;
  for (int it = 0; it < 5; ++it) {
    CK(cudaEventRecord(a));
    gather_async<S><<<sms * blocks_per_sm, wpb * 32, smem>>>(table, idx, n_idx, out);
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  printf("cp.async S=%2d  %2d warps/SM  in flight %3d KB/SM: %.1f us  %.0f GB/s\n", S, warps_per_sm,
         warps_per_sm * S * 512 / 1024, best * 1e3, (double)n_idx * 256 / best / 1e6);
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
  for (int w : {8, 12, 16, 24, 32, 48}) {
    run<8>(sms, w, table, idx, n_idx, out);
    run<16>(sms, w, table, idx, n_idx, out);
    run<24>(sms, w, table, idx, n_idx, out);
    run<32>(sms, w, table, idx, n_idx, out);
  }
  return 0;
}
