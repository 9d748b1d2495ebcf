// gather_bw2.cu — which factor limits random-row gathers: resident warps, loads in flight
// per lane (batch vs rotating pipeline), or the index stream? True residency is enforced
// with __launch_bounds__ + dynamic smem padding and reported.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// rotating pipeline: U loads in flight per lane at all times; indices fetched a batch of G ahead
template <int G, int U>
__global__ void __launch_bounds__(256) gather_pipe(const float4* __restrict__ table, const uint32_t* __restrict__ idx,
                            size_t n_idx, float4* __restrict__ out) {
  extern __shared__ char pad[];
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
  for (int u = 0; u < U; ++u) {
    uint32_t k = __shfl_sync(0xffffffffu, c0, u, G);
    if ((uint32_t)u < L) xv[u] = __ldg(tb + (size_t)k * G);
  }
#pragma unroll 1
  for (uint32_t nb = 0; nb < Lmax; nb += G) {
    uint32_t c2 = 0;
    if (nb + 2 * G + lg < L) c2 = __ldcs(ip + nb + 2 * G + lg);
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const int u = t % U;
      const uint32_t n = nb + t;
      const uint32_t k = (t + U < G) ? __shfl_sync(0xffffffffu, c0, t + U, G) : __shfl_sync(0xffffffffu, c1, t + U - G, G);
      if (n < L) { acc.x += xv[u].x; acc.y += xv[u].y; acc.z += xv[u].z; acc.w += xv[u].w; }
      if (n + U < L) xv[u] = __ldg(tb + (size_t)k * G);
    }
    c0 = c1; c1 = c2;
  }
  if (acc.x == 123.456f) out[group] = acc;
}

template <int G, int U>
void run(const char* name, const float4* table, const uint32_t* idx, size_t n_idx, float4* out, int sms, int ctas_per_sm) {
  // force residency: pad dynamic smem so exactly ctas_per_sm CTAs fit (227 KB usable)
  int smem = (220 * 1024) / ctas_per_sm - 1024;
  CK(cudaFuncSetAttribute(gather_pipe<G, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int occ = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_pipe<G, U>, 256, smem));
  int blocks = sms * occ;
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int w = 0; w < 2; ++w) gather_pipe<G, U><<<blocks, 256, smem>>>(table, idx, n_idx, out);
  CK(cudaEventRecord(a));
  for (int w = 0; w < 5; ++w) gather_pipe<G, U><<<blocks, 256, smem>>>(table, idx, n_idx, out);
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b)); ms /= 5; CK(cudaGetLastError());
  printf("%-28s row=%3dB U=%2d resident warps/SM=%2d (smem pad %3d KB): %7.0f GB/s\n", name, G * 16, U, occ * 8, smem / 1024,
         (double)n_idx * G * 16 / ms / 1e6);
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n_idx = 1u << 24;
  std::mt19937_64 rng(1);
  const size_t rows = 1u << 20;
  for (int skew = 0; skew < 2; ++skew) {
    std::vector<uint32_t> h(n_idx);
    if (skew) for (auto& v : h) { uint32_t k = 0; for (int b = 0; b < 20; ++b) k = (k << 1) | ((rng() >> 40) % 100 >= 76); v = k; }
    else for (auto& v : h) v = (uint32_t)(rng() % (rows / 8));   // 32 MB at 256 B rows: L2-resident uniform
    float4* table; uint32_t* idx; float4* out;
    CK(cudaMalloc(&table, rows * 512)); CK(cudaMemset(table, 0, rows * 512));
    CK(cudaMalloc(&idx, n_idx * 4)); CK(cudaMalloc(&out, (size_t)sms * 64 * 32 * 16));
    CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
    const char* nm = skew ? "rmat-skew 2^20 rows" : "uniform 32MB (L2)";
    for (int ctas : {1, 2, 3, 4, 6, 8}) {
      run<16, 4>(nm, table, idx, n_idx, out, sms, ctas);
      run<16, 8>(nm, table, idx, n_idx, out, sms, ctas);
      run<16, 16>(nm, table, idx, n_idx, out, sms, ctas);
    }
    CK(cudaFree(table)); CK(cudaFree(idx)); CK(cudaFree(out));
  }
  return 0;
}
