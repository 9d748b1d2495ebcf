// gather_bw.cu — ceiling for random X-row gathers on this GPU (development microbenchmark).
// Each group of G = rowbytes/16 lanes loads whole rows of a table at given row indices with
// LDG.128, U independent loads in flight per lane, and reduces them into registers.
//   ./gather_bw
// Prints GB/s of row bytes delivered for: row size, table size (L2-resident or not),
// index distribution (uniform / skewed like R-MAT columns), warps per SM and U.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int G, int U, int POLICY>
__global__ void gather_kernel(const float4* __restrict__ table, const uint32_t* __restrict__ idx,
                              size_t n_idx, int row_f4, float4* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int lg = lane % G;
  const size_t group = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const size_t n_groups = ((size_t)gridDim.x * blockDim.x) / G;
  const size_t per = (n_idx + n_groups - 1) / n_groups;
  size_t lo = group * per, hi = lo + per < n_idx ? lo + per : n_idx;
  float4 acc = make_float4(0, 0, 0, 0);
  for (size_t i = lo; i + U <= hi; i += U) {
    uint32_t k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) k[u] = __ldcs(idx + i + u);
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float4* p = table + (size_t)k[u] * row_f4 + lg;
      if (POLICY == 0) v[u] = __ldg(p);
      else if (POLICY == 1) v[u] = __ldcg(p);   // L2 only
      else {
        asm volatile("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(p));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
  }
  if (acc.x == 123.456f) out[group] = acc;
}

template <int G, int U, int POLICY>
float run(const float4* table, const uint32_t* idx, size_t n_idx, int row_f4, float4* out, int blocks, int threads) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int w = 0; w < 2; ++w) gather_kernel<G, U, POLICY><<<blocks, threads>>>(table, idx, n_idx, row_f4, out);
  CK(cudaEventRecord(a));
  const int it = 5;
  for (int w = 0; w < it; ++w) gather_kernel<G, U, POLICY><<<blocks, threads>>>(table, idx, n_idx, row_f4, out);
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  CK(cudaGetLastError());
  return ms / it;
}

template <int G>
void sweep(const char* name, const float4* table, const uint32_t* idx, size_t n_idx, float4* out, int sms) {
  const int row_f4 = G;
  const double bytes = (double)n_idx * G * 16;
  for (int wps : {16, 32, 64}) {
    int threads = 256, blocks = sms * wps * 32 / threads;
    float t4 = run<G, 4, 0>(table, idx, n_idx, row_f4, out, blocks, threads);
    float t8 = run<G, 8, 0>(table, idx, n_idx, row_f4, out, blocks, threads);
    float t16 = run<G, 16, 0>(table, idx, n_idx, row_f4, out, blocks, threads);
    float t8cg = run<G, 8, 1>(table, idx, n_idx, row_f4, out, blocks, threads);
    float t8el = run<G, 8, 2>(table, idx, n_idx, row_f4, out, blocks, threads);
    printf("%-34s row=%3dB warps/SM=%2d  U4 %7.0f  U8 %7.0f  U16 %7.0f  U8.cg %7.0f  U8.evict_last %7.0f GB/s\n",
           name, G * 16, wps, bytes / t4 / 1e6, bytes / t8 / 1e6, bytes / t16 / 1e6, bytes / t8cg / 1e6, bytes / t8el / 1e6);
  }
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n_idx = 1u << 24;  // 16.8M gathers, like c2's nnz
  std::mt19937_64 rng(1);
  struct Case { const char* name; size_t rows; int skew; };
  // rows of the table; skew 0 = uniform, 1 = R-MAT column distribution (a+c = 0.76 per bit)
  for (int rowb : {128, 256, 512}) {
    const int G = rowb / 16;
    Case cases[] = {{"uniform, table 32 MB (in L2)", (32u << 20) / rowb, 0},
                    {"uniform, table 96 MB", (96u << 20) / rowb, 0},
                    {"uniform, table 2^20 rows", 1u << 20, 0},
                    {"rmat-skew, table 2^20 rows", 1u << 20, 1},
                    {"sequential, table 2^20 rows", 1u << 20, 2}};
    for (auto& c : cases) {
      std::vector<uint32_t> h(n_idx);
      if (c.skew == 0) for (auto& v : h) v = (uint32_t)(rng() % c.rows);
      else if (c.skew == 2) for (size_t i = 0; i < n_idx; ++i) h[i] = (uint32_t)(i % c.rows);
      else for (auto& v : h) { uint32_t k = 0; for (int b = 0; b < 20; ++b) k = (k << 1) | ((rng() >> 40) % 100 >= 76); v = k; }
      float4* table; uint32_t* idx; float4* out;
      CK(cudaMalloc(&table, c.rows * (size_t)rowb)); CK(cudaMemset(table, 0, c.rows * (size_t)rowb));
      CK(cudaMalloc(&idx, n_idx * 4)); CK(cudaMalloc(&out, (size_t)sms * 64 * 32 * 16));
      CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
      if (rowb == 128) sweep<8>(c.name, table, idx, n_idx, out, sms);
      if (rowb == 256) sweep<16>(c.name, table, idx, n_idx, out, sms);
      if (rowb == 512) sweep<32>(c.name, table, idx, n_idx, out, sms);
      CK(cudaFree(table)); CK(cudaFree(idx)); CK(cudaFree(out));
    }
  }
  return 0;
}
