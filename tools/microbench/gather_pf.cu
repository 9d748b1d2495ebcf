// gather_pf.cu — the rotating-pipeline gather of gather_one.cu plus software prefetch of the
// X rows PFD batches ahead (prefetch.global.L2 or prefetch.global.L1): do prefetches raise the
// bytes in flight beyond what the register file holds?
// 256-byte rows, R-MAT-skewed indices over 2^20 rows.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int MODE>
__device__ __forceinline__ void pf(const void* p) {
  if constexpr (MODE == 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  if constexpr (MODE == 2) asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
  if constexpr (MODE == 3) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

// G lanes per row (G*16 bytes = 256 -> G = 16 with one float4, or G = 8 with two float4 per lane)
template <int G, int NT, int U, int MODE, int PFD, int CTAS>
__global__ void __launch_bounds__(64, CTAS) gather_pipe(const float4* __restrict__ table, const uint32_t* __restrict__ idx,
                            size_t n_idx, size_t per_in, float4* __restrict__ out) {
  const int lane = threadIdx.x & 31, lg = lane % G;
  const size_t group = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  size_t per = per_in;
  const size_t lo = group * per;
  const uint32_t L = lo < n_idx ? (uint32_t)((lo + per < n_idx ? lo + per : n_idx) - lo) : 0;
  const uint32_t Lmax = __reduce_max_sync(0xffffffffu, L);
  const uint32_t* ip = idx + lo;
  const float4* tb = table + lg;
  constexpr int RS = G * NT;  // row stride in float4
  float4 acc = make_float4(0, 0, 0, 0);
  uint32_t c0 = 0, c1 = 0;
  if ((uint32_t)lg < L) c0 = __ldcs(ip + lg);
  if ((uint32_t)(G + lg) < L) c1 = __ldcs(ip + G + lg);
  uint32_t cp = 0; bool cpv = false;
  if (MODE) {
    // warm: prefetch rows of the first PFD batches
#pragma unroll 1
    for (int b = 0; b < PFD; ++b) {
      if ((uint32_t)(b * G + lg) < L) {
        uint32_t k = __ldcs(ip + b * G + lg);
        pf<MODE>(table + (size_t)k * RS); pf<MODE>(table + (size_t)k * RS + 8);
      }
    }
  }
  float4 xv[U][NT];
#pragma unroll
  for (int u = 0; u < U; ++u) { uint32_t k = __shfl_sync(0xffffffffu, c0, u, G); if ((uint32_t)u < L) {
#pragma unroll
    for (int t = 0; t < NT; ++t) xv[u][t] = __ldg(tb + (size_t)k * RS + t * G); } }
#pragma unroll 1
  for (uint32_t nb = 0; nb < Lmax; nb += G) {
    uint32_t c2 = 0;
    if (nb + 2 * G + lg < L) c2 = __ldcs(ip + nb + 2 * G + lg);
    if (MODE) {
      if (cpv) { pf<MODE>(table + (size_t)cp * RS); pf<MODE>(table + (size_t)cp * RS + 8); }
      cpv = nb + (PFD + 1) * G + lg < L;
      if (cpv) cp = __ldcs(ip + nb + (PFD + 1) * G + lg);
    }
#pragma unroll
    for (int t = 0; t < G; ++t) {
      const int u = t % U; const uint32_t n = nb + t;
      const uint32_t k = (t + U < G) ? __shfl_sync(0xffffffffu, c0, t + U, G) : __shfl_sync(0xffffffffu, c1, t + U - G, G);
      if (n < L) {
#pragma unroll
        for (int tt = 0; tt < NT; ++tt) { acc.x += xv[u][tt].x; acc.y += xv[u][tt].y; acc.z += xv[u][tt].z; acc.w += xv[u][tt].w; }
      }
      if (n + U < L) {
#pragma unroll
        for (int tt = 0; tt < NT; ++tt) xv[u][tt] = __ldg(tb + (size_t)k * RS + tt * G);
      }
    }
    c0 = c1; c1 = c2;
  }
  if (acc.x == 123.456f) out[group] = acc;
}

static float4* table; static uint32_t* idx; static float4* out; static int sms;
static const size_t n_idx = 1u << 24, rows = 1u << 20;

template <int G, int NT, int U, int MODE, int PFD, int CTAS>
void run(const char* name, size_t per) {
  auto k = gather_pipe<G, NT, U, MODE, PFD, CTAS>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 5));
  cudaFuncAttributes fa; CK(cudaFuncGetAttributes(&fa, k));
  int occ; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 64, 0));
  const size_t n_groups = (n_idx + per - 1) / per;
  const size_t blocks = (n_groups * G + 63) / 64;
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float best = 1e9;
  for (int it = 0; it < 5; ++it) {
    CK(cudaEventRecord(a));
    k<<<(unsigned)blocks, 64>>>(table, idx, n_idx, per, out);
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  printf("%-44s per=%5zu regs=%3d occ=%2d CTAs/SM: %7.1f us  %6.0f GB/s\n", name, per, fa.numRegs, occ, best * 1e3,
         (double)n_idx * 256 / best / 1e6);
}

int main() {
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::mt19937_64 rng(1);
  std::vector<uint32_t> h(n_idx);
  for (auto& v : h) { uint32_t k = 0; for (int b = 0; b < 20; ++b) k = (k << 1) | ((rng() >> 40) % 100 >= 76); v = k; }
  CK(cudaMalloc(&table, rows * 256)); CK(cudaMemset(table, 0, rows * 256));
  CK(cudaMalloc(&idx, n_idx * 4)); CK(cudaMalloc(&out, (size_t)(n_idx / 64 + 1024) * 16));
  CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
  for (size_t per : {(size_t)240, (size_t)960, (size_t)7680}) {
    run<8, 2, 8, 0, 0, 8>("G8 NT2 U8 16w/SM no prefetch", per);
    run<8, 2, 8, 1, 2, 8>("G8 NT2 U8 16w/SM pf.L2 +2 batches", per);
    run<8, 2, 8, 1, 4, 8>("G8 NT2 U8 16w/SM pf.L2 +4 batches", per);
    run<8, 2, 8, 1, 8, 8>("G8 NT2 U8 16w/SM pf.L2 +8 batches", per);
    run<8, 2, 8, 2, 2, 8>("G8 NT2 U8 16w/SM pf.L1 +2 batches", per);
    run<8, 2, 8, 2, 4, 8>("G8 NT2 U8 16w/SM pf.L1 +4 batches", per);
    run<8, 2, 4, 2, 2, 12>("G8 NT2 U4 24w/SM pf.L1 +2 batches", per);
    run<8, 2, 4, 2, 4, 12>("G8 NT2 U4 24w/SM pf.L1 +4 batches", per);
    run<8, 2, 4, 0, 0, 12>("G8 NT2 U4 24w/SM no prefetch", per);
    run<8, 2, 4, 1, 4, 12>("G8 NT2 U4 24w/SM pf.L2 +4 batches", per);
    run<8, 2, 2, 2, 4, 16>("G8 NT2 U2 32w/SM pf.L1 +4 batches", per);
    run<8, 2, 8, 3, 4, 8>("G8 NT2 U8 16w/SM pf.L2::evict_last +4", per);
  }
  return 0;
}
