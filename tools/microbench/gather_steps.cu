// gather_steps.cu — from the pure gather to the SpMM loop, one feature at a time, to see
// which feature costs what. All variants move the same 2^24 random 256-byte rows
// (R-MAT-skewed indices over 2^20 rows) with 16 LDG.128 in flight per lane, 2 CTAs x 8 warps/SM.
//   MAP   0: 16 lanes x 1 float4 per row (U=16 positions)   1: 8 lanes x 2 float4 (U=8)
//   FMA   value stream + fmaf into 8 (or 4) accumulators
//   ROWS  a row ends every ROWLEN positions: store the accumulators (256 B), zero them
//   CHUNK the stream of each lane group restarts (pipeline drained and refilled, new
//         coordinates fetched with dependent loads) every CHUNK positions; 0 = never
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)
constexpr unsigned FULL = 0xffffffffu;

template <int MAP, bool FMA, int ROWLEN, int CHUNK, int STORE = 0>
__global__ void __launch_bounds__(256, 2) k(const float4* __restrict__ table, const uint32_t* __restrict__ idx,
                                             const float* __restrict__ vals, const uint64_t* __restrict__ coords,
                                             size_t n_idx, float4* __restrict__ y) {
  constexpr int G = MAP ? 8 : 16, NT = MAP ? 2 : 1, U = 16 / NT;
  const int lane = threadIdx.x & 31, lg = lane % G;
  const size_t group = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const size_t n_groups = ((size_t)gridDim.x * blockDim.x) / G;
  size_t per = (n_idx + n_groups - 1) / n_groups; per = (per + G - 1) / G * G;
  const size_t lo = group * per;
  const uint32_t Ltot = lo < n_idx ? (uint32_t)((lo + per < n_idx ? lo + per : n_idx) - lo) : 0;
  float4 acc[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t] = make_float4(0, 0, 0, 0);
  uint32_t left = ROWLEN ? ROWLEN : 0x7fffffffu;
  size_t row = group * (per / (ROWLEN ? ROWLEN : 1) + 1);
  const uint32_t step = CHUNK ? CHUNK : 0xffffffffu;
  for (uint32_t base = 0; __any_sync(FULL, base < Ltot); base += (CHUNK ? CHUNK : Ltot)) {
    uint32_t p0 = base;
    if (CHUNK) {  // dependent loads, like chunk coordinates -> row_ptr -> stream
      const uint64_t c = coords[(group * 7 + base / CHUNK) & 0xffff];
      const uint64_t c2 = coords[(c + lg) & 0xffff];
      p0 = base + (uint32_t)((c2 >> 60) & 0);  // value-dependent, always +0
    }
    const uint32_t L = base < Ltot ? (Ltot - base < step ? Ltot - base : step) : 0;
    const uint32_t Lmax = __reduce_max_sync(FULL, L);
    const uint32_t* ip = idx + lo + p0;
    const float* vp = vals + lo + p0;
    const float4* tb = table + lg;
    uint32_t c0 = 0, c1 = 0;
    float v0 = 0, v1 = 0;
    if ((uint32_t)lg < L) { c0 = __ldcs(ip + lg); if (FMA) v0 = __ldcs(vp + lg); }
    if ((uint32_t)(G + lg) < L) { c1 = __ldcs(ip + G + lg); if (FMA) v1 = __ldcs(vp + G + lg); }
    float4 xv[U][NT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t kq = __shfl_sync(FULL, c0, u % G, G);  // U <= G here
      if ((uint32_t)u < L) {
#pragma unroll
        for (int t = 0; t < NT; ++t) xv[u][t] = __ldg(tb + (size_t)kq * 16 + t * G);
      }
    }
#pragma unroll 1
    for (uint32_t nb = 0; nb < Lmax; nb += G) {
      uint32_t c2 = 0;
      float v2 = 0;
      if (nb + 2 * G + lg < L) { c2 = __ldcs(ip + nb + 2 * G + lg); if (FMA) v2 = __ldcs(vp + nb + 2 * G + lg); }
#pragma unroll
      for (int t = 0; t < G; ++t) {
        const int u = t % U;
        const float vq = FMA ? __shfl_sync(FULL, v0, t, G) : 1.0f;
        const uint32_t kq = (t + U < G) ? __shfl_sync(FULL, c0, t + U, G) : __shfl_sync(FULL, c1, t + U - G, G);
        if (nb + t < L) {
#pragma unroll
          for (int tt = 0; tt < NT; ++tt) {
            if (FMA) {
              acc[tt].x = __fmaf_rn(vq, xv[u][tt].x, acc[tt].x); acc[tt].y = __fmaf_rn(vq, xv[u][tt].y, acc[tt].y);
              acc[tt].z = __fmaf_rn(vq, xv[u][tt].z, acc[tt].z); acc[tt].w = __fmaf_rn(vq, xv[u][tt].w, acc[tt].w);
            } else {
              acc[tt].x += xv[u][tt].x; acc[tt].y += xv[u][tt].y; acc[tt].z += xv[u][tt].z; acc[tt].w += xv[u][tt].w;
            }
          }
        }
        if (ROWLEN && --left == 0) {
#pragma unroll
          for (int tt = 0; tt < NT; ++tt) {
            if (STORE == 0) __stcs(y + row * 16 + tt * G + lg, acc[tt]);
            else if (STORE == 1) { if (acc[tt].x == 1.2345e-30f) y[row * 16 + tt * G + lg] = acc[tt]; }
            else if (STORE == 2) __stcs(y + (row & 1023) * 16 + tt * G + lg, acc[tt]);
            else if (STORE == 3) y[row * 16 + tt * G + lg] = acc[tt];
            else if (STORE == 4) __stcg(y + row * 16 + tt * G + lg, acc[tt]);
            if (STORE != 5) acc[tt] = make_float4(0, 0, 0, 0);
            else if (acc[tt].x == 1.2345e-30f) __stcs(y + row * 16 + tt * G + lg, acc[tt]);
          }
          ++row;
          left = ROWLEN;
        }
        if (nb + t + U < L) {
#pragma unroll
          for (int tt = 0; tt < NT; ++tt) xv[u][tt] = __ldg(tb + (size_t)kq * 16 + tt * G);
        }
      }
      c0 = c1; c1 = c2; v0 = v1; v1 = v2;
    }
  }
  if (acc[0].x == 123.456f) y[group] = acc[0];
}

template <int MAP, bool FMA, int ROWLEN, int CHUNK, int STORE = 0>
void run(const char* name, const float4* table, const uint32_t* idx, const float* vals, const uint64_t* coords,
         size_t n_idx, float4* y, int sms) {
  CK(cudaFuncSetAttribute(k<MAP, FMA, ROWLEN, CHUNK, STORE>, cudaFuncAttributePreferredSharedMemoryCarveout, 25));
  cudaFuncAttributes fa; CK(cudaFuncGetAttributes(&fa, k<MAP, FMA, ROWLEN, CHUNK, STORE>));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int w = 0; w < 2; ++w) k<MAP, FMA, ROWLEN, CHUNK, STORE><<<sms * 2, 256>>>(table, idx, vals, coords, n_idx, y);
  CK(cudaEventRecord(a));
  for (int w = 0; w < 5; ++w) k<MAP, FMA, ROWLEN, CHUNK, STORE><<<sms * 2, 256>>>(table, idx, vals, coords, n_idx, y);
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b)); ms /= 5; CK(cudaGetLastError());
  printf("%-58s regs=%3d  %7.1f us  %6.0f GB/s\n", name, fa.numRegs, ms * 1e3, (double)n_idx * 256 / ms / 1e6);
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n_idx = 1u << 24, rows = 1u << 20;
  std::mt19937_64 rng(1);
  std::vector<uint32_t> h(n_idx);
  for (auto& v : h) { uint32_t kk = 0; for (int b = 0; b < 20; ++b) kk = (kk << 1) | ((rng() >> 40) % 100 >= 76); v = kk; }
  std::vector<uint64_t> hc(65536);
  for (auto& v : hc) v = rng() & 0xffff;
  float4 *table, *y; uint32_t* idx; float* vals; uint64_t* coords;
  CK(cudaMalloc(&table, rows * 256)); CK(cudaMemset(table, 0, rows * 256));
  CK(cudaMalloc(&idx, n_idx * 4)); CK(cudaMalloc(&vals, n_idx * 4)); CK(cudaMemset(vals, 0, n_idx * 4));
  CK(cudaMalloc(&coords, 65536 * 8)); CK(cudaMalloc(&y, ((size_t)1 << 21) * 256));
  CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(coords, hc.data(), 65536 * 8, cudaMemcpyHostToDevice));
  run<1, true, 0, 0>("M2 value stream and fmaf, no rows", table, idx, vals, coords, n_idx, y, sms);
  run<1, true, 24, 0, 0>("M3 row end / 24: st.cs + zero", table, idx, vals, coords, n_idx, y, sms);
  run<1, true, 24, 0, 1>("M3 row end / 24: no store (live), zero", table, idx, vals, coords, n_idx, y, sms);
  run<1, true, 24, 0, 5>("M3 row end / 24: no store, no zero (branch only)", table, idx, vals, coords, n_idx, y, sms);
  run<1, true, 24, 0, 2>("M3 row end / 24: st.cs to a hot 256 KB region", table, idx, vals, coords, n_idx, y, sms);
  run<1, true, 24, 0, 3>("M3 row end / 24: default store", table, idx, vals, coords, n_idx, y, sms);
  run<1, true, 24, 0, 4>("M3 row end / 24: st.cg", table, idx, vals, coords, n_idx, y, sms);
  run<1, true, 96, 0, 0>("M3 row end / 96: st.cs + zero", table, idx, vals, coords, n_idx, y, sms);
  run<1, true, 8, 0, 0>("M3 row end / 8: st.cs + zero", table, idx, vals, coords, n_idx, y, sms);
  return 0;
}
