// gather_tma.cu — can bulk-async copies (cp.async.bulk global -> shared, mbarrier completion)
// sustain random 256-byte-row gathers? Each lane issues one row copy per stage; a warp owns
// a ring of S stages of 32 rows; after a stage lands the warp reads it back with LDS.128
// (the consumer side of an SpMM) and re-arms it. Spin loops are bounded so a bug cannot hang
// the GPU.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int ROWB, int S, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) gather_tma(const char* __restrict__ table, const uint32_t* __restrict__ idx,
                                                         size_t n_idx, float* __restrict__ out, int* __restrict__ err) {
  extern __shared__ __align__(128) char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  char* ring = smem + (size_t)w * S * 32 * ROWB;                       // this warp's stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)WARPS * S * 32 * ROWB) + w * S;
  if (lane == 0) for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const size_t warp_g = (size_t)blockIdx.x * WARPS + w, n_warps = (size_t)gridDim.x * WARPS;
  size_t per = (n_idx + n_warps - 1) / n_warps; per = (per + 31) / 32 * 32;
  const size_t lo = warp_g * per, hi = lo + per < n_idx ? lo + per : n_idx;
  const size_t n_steps = lo < hi ? (hi - lo + 31) / 32 : 0;
  auto issue = [&](size_t step) {
    const int s = (int)(step % S);
    const size_t i = lo + step * 32 + lane;
    if (lane == 0) mbar_expect_tx(&bars[s], 32 * ROWB);   // tail steps are padded with row 0
    __syncwarp();
    const uint32_t k = i < hi ? idx[i] : 0u;
    bulk_g2s(ring + ((size_t)s * 32 + lane) * ROWB, table + (size_t)k * ROWB, ROWB, &bars[s]);
  };
  for (size_t st = 0; st < (size_t)S && st < n_steps; ++st) issue(st);
  float4 acc = make_float4(0, 0, 0, 0);
  for (size_t st = 0; st < n_steps; ++st) {
    const int s = (int)(st % S);
    const uint32_t parity = (uint32_t)((st / S) & 1);
    int spins = 0;
    while (!mbar_try_wait(&bars[s], parity)) {
      if (++spins > (1 << 22)) { if (lane == 0) atomicExch(err, 1); return; }
    }
    // consume: every lane reads ROWB/16 float4 of the 32 rows, striped (conflict-free)
    const float4* st4 = reinterpret_cast<const float4*>(ring + (size_t)s * 32 * ROWB);
#pragma unroll 4
    for (int j = 0; j < ROWB / 16; ++j) {
      const float4 v = st4[j * 32 + lane];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async writes
    __syncwarp();
    if (st + S < n_steps) issue(st + S);
  }
  if (acc.x == 123.456f) out[warp_g] = acc.x;
}

template <int ROWB, int S, int WARPS>
void run(const char* name, const char* table, const uint32_t* idx, size_t n_idx, float* out, int* err, int sms) {
  const int smem = WARPS * S * 32 * ROWB + WARPS * S * 8 + 64;
  CK(cudaFuncSetAttribute(gather_tma<ROWB, S, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int occ = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_tma<ROWB, S, WARPS>, WARPS * 32, smem));
  if (occ < 1) { printf("%s: does not fit\n", name); return; }
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  CK(cudaMemset(err, 0, 4));
  for (int w = 0; w < 2; ++w) gather_tma<ROWB, S, WARPS><<<sms * occ, WARPS * 32, smem>>>(table, idx, n_idx, out, err);
  CK(cudaEventRecord(a));
  for (int w = 0; w < 5; ++w) gather_tma<ROWB, S, WARPS><<<sms * occ, WARPS * 32, smem>>>(table, idx, n_idx, out, err);
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b)); ms /= 5; CK(cudaGetLastError());
  int h = 0; CK(cudaMemcpy(&h, err, 4, cudaMemcpyDeviceToHost));
  printf("%-22s row=%3dB stages=%d warps/CTA=%d CTAs/SM=%d in-flight/SM=%3d KB: %8.1f us %7.0f GB/s%s\n", name, ROWB, S, WARPS, occ,
         occ * WARPS * S * 32 * ROWB / 1024, ms * 1e3, (double)n_idx * ROWB / ms / 1e6, h ? "  [TIMEOUT]" : "");
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n_idx = 1u << 24, rows = 1u << 20;
  std::mt19937_64 rng(1);
  std::vector<uint32_t> h(n_idx);
  for (auto& v : h) { uint32_t k = 0; for (int b = 0; b < 20; ++b) k = (k << 1) | ((rng() >> 40) % 100 >= 76); v = k; }
  char* table; uint32_t* idx; float* out; int* err;
  CK(cudaMalloc(&table, rows * 512)); CK(cudaMemset(table, 0, rows * 512));
  CK(cudaMalloc(&idx, n_idx * 4)); CK(cudaMalloc(&out, (size_t)sms * 64 * 4 * 8)); CK(cudaMalloc(&err, 4));
  CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
  run<256, 2, 4>("rmat-skew 2^20 rows", table, idx, n_idx, out, err, sms);
  run<256, 2, 8>("rmat-skew 2^20 rows", table, idx, n_idx, out, err, sms);
  run<256, 3, 8>("rmat-skew 2^20 rows", table, idx, n_idx, out, err, sms);
  run<256, 4, 4>("rmat-skew 2^20 rows", table, idx, n_idx, out, err, sms);
  run<256, 1, 8>("rmat-skew 2^20 rows", table, idx, n_idx, out, err, sms);
  run<128, 2, 8>("rmat-skew 2^20 rows", table, idx, n_idx, out, err, sms);
  run<128, 4, 8>("rmat-skew 2^20 rows", table, idx, n_idx, out, err, sms);
  run<512, 2, 4>("rmat-skew 2^20 rows", table, idx, n_idx, out, err, sms);
  run<512, 2, 8>("rmat-skew 2^20 rows", table, idx, n_idx, out, err, sms);
  return 0;
}
