// l2_fill.cu — how many bytes per clock one SM can pull out of L2 (the ceiling of any
// gather-based SpMM once X is L2-resident), measured three ways:
//   lin   every warp streams its own 512-byte-per-instruction slice of an L2-resident buffer
//         (LDG.128, 8 loads in flight per lane, no reuse inside an SM);
//   row   every 8-lane group reads a different random 256-byte row per step (the SpMM's own
//         access shape at d = 64; uniformly random rows of an L2-resident buffer);
//   cg    as lin, but with ld.global.cg (no L1 allocation).
// Reported: bytes per SM clock per SM (clock64 deltas), and TB/s over the whole chip.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/l2_fill tools/microbench/l2_fill.cu
//   build/l2_fill [buffer MB (a power of two), default 64] [warps per SM, default 32]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CHECK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int kU = 8;

template <int MODE>
__device__ __forceinline__ float4 ld16(const float4* p) {
  float4 r;
  if (MODE == 2)
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  else
    asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// MODE 0 / 2: linear. The buffer is cut into 512-byte warp lines; warp w of the grid reads
// lines w, w + W, w + 2W, ... (W = warps in the grid), rotated by `rot` so that consecutive
// launches do not find their lines in L1.
// MODE 1: random 256-byte rows, one per 8-lane group and step (two LDG.128 per lane).
template <int MODE>
__global__ void __launch_bounds__(128) fill_kernel(const float4* __restrict__ buf, size_t n_vec, int steps,
                                                   unsigned rot, float* sink, long long* cycles) {
  const int lane = threadIdx.x & 31;
  const size_t warp = (size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const size_t n_warps = (size_t)gridDim.x * (blockDim.x >> 5);
  const long long t0 = clock64();
  float acc = 0.f;
  if (MODE == 1) {
    const size_t n_rows = n_vec / 16;  // 256-byte rows
    unsigned long long s = (warp * 4 + lane / 8 + 1) * 0x9E3779B97F4A7C15ull + rot;
    for (int it = 0; it < steps; it += kU) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU / 2; ++u) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        const size_t row = (size_t)(s >> 24) & (n_rows - 1);  // n_rows is a power of two
        const float4* p = buf + row * 16 + (lane & 7);
        v[2 * u] = ld16<MODE>(p);
        v[2 * u + 1] = ld16<MODE>(p + 8);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  } else {
    const size_t n_lines = n_vec / 32;
    size_t line = (warp + (size_t)rot * 7919) % n_lines;
    for (int it = 0; it < steps; it += kU) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        v[u] = ld16<MODE>(buf + line * 32 + lane);
        line += n_warps;
        if (line >= n_lines) line -= n_lines;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  }
  const long long t1 = clock64();
  if (acc == 12345.678f) *sink = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, const float4* buf, size_t n_vec, int sms, int warps_per_sm, float* sink,
         long long* d_cyc) {
  const int ctas = sms * warps_per_sm / 4;
  const int steps = 2048;  // LDG.128 per lane and launch
  cudaEvent_t e0, e1;
  CHECK(cudaEventCreate(&e0));
  CHECK(cudaEventCreate(&e1));
  for (int w = 0; w < 3; ++w) fill_kernel<MODE><<<ctas, 128>>>(buf, n_vec, steps, w, sink, d_cyc);
  CHECK(cudaDeviceSynchronize());
  float best = 1e30f;
  long long best_cyc = 0;
  std::vector<long long> cyc(ctas);
  for (int r = 0; r < 10; ++r) {
    CHECK(cudaEventRecord(e0));
    fill_kernel<MODE><<<ctas, 128>>>(buf, n_vec, steps, 10 + r, sink, d_cyc);
    CHECK(cudaEventRecord(e1));
    CHECK(cudaEventSynchronize(e1));
    float ms;
    CHECK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) {
      best = ms;
      CHECK(cudaMemcpy(cyc.data(), d_cyc, ctas * sizeof(long long), cudaMemcpyDeviceToHost));
      long long mx = 0;
      for (long long c : cyc) mx = c > mx ? c : mx;
      best_cyc = mx;
    }
  }
  const double bytes = (double)ctas * 128 * steps * 16;
  printf("%-4s warps/SM=%2d  %8.1f us  %6.2f TB/s  %6.1f B/clk/SM (longest CTA %lld clk => %.0f MHz)\n", name,
         warps_per_sm, best * 1e3, bytes / best / 1e9, bytes / sms / (double)best_cyc, best_cyc,
         best_cyc / (best * 1e3));
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? atoi(argv[1]) : 64;
  const int wps = argc > 2 ? atoi(argv[2]) : 32;
  cudaDeviceProp prop;
  CHECK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  const size_t n_vec = mb * 1024 * 1024 / 16;
  float4* buf;
  float* sink;
  long long* d_cyc;
  CHECK(cudaMalloc(&buf, n_vec * 16));
  CHECK(cudaMemset(buf, 0, n_vec * 16));
  CHECK(cudaMalloc(&sink, 4));
  CHECK(cudaMalloc(&d_cyc, sizeof(long long) * sms * 64));
  printf("%s, %d SMs, buffer %zu MB\n", prop.name, sms, mb);
  for (int w : {8, 16, 24, wps, 40}) {
    run<0>("lin", buf, n_vec, sms, w, sink, d_cyc);
    run<1>("row", buf, n_vec, sms, w, sink, d_cyc);
    run<2>("cg", buf, n_vec, sms, w, sink, d_cyc);
  }
  return 0;
}
