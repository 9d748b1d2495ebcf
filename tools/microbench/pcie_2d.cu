// pcie_2d.cu — bandwidth of strided (2-D) host<->device copies of column slabs of a row-major
// N x 64 fp32 matrix (pitch 256 B), against the contiguous copy. Decides whether the host
// pipeline can move X and Y as column slabs to overlap the X upload with the Y download.
//   nvcc -O3 -arch=sm_100a -o pcie_2d pcie_2d.cu && ./pcie_2d
#include <cuda_runtime.h>
#include <cstdio>
#include <chrono>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
  const size_t rows = 1 << 20, pitch = 256;
  char *h, *d;
  CK(cudaMallocHost(&h, rows * pitch));
  CK(cudaMalloc(&d, rows * pitch));
  cudaStream_t s, s2; CK(cudaStreamCreate(&s)); CK(cudaStreamCreate(&s2));
  for (int width : {256, 128, 64, 32}) {
    for (int dir = 0; dir < 3; ++dir) {
      CK(cudaDeviceSynchronize());
      auto t0 = std::chrono::steady_clock::now();
      const int reps = 4;
      for (int r = 0; r < reps; ++r) {
        for (int off = 0; off < 256; off += width) {
          if (dir == 0 || dir == 2) CK(cudaMemcpy2DAsync(d + off, pitch, h + off, pitch, width, rows, cudaMemcpyHostToDevice, s));
          if (dir == 1 || dir == 2) CK(cudaMemcpy2DAsync(h + off, pitch, d + off, pitch, width, rows, cudaMemcpyDeviceToHost, dir == 2 ? s2 : s));
        }
      }
      CK(cudaDeviceSynchronize());
      double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
      printf("width %3d B  %s  %.1f GB/s per direction\n", width, dir == 0 ? "h2d" : dir == 1 ? "d2h" : "both", rows * pitch / dt / 1e9);
    }
  }
  return 0;
}
