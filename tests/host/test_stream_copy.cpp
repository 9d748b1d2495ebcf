// CPU test of spmx_stage::stream_copy (csrc/spmx_stage.cuh): the non-temporal copy used to stage
// pageable host arrays must equal memcpy for every size, source and destination alignment, and
// must not write outside [dst, dst + bytes).
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2312_05639_b200/csrc/spmx_stage.cuh"

int main() {
  std::mt19937_64 rng(2312);
  std::vector<unsigned char> src(1 << 16), dst(1 << 16), want(1 << 16);
  for (auto& b : src) b = (unsigned char)rng();
  const size_t sizes[] = {0, 1, 15, 16, 17, 63, 64, 65, 255, 256, 257, 271, 272, 1000, 4096, 4097, 30000};
  long cases = 0;
  for (size_t n : sizes)
    for (size_t so = 0; so < 19; ++so)
      for (size_t dof = 0; dof < 19; ++dof) {
        std::memset(dst.data(), 0xA5, dst.size());
        std::memset(want.data(), 0xA5, want.size());
        std::memcpy(want.data() + 64 + dof, src.data() + so, n);
        spmx_stage::stream_copy(dst.data() + 64 + dof, src.data() + so, n);
        if (std::memcmp(dst.data(), want.data(), dst.size()) != 0) {
          std::printf("FAIL n=%zu src+%zu dst+%zu\n", n, so, dof);
          return 1;
        }
        ++cases;
      }
  std::printf("stream_copy ok: %ld cases, streaming=%d\n", cases, SPMX_STAGE_STREAMING);
  return 0;
}
