// spmx_io_tool.cpp — exercises paper_2312_05639_b200/host/spmx_io.hpp from the command line so
// that tests/test_host_io_cpu.py can compare its outputs byte for byte with files written by the
// unmodified reference (tests/golden/io/). Host only: no CUDA.
//   spmx_io_tool random-csr <rows> <avg> <skew> <seed> <out.jspm>
//   spmx_io_tool random-dense <rows> <cols> <seed> <out.f32>
//   spmx_io_tool jspm-to-mtx <in.jspm> <out.mtx>
//   spmx_io_tool mtx-to-jspm <in.mtx> <out.jspm>
//   spmx_io_tool copy-jspm <in.jspm> <out.jspm>
//   spmx_io_tool validate <in.jspm|in.mtx>
//   spmx_io_tool config <c1..c5> <scale|0> <rows|0> <out.jspm> <out_x.f32>   (host/spmx_workloads.hpp)
#include <cstdio>
#include <cstring>
#include <string>

#include "../../paper_2312_05639_b200/host/spmx_io.hpp"
#include "../../paper_2312_05639_b200/host/spmx_workloads.hpp"

static bool ends_with(const std::string& s, const char* suf) {
  const size_t n = std::strlen(suf);
  return s.size() >= n && s.compare(s.size() - n, n, suf) == 0;
}

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "random-csr" && argc == 7) {
      spmx::save_csr_cache(spmx::random_csr(std::atoll(argv[2]), std::atof(argv[3]), std::atof(argv[4]),
                                            std::strtoull(argv[5], nullptr, 10)), argv[6]);
    } else if (cmd == "random-dense" && argc == 6) {
      spmx::DenseMatrix x = spmx::random_dense(std::atoll(argv[2]), std::atoll(argv[3]),
                                               std::strtoull(argv[4], nullptr, 10));
      FILE* f = std::fopen(argv[5], "wb");
      if (!f) throw std::runtime_error("cannot open for write");
      std::fwrite(x.data.data(), 4, x.data.size(), f);
      std::fclose(f);
    } else if (cmd == "jspm-to-mtx" && argc == 4) {
      spmx::write_matrix_market(spmx::load_csr_cache(argv[2]), argv[3]);
    } else if (cmd == "mtx-to-jspm" && argc == 4) {
      spmx::save_csr_cache(spmx::load_matrix_market(argv[2]), argv[3]);
    } else if (cmd == "copy-jspm" && argc == 4) {
      spmx::save_csr_cache(spmx::load_csr_cache(argv[2]), argv[3]);
    } else if (cmd == "config" && argc == 7) {
      spmx::workloads::Config c = spmx::workloads::make_config(argv[2], std::atoi(argv[3]), std::atoll(argv[4]));
      spmx::save_csr_cache(c.a, argv[5]);
      FILE* f = std::fopen(argv[6], "wb");
      if (!f) throw std::runtime_error("cannot open for write");
      std::fwrite(c.x.data.data(), 4, c.x.data.size(), f);
      std::fclose(f);
    } else if (cmd == "validate" && argc == 3) {
      const spmx::CsrMatrix a = ends_with(argv[2], ".jspm") ? spmx::load_csr_cache(argv[2])
                                                            : spmx::load_matrix_market(argv[2]);
      const auto bad = spmx::validate_csr(a);
      std::printf("m=%lld n=%lld nnz=%lld violations=%zu\n", (long long)a.m, (long long)a.n,
                  (long long)a.nnz, bad.size());
    } else {
      std::fprintf(stderr, "usage: see the header of tests/host/spmx_io_tool.cpp\n");
      return 1;
    }
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "invalid_argument: %s\n", e.what());
    return 3;
  } catch (const std::runtime_error& e) {
    std::fprintf(stderr, "runtime_error: %s\n", e.what());
    return 2;
  }
  return 0;
}
