// spmx_io.hpp — the data formats and generators either side of the SpMM path
// (SURVEY.md §8 f3): the reference's `.jspm` binary cache, Matrix Market coordinate files,
// and its two deterministic generators, with the reference's names and error behaviour
// (include/spmx/csr.hpp:22-34, include/spmx/mmio.hpp, include/spmx/dense.hpp:23-25) so that
// matrices move between the reference and this library unchanged. Pure host code, no CUDA;
// include after (or without) spmx_b200.hpp.
//
// Byte-level parity with the reference is pinned by tests/test_host_io_cpu.py against files
// the unmodified reference wrote (tests/golden/io/).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "spmx_types.hpp"

namespace spmx {

// ---- validate_csr (csr.hpp:22-24, csr.cpp:18-42): one message per violated invariant ------
inline std::vector<std::string> validate_csr(const CsrMatrix& a) {
  std::vector<std::string> bad;
  if (a.m < 0 || a.n < 0 || a.nnz < 0) bad.emplace_back("negative dimension");
  if (a.row_ptr.size() != size_t(a.m) + 1) {
    bad.emplace_back("row_ptr length " + std::to_string(a.row_ptr.size()) + " != m+1");
    return bad;
  }
  if (a.row_ptr.front() != 0) bad.emplace_back("row_ptr[0] != 0");
  if (a.row_ptr.back() != uint64_t(a.nnz))
    bad.emplace_back("row_ptr[m] = " + std::to_string(a.row_ptr.back()) + " != nnz");
  const auto dip = std::adjacent_find(a.row_ptr.begin(), a.row_ptr.end(), std::greater<uint64_t>());
  if (dip != a.row_ptr.end())
    bad.emplace_back("row_ptr not nondecreasing at " + std::to_string(dip - a.row_ptr.begin() + 1));
  if (a.col_indices.size() != size_t(a.nnz)) bad.emplace_back("col_indices length != nnz");
  if (a.vals.size() != size_t(a.nnz)) bad.emplace_back("vals length != nnz");
  const auto oob = std::find_if(a.col_indices.begin(), a.col_indices.end(),
                                [&](uint32_t c) { return int64_t(c) >= a.n; });
  if (oob != a.col_indices.end())
    bad.emplace_back("column index out of range at " + std::to_string(oob - a.col_indices.begin()));
  return bad;
}

namespace io_detail {

struct File {
  FILE* f;
  std::string path;
  File(const std::string& p, const char* mode, const char* fail) : f(std::fopen(p.c_str(), mode)), path(p) {
    if (!f) throw std::runtime_error(std::string(fail) + p);
  }
  ~File() { if (f) std::fclose(f); }
  void put(const void* src, size_t bytes) {
    if (bytes && std::fwrite(src, 1, bytes, f) != bytes) throw std::runtime_error("short write: " + path);
  }
  void get(void* dst, size_t bytes) {
    if (bytes && std::fread(dst, 1, bytes, f) != bytes)
      throw std::runtime_error("truncated cache file: " + path);
  }
};

}  // namespace io_detail

// ---- `.jspm` cache (csr.hpp:26-29): "JSPM", u32 version = 1, u64 m, n, nnz, then row_ptr (u64),
//      col_indices (u32), vals (f32), little-endian ----------------------------------------------
inline void save_csr_cache(const CsrMatrix& a, const std::string& path) {
  io_detail::File out(path, "wb", "cannot open for write: ");
  const uint32_t version = 1;
  const uint64_t dims[3] = {uint64_t(a.m), uint64_t(a.n), uint64_t(a.nnz)};
  out.put("JSPM", 4);
  out.put(&version, sizeof version);
  out.put(dims, sizeof dims);
  out.put(a.row_ptr.data(), a.row_ptr.size() * sizeof(uint64_t));
  out.put(a.col_indices.data(), a.col_indices.size() * sizeof(uint32_t));
  out.put(a.vals.data(), a.vals.size() * sizeof(float));
}

inline CsrMatrix load_csr_cache(const std::string& path) {
  io_detail::File in(path, "rb", "cannot open: ");
  char magic[4];
  uint32_t version = 0;
  uint64_t dims[3];
  in.get(magic, 4);
  if (std::memcmp(magic, "JSPM", 4) != 0) throw std::runtime_error("not a JSPM cache file: " + path);
  in.get(&version, sizeof version);
  if (version != 1) throw std::runtime_error("unsupported cache version " + std::to_string(version));
  in.get(dims, sizeof dims);
  CsrMatrix a;
  a.m = int64_t(dims[0]);
  a.n = int64_t(dims[1]);
  a.nnz = int64_t(dims[2]);
  a.row_ptr.resize(size_t(a.m) + 1);
  a.col_indices.resize(size_t(a.nnz));
  a.vals.resize(size_t(a.nnz));
  in.get(a.row_ptr.data(), a.row_ptr.size() * sizeof(uint64_t));
  in.get(a.col_indices.data(), a.col_indices.size() * sizeof(uint32_t));
  in.get(a.vals.data(), a.vals.size() * sizeof(float));
  const auto bad = validate_csr(a);
  if (!bad.empty()) throw std::runtime_error("invalid CSR in cache " + path + ": " + bad.front());
  return a;
}

// ---- Matrix Market coordinate files (mmio.hpp:11-19) ---------------------------------------------
// real / integer / pattern, general / symmetric -> canonical CSR: sorted by (row, column),
// symmetric entries mirrored, duplicates summed in file order, pattern values 1. Malformed input
// raises std::runtime_error("<path>:<line>: <what>"); the array (dense) class is rejected.
inline CsrMatrix load_matrix_market(const std::string& path) {
  io_detail::File in(path, "r", "cannot open: ");
  long lineno = 0;
  auto fail = [&](const std::string& what) -> void {
    throw std::runtime_error(path + ":" + std::to_string(lineno) + ": " + what);
  };
  std::string line;
  auto next_line = [&]() -> bool {
    line.clear();
    int ch;
    bool any = false;
    while ((ch = std::fgetc(in.f)) != EOF) {
      any = true;
      if (ch == '\n') break;
      line.push_back(char(ch));
    }
    if (any) ++lineno;
    return any;
  };
  auto words = [](const std::string& s) {
    std::vector<std::string> w;
    size_t i = 0;
    while (i < s.size()) {
      while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
      size_t j = i;
      while (j < s.size() && !std::isspace((unsigned char)s[j])) ++j;
      if (j > i) w.emplace_back(s.substr(i, j - i));
      i = j;
    }
    return w;
  };
  if (!next_line()) { lineno = 1; fail("empty file"); }
  std::vector<std::string> head = words(line);
  head.resize(5);
  if (head[0] != "%%MatrixMarket" || head[1] != "matrix") fail("missing MatrixMarket banner");
  if (head[2] == "array") fail("array (dense) format not supported");
  if (head[2] != "coordinate") fail("unknown format class: " + head[2]);
  const bool pattern = head[3] == "pattern";
  if (!pattern && head[3] != "real" && head[3] != "integer") fail("unsupported field type: " + head[3]);
  const bool symmetric = head[4] == "symmetric";
  if (!symmetric && head[4] != "general") fail("unsupported symmetry: " + head[4]);

  auto to_int = [](const std::string& s, int64_t& out) {
    char* end = nullptr;
    out = std::strtoll(s.c_str(), &end, 10);
    return end != s.c_str() && *end == '\0';
  };
  auto to_real = [](const std::string& s, double& out) {
    char* end = nullptr;
    out = std::strtod(s.c_str(), &end);
    return end != s.c_str() && *end == '\0';
  };
  int64_t m = 0, n = 0, entries = 0;
  for (;;) {
    if (!next_line()) fail("missing size line");
    if (line.empty() || line[0] == '%') continue;
    const auto w = words(line);
    if (w.size() < 3 || !to_int(w[0], m) || !to_int(w[1], n) || !to_int(w[2], entries)) fail("bad size line");
    break;
  }
  if (m < 0 || n < 0 || entries < 0) fail("negative size");

  struct Entry { int64_t r, c; float v; };
  std::vector<Entry> coo;
  coo.reserve(size_t(symmetric ? 2 * entries : entries));
  for (int64_t seen = 0; seen < entries;) {
    if (!next_line()) fail("unexpected end of file");
    if (line.empty() || line[0] == '%') continue;
    const auto w = words(line);
    int64_t i = 0, j = 0;
    double v = 1.0;
    if (w.size() < 2 || !to_int(w[0], i) || !to_int(w[1], j) ||
        (!pattern && (w.size() < 3 || !to_real(w[2], v))))
      fail("bad entry");
    if (i < 1 || i > m || j < 1 || j > n) fail("entry index out of range");
    coo.push_back({i - 1, j - 1, float(v)});
    if (symmetric && i != j) coo.push_back({j - 1, i - 1, float(v)});
    ++seen;
  }
  // canonical order by (row, column). Duplicates are then summed left to right in float, so the
  // order among equal keys decides the last bit of a sum of three or more: std::sort with a
  // (row, column) comparator is what the reference calls (mmio.cpp:72-74), and the same library
  // algorithm on the same sequence yields the same permutation, hence the same bits.
  std::sort(coo.begin(), coo.end(), [](const Entry& a, const Entry& b) {
    return a.r != b.r ? a.r < b.r : a.c < b.c;
  });
  CsrMatrix a;
  a.m = m;
  a.n = n;
  a.row_ptr.assign(size_t(m) + 1, 0);
  for (size_t k = 0; k < coo.size();) {
    size_t k2 = k;
    float sum = 0.0f;
    bool first = true;
    while (k2 < coo.size() && coo[k2].r == coo[k].r && coo[k2].c == coo[k].c) {
      sum = first ? coo[k2].v : sum + coo[k2].v;
      first = false;
      ++k2;
    }
    a.col_indices.push_back(uint32_t(coo[k].c));
    a.vals.push_back(sum);
    ++a.row_ptr[size_t(coo[k].r) + 1];
    k = k2;
  }
  std::partial_sum(a.row_ptr.begin(), a.row_ptr.end(), a.row_ptr.begin());
  a.nnz = int64_t(a.col_indices.size());
  return a;
}

// "matrix coordinate real general", 1-based, values printed with %.9g
inline void write_matrix_market(const CsrMatrix& a, const std::string& path) {
  io_detail::File out(path, "w", "cannot open for write: ");
  std::fprintf(out.f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n",
               (long long)a.m, (long long)a.n, (long long)a.nnz);
  for (int64_t i = 0; i < a.m; ++i)
    for (uint64_t k = a.row_ptr[size_t(i)]; k < a.row_ptr[size_t(i) + 1]; ++k)
      std::fprintf(out.f, "%lld %u %.9g\n", (long long)(i + 1), a.col_indices[k] + 1u, double(a.vals[k]));
  if (std::ferror(out.f)) throw std::runtime_error("write failed: " + path);
}

// ---- generators, deterministic in the seed and bit-compatible with the reference -----------------
// random_dense (dense.hpp:23-25): one mt19937_64 draw per element, top 24 bits * 2^-24 in [0,1).
inline DenseMatrix random_dense(int64_t rows, int64_t cols, uint64_t seed) {
  if (rows < 1 || cols < 1) throw std::invalid_argument("random_dense: zero dimension");
  DenseMatrix x(rows, cols);
  std::mt19937_64 gen(seed);
  std::generate(x.data.begin(), x.data.end(), [&] { return float(gen() >> 40) * 0x1p-24f; });
  return x;
}

// random_csr (csr.hpp:31-34): square; per row two 53-bit uniforms pick the length
// floor(avg * (skew > 0 ? max(u,1e-9)^-skew * (1-skew) : 1) + u2) clipped to [0, rows]; then per
// row `len` columns gen() % rows, sorted (duplicates kept); then one 24-bit value per nonzero.
inline CsrMatrix random_csr(int64_t rows, double avg_row_nnz, double skew, uint64_t seed) {
  if (rows < 0 || avg_row_nnz < 0) throw std::invalid_argument("random_csr: bad shape");
  std::mt19937_64 gen(seed);
  const auto u53 = [&] { return double(gen() >> 11) * 0x1p-53; };
  CsrMatrix a;
  a.m = a.n = rows;
  a.row_ptr.assign(size_t(rows) + 1, 0);
  for (int64_t i = 0; i < rows; ++i) {
    const double u = u53();
    const double scale = skew > 0 ? std::pow(std::max(u, 1e-9), -skew) * (1.0 - skew) : 1.0;
    const double len = std::floor(avg_row_nnz * scale + u53());
    a.row_ptr[size_t(i) + 1] = a.row_ptr[size_t(i)] + uint64_t(std::clamp(len, 0.0, double(rows)));
  }
  a.nnz = int64_t(a.row_ptr.back());
  a.col_indices.resize(size_t(a.nnz));
  a.vals.resize(size_t(a.nnz));
  for (int64_t i = 0; i < rows; ++i) {
    auto first = a.col_indices.begin() + long(a.row_ptr[size_t(i)]);
    auto last = a.col_indices.begin() + long(a.row_ptr[size_t(i) + 1]);
    std::generate(first, last, [&] { return uint32_t(gen() % uint64_t(rows)); });
    std::sort(first, last);
  }
  std::generate(a.vals.begin(), a.vals.end(), [&] { return float(gen() >> 40) * 0x1p-24f; });
  return a;
}

}  // namespace spmx
