// spmx_workloads.hpp — host C++ generators for BASELINE.json's five configurations.
//
// The reference ships no generator for these distributions (its random_csr, src/csr.cpp:106-133,
// makes power-law row lengths with duplicate columns; random_dense is U[0,1)), and the paper's
// SuiteSparse inputs are not available, so seeded synthetic matrices with the stated shapes stand
// in for them. These functions are the C++ twin of
// paper_2312_05639_b200/workloads.py: the same counter-based hash (splitmix64 finaliser of
// (seed, stream, index)), hence the SAME arrays — integer structure and the uniform values are
// bit-identical to what the Python generator produces on a CPU or CUDA tensor; N(0,1) values
// (config c3) come from the same fp64 Box-Muller formula and agree to the last bit wherever the
// two libm's do (tests/test_host_workloads_cpu.py). Host only: no CUDA.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "spmx_types.hpp"

namespace spmx {
namespace workloads {

inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + stream * 0xD1B54A32D192ED03ull + 0x2545F4914F6CDD1Dull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// 64 hashed bits of (seed, stream, index)
struct Hash {
  uint64_t key;
  Hash(uint64_t seed, uint64_t stream) : key(stream_key(seed, stream)) {}
  uint64_t operator()(uint64_t idx) const { return mix64(mix64(idx) ^ key); }
};
inline uint64_t u24(uint64_t h) { return h >> 40; }
inline float uniform_pm1(uint64_t h) { return float(u24(h)) * 0x1p-23f - 1.0f; }       // U[-1,1), 2^-23 grid
inline float uniform_01_open_left(uint64_t h) { return float(u24(h) + 1) * 0x1p-24f; }   // U(0,1], 2^-24 grid
inline float normal01(uint64_t h) {  // Box-Muller from two 26-bit uniforms of one hash, in fp64
  const double u1 = (double(h >> 38) + 1.0) * 0x1p-26;
  const double u2 = double(h & ((1ull << 26) - 1)) * 0x1p-26;
  return float(std::sqrt(-2.0 * std::log(u1)) * std::cos((2.0 * 3.141592653589793) * u2));
}
enum class Dist { UniformPm1, Uniform01, Normal };
inline float draw(Dist d, uint64_t h) {
  return d == Dist::UniformPm1 ? uniform_pm1(h) : d == Dist::Uniform01 ? uniform_01_open_left(h) : normal01(h);
}

// X: rows x d, element (i, j) keyed by its flat index on stream 7
inline DenseMatrix dense(int64_t rows, int64_t d, uint64_t seed, Dist dist) {
  DenseMatrix x(rows, d);
  const Hash h(seed, 7);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows * d; ++i) x.data[size_t(i)] = draw(dist, h(uint64_t(i)));
  return x;
}

// CSR from sorted (row << 32 | col) keys; value k keyed by its position in CSR order (stream 3)
inline CsrMatrix csr_from_sorted_keys(const std::vector<uint64_t>& keys, int64_t m, int64_t n,
                                      uint64_t seed, Dist val_dist) {
  CsrMatrix a;
  a.m = m;
  a.n = n;
  a.nnz = int64_t(keys.size());
  a.row_ptr.assign(size_t(m) + 1, 0);
  a.col_indices.resize(keys.size());
  a.vals.resize(keys.size());
  for (uint64_t k : keys) ++a.row_ptr[size_t(k >> 32) + 1];
  for (int64_t r = 0; r < m; ++r) a.row_ptr[size_t(r) + 1] += a.row_ptr[size_t(r)];
  const Hash h(seed, 3);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < a.nnz; ++k) {
    a.col_indices[size_t(k)] = uint32_t(keys[size_t(k)] & 0xffffffffull);
    a.vals[size_t(k)] = draw(val_dist, h(uint64_t(k)));
  }
  return a;
}

// c1: exactly `deg` distinct uniformly random columns per row (the deg smallest of n hashed
// scores), sorted; values U[-1,1)
inline CsrMatrix uniform_fixed_degree(int64_t m, int64_t n, int deg, uint64_t seed) {
  if (deg > n) throw std::invalid_argument("uniform_fixed_degree: deg > n");
  std::vector<uint64_t> keys(size_t(m) * size_t(deg));
  const Hash h(seed, 1);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < m; ++r) {
    std::vector<std::pair<uint64_t, uint32_t>> score((size_t)n);
    for (int64_t c = 0; c < n; ++c) score[size_t(c)] = {h(uint64_t(r * n + c)) >> 1, uint32_t(c)};
    std::partial_sort(score.begin(), score.begin() + deg, score.end());
    std::vector<uint32_t> cols(size_t(deg), 0u);
    for (int k = 0; k < deg; ++k) cols[size_t(k)] = score[size_t(k)].second;
    std::sort(cols.begin(), cols.end());
    for (int k = 0; k < deg; ++k) keys[size_t(r) * size_t(deg) + size_t(k)] = (uint64_t(r) << 32) | cols[size_t(k)];
  }
  return csr_from_sorted_keys(keys, m, n, seed, Dist::UniformPm1);
}

// c2, c4, c5: R-MAT, edge_factor * 2^scale draws, one quadrant per bit level with probabilities
// (a, b, c, d) = (top-left, top-right, bottom-left, bottom-right), duplicate edges merged, columns
// sorted per row, one U(0,1] value per surviving edge
inline CsrMatrix rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed) {
  const uint64_t ta = uint64_t(std::llround(a * double(1 << 24)));
  const uint64_t tab = uint64_t(std::llround((a + b) * double(1 << 24)));
  const uint64_t tabc = uint64_t(std::llround((a + b + c) * double(1 << 24)));
  const int64_t n = int64_t(1) << scale;
  const int64_t e_total = int64_t(edge_factor) * n;
  std::vector<uint64_t> keys((size_t)e_total, 0);
  std::vector<Hash> level;
  for (int lvl = 0; lvl < scale; ++lvl) level.emplace_back(seed, 100 + uint64_t(lvl));
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < e_total; ++e) {
    uint64_t row = 0, col = 0;
    for (int lvl = 0; lvl < scale; ++lvl) {
      const uint64_t u = u24(level[size_t(lvl)](uint64_t(e)));
      const bool right = (u >= ta && u < tab) || u >= tabc;  // quadrants b, d
      const bool down = u >= tab;                            // quadrants c, d
      row = (row << 1) | uint64_t(down);
      col = (col << 1) | uint64_t(right);
    }
    keys[size_t(e)] = (row << 32) | col;
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  return csr_from_sorted_keys(keys, n, n, seed, Dist::Uniform01);
}

// integer CDF thresholds (scaled by 2^53) of Poisson(lam) clipped to [lo, hi]
inline std::vector<uint64_t> poisson_clipped_table(double lam, int lo, int hi) {
  std::vector<double> prob(size_t(hi) + 1, 0.0);
  for (int k = 0; k < 4 * hi; ++k) {
    const double p = std::exp(-lam + k * std::log(lam) - std::lgamma(double(k) + 1.0));
    prob[size_t(std::min(std::max(k, lo), hi))] += p;
  }
  double total = 0.0;
  for (double p : prob) total += p;
  std::vector<uint64_t> cdf;
  double acc = 0.0;
  for (int k = lo; k <= hi; ++k) {
    acc += prob[size_t(k)] / total;
    cdf.push_back(std::min<uint64_t>(uint64_t(acc * 9007199254740992.0), 1ull << 53));
  }
  cdf.back() = 1ull << 53;
  return cdf;
}

// c3: nnz per row ~ Poisson(lam) clipped to [lo, hi]; each column uniform in
// [i - half_band, i + half_band], clamped to [0, m); sorted per row, duplicates KEPT; values N(0,1)
inline CsrMatrix banded_poisson(int64_t m, double lam, int lo, int hi, int64_t half_band, uint64_t seed) {
  const std::vector<uint64_t> table = poisson_clipped_table(lam, lo, hi);
  const Hash hl(seed, 1), hc(seed, 2);
  std::vector<uint64_t> start(size_t(m) + 1, 0);
  for (int64_t r = 0; r < m; ++r) {
    const uint64_t u53 = hl(uint64_t(r)) >> 11;
    int len = int(std::upper_bound(table.begin(), table.end(), u53) - table.begin()) + lo;
    len = std::min(std::max(len, lo), hi);
    start[size_t(r) + 1] = start[size_t(r)] + uint64_t(len);
  }
  std::vector<uint64_t> keys((size_t)start[size_t(m)]);
  const uint64_t width = uint64_t(2 * half_band + 1);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < m; ++r) {
    for (uint64_t k = start[size_t(r)]; k < start[size_t(r) + 1]; ++k) {
      const int64_t off = int64_t((hc(k) >> 1) % width) - half_band;
      const int64_t col = std::min<int64_t>(std::max<int64_t>(r + off, 0), m - 1);
      keys[size_t(k)] = (uint64_t(r) << 32) | uint64_t(col);
    }
    std::sort(keys.begin() + int64_t(start[size_t(r)]), keys.begin() + int64_t(start[size_t(r) + 1]));
  }
  return csr_from_sorted_keys(keys, m, m, seed, Dist::Normal);
}

struct Config {
  std::string name;
  CsrMatrix a;
  DenseMatrix x;
  int d = 0;
  uint64_t seed = 0;
};

inline int config_index(const std::string& name) {
  if (name.size() == 2 && name[0] == 'c' && name[1] >= '1' && name[1] <= '5') return name[1] - '0';
  throw std::invalid_argument("unknown config: " + name + " (c1 .. c5)");
}
inline uint64_t make_config_seed(const std::string& name) { return uint64_t(config_index(name)); }
inline int config_width(const std::string& name) {
  static const int d[] = {0, 32, 64, 128, 32, 128};
  return d[config_index(name)];
}

// BASELINE.json config `name` ("c1" .. "c5"). scale > 0 shrinks an R-MAT config to 2^scale rows,
// rows > 0 shrinks c1 / c3 (siblings with the same distribution, for small tests).
inline Config make_config(const std::string& name, int scale = 0, int64_t rows = 0) {
  Config c;
  c.name = name;
  if (name == "c1") {
    const int64_t m = rows > 0 ? rows : 4096;
    c.seed = 1; c.d = 32;
    c.a = uniform_fixed_degree(m, m, 16, c.seed);
    c.x = dense(c.a.n, c.d, c.seed, Dist::UniformPm1);
  } else if (name == "c2") {
    c.seed = 2; c.d = 64;
    c.a = rmat(scale > 0 ? scale : 20, 16, 0.57, 0.19, 0.19, c.seed);
    c.x = dense(c.a.n, c.d, c.seed, Dist::UniformPm1);
  } else if (name == "c3") {
    const int64_t m = rows > 0 ? rows : (int64_t(1) << 22);
    c.seed = 3; c.d = 128;
    c.a = banded_poisson(m, 32.0, 1, 64, std::min<int64_t>(65536, std::max<int64_t>(1, m / 4)), c.seed);
    c.x = dense(c.a.n, c.d, c.seed, Dist::Normal);
  } else if (name == "c4") {
    c.seed = 4; c.d = 32;
    c.a = rmat(scale > 0 ? scale : 22, 32, 0.65, 0.15, 0.15, c.seed);
    c.x = dense(c.a.n, c.d, c.seed, Dist::UniformPm1);
  } else if (name == "c5") {
    c.seed = 5; c.d = 128;
    c.a = rmat(scale > 0 ? scale : 24, 16, 0.57, 0.19, 0.19, c.seed);
    c.x = dense(c.a.n, c.d, c.seed, Dist::UniformPm1);
  } else {
    throw std::invalid_argument("unknown config: " + name + " (c1 .. c5)");
  }
  return c;
}

}  // namespace workloads
}  // namespace spmx
