// test_host_mirror.cpp — the reference's executor/partition test cases, written against the
// C++ host mirror (paper_2312_05639_b200/host/spmx_b200.hpp) exactly as they would be written
// against the reference's headers. Cases follow /root/reference/proj/tests/test_executor.cpp,
// test_partition.cpp and acceptance.cpp (criteria 2, 3, 5); expected values come from the
// test-only oracle (oracle/liboracle.so). Needs a GPU. Prints one line per case; exit code 1
// on any failure.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "../../paper_2312_05639_b200/host/spmx_b200.hpp"

extern "C" {  // oracle/spmx_oracle.c
int oracle_spmm_unfused(int64_t, int64_t, const uint64_t*, const uint32_t*, const float*, const float*,
                        int64_t, int64_t, float*);
int oracle_spmm_fused(int64_t, int64_t, const uint64_t*, const uint32_t*, const float*, const float*,
                      int64_t, int64_t, float*, int, int*);
uint64_t oracle_checksum(const float*, size_t);
int oracle_split_nnz(uint64_t, uint64_t, const uint64_t*, unsigned, uint64_t*);
int oracle_split_merge(uint64_t, uint64_t, const uint64_t*, unsigned, uint64_t*);
int oracle_split_rows_static(uint64_t, unsigned, uint64_t*);
void oracle_merge_walk(uint64_t, const uint64_t*, uint64_t, uint64_t, uint64_t*, uint64_t*);
}

using namespace spmx;

static int g_fail = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    if (!(cond)) {                                                               \
      std::printf("  CHECK failed at line %d: %s\n", __LINE__, #cond);           \
      ++g_fail;                                                                  \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                              \
  do {                                                                           \
    bool ok_ = false;                                                            \
    try { (void)(expr); } catch (const type&) { ok_ = true; } catch (...) {}     \
    if (!ok_) { std::printf("  expected " #type " at line %d\n", __LINE__); ++g_fail; } \
  } while (0)

static CsrMatrix from_row_lengths(std::initializer_list<uint64_t> lens) {
  CsrMatrix a;
  a.m = int64_t(lens.size());
  a.n = 1;
  a.row_ptr.assign(1, 0);
  for (uint64_t l : lens) a.row_ptr.push_back(a.row_ptr.back() + l);
  a.nnz = int64_t(a.row_ptr.back());
  a.col_indices.assign(size_t(a.nnz), 0);
  a.vals.assign(size_t(a.nnz), 1.0f);
  return a;
}

static CsrMatrix identity(int64_t n) {
  CsrMatrix a;
  a.m = a.n = a.nnz = n;
  for (int64_t i = 0; i <= n; ++i) a.row_ptr.push_back(uint64_t(i));
  for (int64_t i = 0; i < n; ++i) { a.col_indices.push_back(uint32_t(i)); a.vals.push_back(1.0f); }
  return a;
}

static CsrMatrix random_rect(int64_t m, int64_t n, double density, std::mt19937_64& rng) {
  CsrMatrix a;
  a.m = m; a.n = n;
  a.row_ptr.assign(1, 0);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < n; ++j)
      if (uni(rng) < density) { a.col_indices.push_back(uint32_t(j)); a.vals.push_back(float(rng() >> 40) * 0x1p-24f); }
    a.row_ptr.push_back(a.col_indices.size());
  }
  a.nnz = int64_t(a.col_indices.size());
  return a;
}

static DenseMatrix random_dense(int64_t rows, int64_t cols, uint64_t seed) {
  DenseMatrix x(rows, cols);
  std::mt19937_64 rng(seed);
  for (auto& v : x.data) v = float(rng() >> 40) * 0x1p-24f;
  return x;
}

static std::vector<RunConfig> all_configs(Backend backend, unsigned threads) {
  std::vector<RunConfig> out;
  for (Strategy s : {Strategy::RowSplit, Strategy::NnzSplit, Strategy::MergeSplit})
    for (bool dyn : {false, true}) {
      if (dyn && s != Strategy::RowSplit) continue;
      RunConfig cfg;
      cfg.strategy = s; cfg.dynamic_dispatch = dyn; cfg.threads = threads; cfg.backend = backend;
      cfg.batch_size = 16;
      out.push_back(cfg);
    }
  return out;
}

static std::vector<RowRange> flat_to_ranges(const std::vector<uint64_t>& f) {
  std::vector<RowRange> r(f.size() / 2);
  for (size_t t = 0; t < r.size(); ++t) r[t] = {f[2 * t], f[2 * t + 1]};
  return r;
}

static void partition_cases() {
  std::printf("partition goldens and errors\n");
  CHECK((split_rows_static(10, 4) == std::vector<RowRange>{{0, 3}, {3, 6}, {6, 8}, {8, 10}}));
  CHECK((split_rows_static(2, 4) == std::vector<RowRange>{{0, 1}, {1, 2}, {2, 2}, {2, 2}}));
  CHECK_THROWS_AS(split_rows_static(5, 0), std::invalid_argument);
  CsrMatrix a = from_row_lengths({4, 1, 1, 2});
  CHECK((split_nnz(a, 2) == std::vector<RowRange>{{0, 1}, {1, 4}}));
  CHECK((split_nnz(a, 1) == std::vector<RowRange>{{0, 4}}));
  CHECK((split_nnz(from_row_lengths({0, 0, 0}), 2) == std::vector<RowRange>{{0, 0}, {0, 3}}));
  CHECK_THROWS_AS(split_nnz(a, 0), std::invalid_argument);
  const uint64_t* row_end = a.row_ptr.data() + 1;
  CHECK(merge_path_search(0, row_end, 4, 8).i == 0);
  CHECK(merge_path_search(12, row_end, 4, 8).i == 4);
  CHECK(merge_path_search(12, row_end, 4, 8).j == 8);
  CHECK(merge_path_search(6, row_end, 4, 8).i == 1);
  CHECK(merge_path_search(6, row_end, 4, 8).j == 5);
  CHECK_THROWS_AS(merge_path_search(13, row_end, 4, 8), std::invalid_argument);
  CHECK((split_merge(a, 2) == std::vector<RowRange>{{0, 1}, {1, 4}}));
  CHECK((split_merge(from_row_lengths({3, 3, 3, 3, 3, 3}), 3) == std::vector<RowRange>{{0, 2}, {2, 4}, {4, 6}}));
  CsrMatrix b = from_row_lengths({2, 2, 2});
  WorkPartition p = make_partition(b, Strategy::RowSplit, 4, true, 128);
  CHECK(p.dynamic.has_value());
  CHECK(p.ranges.empty());
  CHECK_THROWS_AS(make_partition(b, Strategy::NnzSplit, 4, true, 128), std::invalid_argument);
  CHECK_THROWS_AS(make_partition(b, Strategy::RowSplit, 4, true, 0), std::invalid_argument);
  CHECK(make_partition(b, Strategy::MergeSplit, 2, false, 128).ranges.size() == 2);

  std::printf("partition vs oracle on random instances, every merge diagonal\n");
  std::mt19937_64 rng(17);
  for (int it = 0; it < 25; ++it) {
    CsrMatrix r = random_rect(1 + int64_t(rng() % 30), 20, 0.2, rng);
    const uint64_t m = uint64_t(r.m), nnz = uint64_t(r.nnz);
    unsigned t = 1 + unsigned(rng() % 12);
    std::vector<uint64_t> f(2 * t);
    oracle_split_nnz(m, nnz, r.row_ptr.data(), t, f.data());
    CHECK(split_nnz(r, t) == flat_to_ranges(f));
    oracle_split_merge(m, nnz, r.row_ptr.data(), t, f.data());
    CHECK(split_merge(r, t) == flat_to_ranges(f));
    oracle_split_rows_static(m, t, f.data());
    CHECK(split_rows_static(m, t) == flat_to_ranges(f));
    std::vector<uint64_t> ks;
    for (uint64_t k = 0; k <= m + nnz; ++k) ks.push_back(k);
    auto got = merge_path_search(r, ks);
    for (uint64_t k = 0; k <= m + nnz; ++k) {
      uint64_t wi, wj;
      oracle_merge_walk(k, r.row_ptr.data() + 1, m, nnz, &wi, &wj);
      if (got[k].i != wi || got[k].j != wj) { CHECK(false && "merge_path_search != merge_walk"); break; }
    }
  }
}

static void executor_cases() {
  std::printf("identity returns X bitwise under every configuration\n");
  {
    CsrMatrix a = identity(64);
    DenseMatrix x = random_dense(64, 45, 3);
    for (Backend backend : {Backend::Interp, Backend::Native})
      for (unsigned t : {1u, 3u, 8u})
        for (const RunConfig& cfg : all_configs(backend, t)) {
          auto [y, report] = run_spmm(a, x, cfg);
          CHECK(y.data == x.data);
          if (!cfg.dynamic_dispatch) CHECK(report.threads == t);
        }
  }
  std::printf("result invariant across strategies and T (checksum), tolerance vs reference\n");
  {
    std::mt19937_64 rng(51);
    CsrMatrix a = random_rect(200, 200, 0.05, rng);
    DenseMatrix x = random_dense(200, 45, 9);
    DenseMatrix fused(200, 45), unfused(200, 45);
    oracle_spmm_fused(a.m, a.n, a.row_ptr.data(), a.col_indices.data(), a.vals.data(), x.data.data(),
                      x.rows, x.cols, fused.data.data(), 1, nullptr);
    oracle_spmm_unfused(a.m, a.n, a.row_ptr.data(), a.col_indices.data(), a.vals.data(),
                        x.data.data(), x.rows, x.cols, unfused.data.data());
    const uint64_t want = oracle_checksum(fused.data.data(), fused.data.size());
    int checked = 0;
    for (unsigned t : {1u, 2u, 4u, 7u}) {
      for (const RunConfig& cfg : all_configs(Backend::Interp, t)) {  // exact order: bitwise
        CHECK(checksum(run_spmm(a, x, cfg).first) == want);
        ++checked;
      }
      for (const RunConfig& cfg : all_configs(Backend::Native, t)) {  // default mode: 1e-5
        DenseMatrix y = run_spmm(a, x, cfg).first;
        CHECK(max_relative_error(y, unfused) <= kVerifyTolerance);
      }
    }
    CHECK(checked >= 16);
    // spmm_reference of the mirror (device) is bitwise the reference's Alg. 1
    CHECK(spmm_reference(a, x).data == unfused.data);
  }
  std::printf("verify path and report bookkeeping\n");
  {
    std::mt19937_64 rng(53);
    CsrMatrix a = random_rect(80, 80, 0.1, rng);
    DenseMatrix x = random_dense(80, 20, 1);
    RunConfig cfg;
    cfg.threads = 2; cfg.verify = true; cfg.dynamic_dispatch = false;
    auto [y, report] = run_spmm(a, x, cfg);
    CHECK(report.max_rel_err.has_value());
    CHECK(*report.max_rel_err <= kVerifyTolerance);
    CHECK(*report.max_rel_err == max_relative_error(y, spmm_reference(a, x)));
    CsrMatrix id = identity(32);
    DenseMatrix x8 = random_dense(32, 8, 4);
    RunConfig c3; c3.threads = 1; c3.trials = 3; c3.dynamic_dispatch = false;
    RunReport rep = run_spmm(id, x8, c3).second;
    CHECK(rep.times_s.size() == 3);
    double sum = 0;
    for (double t : rep.times_s) { CHECK(t >= 0.0); sum += t; }
    CHECK(std::fabs(rep.mean_s - sum / 3) <= 1e-12 * (1 + sum));
    CHECK(std::fabs(rep.gflops - 2.0 * 32 * 8 / rep.mean_s / 1e9) <= 1e-9 * rep.gflops);
  }
  std::printf("run_spmm rejects bad configurations\n");
  {
    CsrMatrix a = identity(4);
    DenseMatrix x = random_dense(4, 4, 1);
    RunConfig cfg;
    cfg.strategy = Strategy::NnzSplit; cfg.dynamic_dispatch = true;
    CHECK_THROWS_AS(run_spmm(a, x, cfg), std::invalid_argument);
    RunConfig ok;
    DenseMatrix bad = random_dense(5, 4, 1);
    CHECK_THROWS_AS(run_spmm(a, bad, ok), std::invalid_argument);
    RunConfig zero_trials; zero_trials.trials = 0;
    CHECK_THROWS_AS(run_spmm(a, x, zero_trials), std::invalid_argument);
    RunConfig zero_batch; zero_batch.batch_size = 0;
    CHECK_THROWS_AS(run_spmm(a, x, zero_batch), std::invalid_argument);
    CsrMatrix broken = identity(4);
    broken.col_indices[2] = 9;  // column out of range
    CHECK_THROWS_AS(run_spmm(broken, x, ok), std::invalid_argument);
  }
  std::printf("acceptance-style sweep: 60 random instances x cells x T x backends\n");
  {
    const int d_pool[] = {1, 2, 3, 4, 5, 7, 8, 15, 16, 17, 31, 32, 45, 64, 100};
    std::mt19937_64 rng(2026);
    for (int it = 0; it < 60; ++it) {
      int64_t m = 1 + int64_t(rng() % 200), n = 1 + int64_t(rng() % 200);
      double density = 0.005 + 0.195 * double(rng() % 1000) / 1000.0;
      CsrMatrix a = random_rect(m, n, density, rng);
      int d = d_pool[rng() % 15];
      DenseMatrix x = random_dense(n, d, rng());
      DenseMatrix fused(m, d), unfused(m, d);
      oracle_spmm_fused(m, n, a.row_ptr.data(), a.col_indices.data(), a.vals.data(), x.data.data(), n, d,
                        fused.data.data(), 1, nullptr);
      oracle_spmm_unfused(m, n, a.row_ptr.data(), a.col_indices.data(), a.vals.data(), x.data.data(), n, d,
                          unfused.data.data());
      const uint64_t want = oracle_checksum(fused.data.data(), fused.data.size());
      for (unsigned t : {1u, 4u, 8u})
        for (const RunConfig& base : all_configs(Backend::Interp, t)) {
          RunConfig cfg = base;
          cfg.batch_size = 32;
          if (checksum(run_spmm(a, x, cfg).first) != want) { CHECK(false && "exact-order checksum"); }
          cfg.backend = Backend::Native;
          if (max_relative_error(run_spmm(a, x, cfg).first, unfused) > kVerifyTolerance) { CHECK(false && "1e-5"); }
        }
    }
  }
}

// RunConfig.gpus / shards: the same run_spmm call through the library's multi-GPU driver. On this
// one-GPU box the row blocks of split_nnz(A, S) / split_merge(A, S) all live on device 0; the
// result must not depend on how the rows were divided (test_executor.cpp:67-87 one level up).
static void multi_gpu_cases() {
  std::printf("multi-GPU driver through run_spmm (row blocks on one device)\n");
  std::mt19937_64 rng(77);
  CsrMatrix a = random_rect(3000, 900, 0.02, rng);
  DenseMatrix x = random_dense(a.n, 45, 5);
  DenseMatrix fused(a.m, 45), unfused(a.m, 45);
  oracle_spmm_fused(a.m, a.n, a.row_ptr.data(), a.col_indices.data(), a.vals.data(), x.data.data(), a.n, 45,
                    fused.data.data(), 1, nullptr);
  oracle_spmm_unfused(a.m, a.n, a.row_ptr.data(), a.col_indices.data(), a.vals.data(), x.data.data(), a.n, 45,
                      unfused.data.data());
  const uint64_t want = oracle_checksum(fused.data.data(), fused.data.size());
  for (unsigned shards : {2u, 5u, 8u})
    for (bool by_merge : {false, true})
      for (const RunConfig& base : all_configs(Backend::Interp, 4)) {
        RunConfig cfg = base;
        cfg.gpus = 1;
        cfg.shards = shards;
        cfg.shard_by_merge = by_merge;
        cfg.trials = 2;
        auto [y, rep] = run_spmm(a, x, cfg);
        CHECK(checksum(y) == want);
        CHECK(rep.times_s.size() == 2 && rep.gpus == 1 && rep.shard_rows.size() == shards);
        std::vector<uint64_t> flat(2 * size_t(shards));
        if (by_merge) oracle_split_merge(uint64_t(a.m), uint64_t(a.nnz), a.row_ptr.data(), shards, flat.data());
        else oracle_split_nnz(uint64_t(a.m), uint64_t(a.nnz), a.row_ptr.data(), shards, flat.data());
        for (unsigned t = 0; t < shards; ++t)
          CHECK(rep.shard_rows[t].begin == flat[2 * t] && rep.shard_rows[t].end == flat[2 * t + 1]);
        cfg.backend = Backend::Native;
        cfg.verify = true;
        auto [y2, rep2] = run_spmm(a, x, cfg);
        CHECK(rep2.max_rel_err && *rep2.max_rel_err <= kVerifyTolerance);
        CHECK(max_relative_error(y2, unfused) <= kVerifyTolerance);
      }
  RunConfig bad;
  bad.gpus = 64;  // more GPUs than the box has
  bad.dynamic_dispatch = false;
  CHECK_THROWS_AS(run_spmm(a, x, bad), std::invalid_argument);
}

int main() {
  try {
    partition_cases();
    executor_cases();
    multi_gpu_cases();
  } catch (const std::exception& e) {
    std::printf("unexpected exception: %s\n", e.what());
    return 2;
  }
  std::printf("%s (%d failed checks)\n", g_fail == 0 ? "host mirror: ALL PASS" : "host mirror: FAILURES", g_fail);
  return g_fail == 0 ? 0 : 1;
}
