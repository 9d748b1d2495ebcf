// ref_shim.cpp — C-ABI shim over the UNMODIFIED reference library (spmx).
//
// TEST INFRASTRUCTURE ONLY (see oracle/spmx_oracle.c for the rules). This file
// is our own code; it includes the reference's public headers from where they
// lie (/root/reference/proj/include, plus the header-only test generators in
// /root/reference/proj/tests/oracles.hpp) and is compiled together with the
// reference's own .cpp files by oracle/Makefile, target `ref` into
// oracle/_ref/libspmx_ref.so. No reference source is copied into this repo.
//
// Purpose: (1) pin oracle/spmx_oracle.c against the real thing, (2) generate the
// golden fixtures under tests/golden/, (3) serve as the "reference" CPU
// baseline arm of bench.py.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracles.hpp"  // reference tests/oracles.hpp: random_csr_rect, merge_walk
#include "spmx/csr.hpp"
#include "spmx/dense.hpp"
#include "spmx/executor.hpp"
#include "spmx/mmio.hpp"
#include "spmx/partition.hpp"
#include "spmx/reference.hpp"

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

spmx::CsrMatrix make_csr(int64_t m, int64_t n, int64_t nnz, const uint64_t* row_ptr,
                         const uint32_t* col, const float* vals) {
  spmx::CsrMatrix a;
  a.m = m;
  a.n = n;
  a.nnz = nnz;
  a.row_ptr.assign(row_ptr, row_ptr + m + 1);
  if (col) a.col_indices.assign(col, col + nnz);
  if (vals) a.vals.assign(vals, vals + nnz);
  return a;
}

spmx::Strategy to_strategy(int s) {
  switch (s) {
    case 0: return spmx::Strategy::RowSplit;
    case 1: return spmx::Strategy::NnzSplit;
    case 2: return spmx::Strategy::MergeSplit;
  }
  throw std::invalid_argument("ref_shim: bad strategy code");
}

void put_ranges(const std::vector<spmx::RowRange>& r, uint64_t* out) {
  for (size_t t = 0; t < r.size(); ++t) {
    out[2 * t] = r[t].begin;
    out[2 * t + 1] = r[t].end;
  }
}

struct Holder {
  spmx::CsrMatrix a;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- persistent CSR handle (avoids re-copying big inputs per call) ---------
void* ref_csr_create(int64_t m, int64_t n, int64_t nnz, const uint64_t* row_ptr,
                     const uint32_t* col, const float* vals) {
  auto* h = new Holder;
  h->a = make_csr(m, n, nnz, row_ptr, col, vals);
  return h;
}
void ref_csr_destroy(void* h) { delete static_cast<Holder*>(h); }

// run_spmm on a handle. backend: 0 native (JIT), 1 interpreter.
// times_s must hold `trials` doubles. y must hold m*d floats.
int ref_run_spmm(void* h, const float* x, int64_t x_rows, int64_t d, float* y, int strategy,
                 int dynamic, unsigned threads, int backend, uint64_t batch, unsigned trials,
                 double* times_s, double* codegen_s, unsigned* threads_used, double* gflops) {
  return guarded([&] {
    const spmx::CsrMatrix& a = static_cast<Holder*>(h)->a;
    spmx::DenseMatrix xm;
    xm.rows = x_rows;
    xm.cols = d;
    xm.data.assign(x, x + size_t(x_rows) * size_t(d));
    spmx::RunConfig cfg;
    cfg.strategy = to_strategy(strategy);
    cfg.dynamic_dispatch = dynamic != 0;
    cfg.threads = threads;
    cfg.backend = backend == 0 ? spmx::Backend::Native : spmx::Backend::Interp;
    cfg.batch_size = batch;
    cfg.trials = trials;
    auto [ym, rep] = spmx::run_spmm(a, xm, cfg);
    if (y) std::memcpy(y, ym.data.data(), ym.data.size() * sizeof(float));
    if (times_s)
      for (size_t i = 0; i < rep.times_s.size(); ++i) times_s[i] = rep.times_s[i];
    if (codegen_s) *codegen_s = rep.codegen_s;
    if (threads_used) *threads_used = rep.threads;
    if (gflops) *gflops = rep.gflops;
  });
}

int ref_spmm_reference(void* h, const float* x, int64_t x_rows, int64_t d, float* y) {
  return guarded([&] {
    const spmx::CsrMatrix& a = static_cast<Holder*>(h)->a;
    spmx::DenseMatrix xm;
    xm.rows = x_rows;
    xm.cols = d;
    xm.data.assign(x, x + size_t(x_rows) * size_t(d));
    spmx::DenseMatrix ym = spmx::spmm_reference(a, xm);
    std::memcpy(y, ym.data.data(), ym.data.size() * sizeof(float));
  });
}

int ref_validate_csr_count(void* h) {
  return int(spmx::validate_csr(static_cast<Holder*>(h)->a).size());
}

// ---- partitioner -----------------------------------------------------------
int ref_split_rows_static(uint64_t m, unsigned parts, uint64_t* out) {
  return guarded([&] { put_ranges(spmx::split_rows_static(m, parts), out); });
}
int ref_split_nnz(void* h, unsigned parts, uint64_t* out) {
  return guarded([&] { put_ranges(spmx::split_nnz(static_cast<Holder*>(h)->a, parts), out); });
}
int ref_split_merge(void* h, unsigned parts, uint64_t* out) {
  return guarded(
      [&] { put_ranges(spmx::split_merge(static_cast<Holder*>(h)->a, parts), out); });
}
int ref_merge_path_search(void* h, uint64_t k, uint64_t* out_i, uint64_t* out_j) {
  return guarded([&] {
    const spmx::CsrMatrix& a = static_cast<Holder*>(h)->a;
    spmx::MergeCoordinate c =
        spmx::merge_path_search(k, a.row_ptr.data() + 1, uint64_t(a.m), uint64_t(a.nnz));
    *out_i = c.i;
    *out_j = c.j;
  });
}
int ref_merge_walk(void* h, uint64_t k, uint64_t* out_i, uint64_t* out_j) {
  return guarded([&] {
    const spmx::CsrMatrix& a = static_cast<Holder*>(h)->a;
    spmx::MergeCoordinate c =
        spmx::test::merge_walk(k, a.row_ptr.data() + 1, uint64_t(a.m), uint64_t(a.nnz));
    *out_i = c.i;
    *out_j = c.j;
  });
}
int ref_make_partition(void* h, int strategy, unsigned parts, int dynamic, uint64_t batch,
                       uint64_t* out, int* n_ranges, int* has_dynamic) {
  return guarded([&] {
    spmx::WorkPartition p = spmx::make_partition(static_cast<Holder*>(h)->a,
                                                 to_strategy(strategy), parts, dynamic != 0, batch);
    if (out) put_ranges(p.ranges, out);
    if (n_ranges) *n_ranges = int(p.ranges.size());
    if (has_dynamic) *has_dynamic = p.dynamic.has_value() ? 1 : 0;
  });
}

// ---- metrics ---------------------------------------------------------------
uint64_t ref_checksum(const float* data, int64_t rows, int64_t cols) {
  spmx::DenseMatrix y;
  y.rows = rows;
  y.cols = cols;
  y.data.assign(data, data + size_t(rows) * size_t(cols));
  return spmx::checksum(y);
}
double ref_max_relative_error(const float* y, const float* ref, int64_t count) {
  spmx::DenseMatrix a, b;
  a.rows = b.rows = count;
  a.cols = b.cols = 1;
  a.data.assign(y, y + count);
  b.data.assign(ref, ref + count);
  return spmx::max_relative_error(a, b);
}

// ---- the reference's own generators (for reproducing its test instances) ----
void* ref_rng_create(uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_destroy(void* r) { delete static_cast<std::mt19937_64*>(r); }
uint64_t ref_rng_next(void* r) { return (*static_cast<std::mt19937_64*>(r))(); }

// tests/oracles.hpp:53-72, advancing the caller's generator exactly as the
// reference's tests do. Returns a CSR handle; read it back with ref_csr_dims /
// ref_csr_copy.
void* ref_random_csr_rect(void* rng, int64_t m, int64_t n, double density) {
  auto* h = new Holder;
  h->a = spmx::test::random_csr_rect(m, n, density, *static_cast<std::mt19937_64*>(rng));
  return h;
}
void* ref_random_csr(int64_t rows, double avg_row_nnz, double skew, uint64_t seed) {
  auto* h = new Holder;
  h->a = spmx::random_csr(rows, avg_row_nnz, skew, seed);
  return h;
}
void ref_csr_dims(void* h, int64_t* m, int64_t* n, int64_t* nnz) {
  const spmx::CsrMatrix& a = static_cast<Holder*>(h)->a;
  *m = a.m;
  *n = a.n;
  *nnz = a.nnz;
}
void ref_csr_copy(void* h, uint64_t* row_ptr, uint32_t* col, float* vals) {
  const spmx::CsrMatrix& a = static_cast<Holder*>(h)->a;
  std::memcpy(row_ptr, a.row_ptr.data(), a.row_ptr.size() * sizeof(uint64_t));
  if (!a.col_indices.empty())
    std::memcpy(col, a.col_indices.data(), a.col_indices.size() * sizeof(uint32_t));
  if (!a.vals.empty()) std::memcpy(vals, a.vals.data(), a.vals.size() * sizeof(float));
}
// ---- file formats (csr.cpp:65-104, mmio.cpp:20-110) ----------------------------------
int ref_save_csr_cache(void* h, const char* path) {
  return guarded([&] { spmx::save_csr_cache(static_cast<Holder*>(h)->a, path); });
}
void* ref_load_csr_cache(const char* path) {
  Holder* h = nullptr;
  if (guarded([&] { h = new Holder; h->a = spmx::load_csr_cache(path); }) != 0) { delete h; return nullptr; }
  return h;
}
void* ref_load_matrix_market(const char* path) {
  Holder* h = nullptr;
  if (guarded([&] { h = new Holder; h->a = spmx::load_matrix_market(path); }) != 0) { delete h; return nullptr; }
  return h;
}
int ref_write_matrix_market(void* h, const char* path) {
  return guarded([&] { spmx::write_matrix_market(static_cast<Holder*>(h)->a, path); });
}

int ref_random_dense(int64_t rows, int64_t cols, uint64_t seed, float* out) {
  return guarded([&] {
    spmx::DenseMatrix x = spmx::random_dense(rows, cols, seed);
    std::memcpy(out, x.data.data(), x.data.size() * sizeof(float));
  });
}

}  // extern "C"
