// spmx_types.hpp — the reference's two data types (include/spmx/csr.hpp:10-20,
// include/spmx/dense.hpp:9-21), shared by the device-backed API (spmx_b200.hpp) and the
// host-only file formats / generators (spmx_io.hpp).
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

namespace spmx {

struct CsrMatrix {
  int64_t m = 0, n = 0, nnz = 0;
  std::vector<uint64_t> row_ptr;
  std::vector<uint32_t> col_indices;
  std::vector<float> vals;
  uint64_t row_nnz(int64_t i) const { return row_ptr[size_t(i) + 1] - row_ptr[size_t(i)]; }
  uint64_t max_row_nnz() const {
    uint64_t best = 0;
    for (int64_t i = 0; i < m; ++i) best = std::max(best, row_nnz(i));
    return best;
  }
};

struct DenseMatrix {
  int64_t rows = 0, cols = 0;
  std::vector<float> data;
  DenseMatrix() = default;
  DenseMatrix(int64_t r, int64_t c) : rows(r), cols(c), data(size_t(r) * size_t(c), 0.0f) {}
  float& at(int64_t i, int64_t j) { return data[size_t(i) * size_t(cols) + size_t(j)]; }
  float at(int64_t i, int64_t j) const { return data[size_t(i) * size_t(cols) + size_t(j)]; }
  const float* row(int64_t i) const { return data.data() + size_t(i) * size_t(cols); }
  float* row(int64_t i) { return data.data() + size_t(i) * size_t(cols); }
};

}  // namespace spmx
