/*
 * spmx_oracle.c — CPU restatement of the reference's CSR SpMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing under paper_2312_05639_b200/ may link,
 * import or call this file. Allowed users: tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs, and there only as the
 * checker or as the reported CPU baseline, never as the thing shipped.
 *
 * Parity status: PINNED. Every function below is checked (tests/test_oracle_*.py)
 * against (a) the reference's own golden vectors restated in tests/golden/ and
 * (b) outputs of the unmodified reference library compiled from
 * /root/reference/proj/src into oracle/_ref/libspmx_ref.so (oracle/Makefile, target `ref`).
 *
 * Each function cites the reference file:line it follows
 * (paths relative to /root/reference/proj).
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC (see oracle/Makefile).
 * -ffp-contract=off matters: oracle_spmm_unfused must stay mul-then-add with
 * two roundings (reference CMakeLists.txt:14-16), the fused variant calls
 * fmaf() explicitly.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_EINVAL 1 /* the reference throws std::invalid_argument here */

/* ---- SpMM ---------------------------------------------------------------- */

/* Serial, unfused, column-outer: follows src/reference.cpp:10-25 (Alg. 1).
 * For each (i, j): ret = 0; for idx in row i (CSR order): ret += v * X[k][j]. */
int oracle_spmm_unfused(int64_t m, int64_t n, const uint64_t* row_ptr, const uint32_t* col,
                        const float* vals, const float* x, int64_t x_rows, int64_t d, float* y) {
  if (n != x_rows) return ORACLE_EINVAL; /* reference.cpp:11 */
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t j = 0; j < d; ++j) {
      float ret = 0.0f;
      for (uint64_t idx = row_ptr[i]; idx < row_ptr[i + 1]; ++idx) {
        float prod = vals[idx] * x[(size_t)col[idx] * (size_t)d + (size_t)j];
        ret = ret + prod;
      }
      y[(size_t)i * (size_t)d + (size_t)j] = ret;
    }
  }
  return ORACLE_OK;
}

/* One row range with fused multiply-add in CSR order: follows
 * src/interp.cpp:26-57 (run_row). The register tiling of the plan does not
 * change any element's accumulation chain (each (row, j) is an independent
 * fmaf chain over the row's nonzeros in CSR order), so the tiles collapse to
 * a plain j loop. Every row in [row_begin,row_end) is stored, empty rows as
 * zeros (interp.cpp:53); an empty range writes nothing. */
static void fused_rows(const uint64_t* row_ptr, const uint32_t* col, const float* vals,
                       const float* x, int64_t d, float* y, uint64_t row_begin,
                       uint64_t row_end) {
  float* acc = (float*)malloc(sizeof(float) * (size_t)(d > 0 ? d : 1));
  for (uint64_t r = row_begin; r < row_end; ++r) {
    for (int64_t j = 0; j < d; ++j) acc[j] = 0.0f;
    for (uint64_t idx = row_ptr[r]; idx < row_ptr[r + 1]; ++idx) {
      const float v = vals[idx];
      const float* xrow = x + (size_t)col[idx] * (size_t)d;
      for (int64_t j = 0; j < d; ++j) acc[j] = fmaf(v, xrow[j], acc[j]); /* interp.cpp:43 */
    }
    memcpy(y + (size_t)r * (size_t)d, acc, sizeof(float) * (size_t)d);
  }
  free(acc);
}

int oracle_spmm_fused_range(int64_t m, int64_t n, const uint64_t* row_ptr, const uint32_t* col,
                            const float* vals, const float* x, int64_t x_rows, int64_t d,
                            float* y, uint64_t row_begin, uint64_t row_end) {
  if (n != x_rows) return ORACLE_EINVAL; /* interp.cpp:13 */
  if (row_end > (uint64_t)m || row_begin > row_end) return ORACLE_EINVAL;
  fused_rows(row_ptr, col, vals, x, d, y, row_begin, row_end);
  return ORACLE_OK;
}

/* Whole matrix, fused, optionally multi-threaded over static row blocks
 * (executor.cpp:70-97 with Backend::Interp semantics; the result does not
 * depend on the thread count because rows are single-writer).
 * threads <= 0 means "all logical cores" (executor.cpp:42). Returns the
 * thread count used through *threads_used when non-null. */
int oracle_spmm_fused(int64_t m, int64_t n, const uint64_t* row_ptr, const uint32_t* col,
                      const float* vals, const float* x, int64_t x_rows, int64_t d, float* y,
                      int threads, int* threads_used) {
  if (n != x_rows) return ORACLE_EINVAL;
  int t = threads;
#ifdef _OPENMP
  if (t <= 0) t = omp_get_max_threads();
#else
  t = 1;
#endif
  if (threads_used) *threads_used = t;
  /* dynamic row batches of 128, the reference's default dispatch
   * (partition.hpp:27, executor.hpp:22,27) */
#pragma omp parallel for schedule(dynamic, 1) num_threads(t)
  for (int64_t b = 0; b < (m + 127) / 128; ++b) {
    uint64_t lo = (uint64_t)b * 128u;
    uint64_t hi = lo + 128u < (uint64_t)m ? lo + 128u : (uint64_t)m;
    fused_rows(row_ptr, col, vals, x, d, y, lo, hi);
  }
  return ORACLE_OK;
}

/* Per-element magnitude bound S[i][j] = sum_idx |a * x| in fp64, used by the
 * north_star tolerance |y - y_ref| <= 1e-5 * S + 1e-6 (BASELINE.json). */
int oracle_abs_bound(int64_t m, const uint64_t* row_ptr, const uint32_t* col, const float* vals,
                     const float* x, int64_t d, double* s) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < m; ++i) {
    double* srow = s + (size_t)i * (size_t)d;
    for (int64_t j = 0; j < d; ++j) srow[j] = 0.0;
    for (uint64_t idx = row_ptr[i]; idx < row_ptr[i + 1]; ++idx) {
      const double v = (double)vals[idx];
      const float* xrow = x + (size_t)col[idx] * (size_t)d;
      for (int64_t j = 0; j < d; ++j) srow[j] += fabs(v * (double)xrow[j]);
    }
  }
  return ORACLE_OK;
}

/* ---- metrics ------------------------------------------------------------- */

/* max_i |y_i - ref_i| / max(|ref_i|, 1e-6): follows src/executor.cpp:27-34. */
double oracle_max_relative_error(const float* y, const float* ref, size_t count) {
  double worst = 0.0;
  for (size_t i = 0; i < count; ++i) {
    double denom = fabs((double)ref[i]);
    if (denom < 1e-6) denom = 1e-6;
    double e = fabs((double)y[i] - (double)ref[i]) / denom;
    if (e > worst) worst = e;
  }
  return worst;
}

/* FNV-1a-64 over the raw little-endian f32 bytes: follows src/dense.cpp:17-28. */
uint64_t oracle_checksum(const float* data, size_t count) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < count; ++i) {
    uint32_t bits;
    memcpy(&bits, &data[i], 4);
    for (int s = 0; s < 32; s += 8) {
      h ^= (uint64_t)((bits >> s) & 0xffu);
      h *= 0x100000001b3ull;
    }
  }
  return h;
}

/* ---- partitioner ---------------------------------------------------------- */
/* Ranges are written as out[2*t] = begin, out[2*t+1] = end (half-open). */

/* follows src/partition.cpp:17-27 */
int oracle_split_rows_static(uint64_t m, unsigned parts, uint64_t* out) {
  if (parts == 0) return ORACLE_EINVAL;
  uint64_t base = m / parts, rem = m % parts, begin = 0;
  for (unsigned t = 0; t < parts; ++t) {
    uint64_t size = base + (t < rem ? 1u : 0u);
    out[2 * t] = begin;
    out[2 * t + 1] = begin + size;
    begin += size;
  }
  return ORACLE_OK;
}

/* first index in row_ptr[0..m] whose value is >= target (std::lower_bound) */
static uint64_t lower_bound_u64(const uint64_t* a, uint64_t count, uint64_t target) {
  uint64_t lo = 0, hi = count;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < target)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

/* follows src/partition.cpp:35-51 */
int oracle_split_nnz(uint64_t m, uint64_t nnz, const uint64_t* row_ptr, unsigned parts,
                     uint64_t* out) {
  if (parts == 0) return ORACLE_EINVAL;
  uint64_t prev = 0;
  for (unsigned t = 1; t < parts; ++t) {
    uint64_t target = ((uint64_t)t * nnz + parts - 1) / parts; /* :42 */
    uint64_t r = lower_bound_u64(row_ptr, m + 1, target);      /* :43-44 */
    if (r > m) r = m;
    if (r < prev) r = prev; /* :45 */
    out[2 * (t - 1)] = prev;
    out[2 * (t - 1) + 1] = r;
    prev = r;
  }
  out[2 * (parts - 1)] = prev;
  out[2 * (parts - 1) + 1] = m;
  return ORACLE_OK;
}

/* follows src/partition.cpp:53-67; row_end[r] == row_ptr[r+1] */
int oracle_merge_path_search(uint64_t k, const uint64_t* row_end, uint64_t m, uint64_t nnz,
                             uint64_t* out_i, uint64_t* out_j) {
  if (k > m + nnz) return ORACLE_EINVAL; /* :55 */
  uint64_t lo = k > nnz ? k - nnz : 0;
  uint64_t hi = k < m ? k : m;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (row_end[mid] <= k - mid - 1)
      lo = mid + 1;
    else
      hi = mid;
  }
  *out_i = lo;
  *out_j = k - lo;
  return ORACLE_OK;
}

/* follows src/partition.cpp:69-84 (row-snapped: .j is discarded) */
int oracle_split_merge(uint64_t m, uint64_t nnz, const uint64_t* row_ptr, unsigned parts,
                       uint64_t* out) {
  if (parts == 0) return ORACLE_EINVAL;
  const uint64_t* row_end = row_ptr + 1;
  uint64_t prev = 0;
  for (unsigned t = 1; t < parts; ++t) {
    uint64_t k = ((uint64_t)t * (m + nnz) + parts - 1) / parts; /* :76 */
    uint64_t i, j;
    oracle_merge_path_search(k, row_end, m, nnz, &i, &j);
    uint64_t r = i < prev ? prev : i; /* :78 */
    out[2 * (t - 1)] = prev;
    out[2 * (t - 1) + 1] = r;
    prev = r;
  }
  out[2 * (parts - 1)] = prev;
  out[2 * (parts - 1) + 1] = m;
  return ORACLE_OK;
}

/* Sequential merge walk, the reference tests' independent check of the
 * binary search: follows tests/oracles.hpp:40-50. */
void oracle_merge_walk(uint64_t k, const uint64_t* row_end, uint64_t m, uint64_t nnz,
                       uint64_t* out_i, uint64_t* out_j) {
  uint64_t i = 0, j = 0;
  while (i + j < k) {
    if (i < m && (j >= nnz || row_end[i] <= j))
      ++i;
    else
      ++j;
  }
  *out_i = i;
  *out_j = j;
}

/* Dynamic dispatch claim (single-threaded restatement): follows
 * src/partition.cpp:29-33. Returns 1 and the claimed range, or 0 when the
 * counter has passed m. */
int oracle_next_batch(uint64_t* counter, uint64_t batch, uint64_t m, uint64_t* begin,
                      uint64_t* end) {
  uint64_t v = *counter;
  *counter += batch;
  if (v >= m) return 0;
  *begin = v;
  *end = v + batch < m ? v + batch : m;
  return 1;
}

/* CSR invariants: follows src/csr.cpp:18-42. Returns 0 when valid, else a
 * small code naming the first violated invariant. */
int oracle_validate_csr(int64_t m, int64_t n, int64_t nnz, const uint64_t* row_ptr,
                        const uint32_t* col) {
  if (m < 0 || n < 0 || nnz < 0) return 1;
  if (row_ptr[0] != 0) return 2;
  if (row_ptr[m] != (uint64_t)nnz) return 3;
  for (int64_t i = 0; i < m; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) return 4;
  for (int64_t k = 0; k < nnz; ++k)
    if ((int64_t)col[k] >= n) return 5;
  return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
