// spmx_partition.cuh — the reference's workload partitioner on the device.
//
// Every boundary is computed independently by one thread with the reference's own
// integer arithmetic, so the result is bit-exact with src/partition.cpp run serially
// (the reference's running `max(prev, r)` clamps are no-ops for a valid CSR because
// targets, and therefore the search results, are nondecreasing in t; a CSR that
// breaks that is rejected at upload by validate_csr_kernel).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace spmx_dev {

typedef unsigned long long u64;

// split_rows_static, src/partition.cpp:17-27: boundary t = t*base + min(t, rem).
__global__ void row_boundaries_kernel(u64 m, unsigned parts, u64* __restrict__ bnd) {
  const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > parts) return;
  const u64 base = m / parts, rem = m % parts;
  bnd[t] = t * base + (t < rem ? t : rem);
}

// first index in a[0..count) with a[idx] >= target (std::lower_bound)
__device__ __forceinline__ u64 lower_bound_dev(const u64* __restrict__ a, u64 count, u64 target) {
  u64 lo = 0, hi = count;
  while (lo < hi) {
    const u64 mid = lo + (hi - lo) / 2;
    if (__ldg(a + mid) < target)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// split_nnz, src/partition.cpp:35-51: boundary t (1 <= t < T) is the first row r with
// row_ptr[r] >= ceil(t*nnz/T), searched over all m+1 entries and clamped to m.
__global__ void nnz_boundaries_kernel(const u64* __restrict__ row_ptr, u64 m, u64 nnz,
                                      unsigned parts, u64* __restrict__ bnd) {
  const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > parts) return;
  if (t == 0) { bnd[0] = 0; return; }
  if (t == parts) { bnd[t] = m; return; }
  const u64 target = (t * nnz + parts - 1) / parts;  // same u64 arithmetic as partition.cpp:42
  u64 r = lower_bound_dev(row_ptr, m + 1, target);
  bnd[t] = r < m ? r : m;
}

// merge_path_search, src/partition.cpp:53-67. row_end[r] == row_ptr[r+1].
__device__ __forceinline__ void merge_search_dev(const u64* __restrict__ row_ptr, u64 m, u64 nnz,
                                                 u64 k, u64& out_i, u64& out_j) {
  const u64* __restrict__ row_end = row_ptr + 1;
  u64 lo = k > nnz ? k - nnz : 0;
  u64 hi = k < m ? k : m;
  while (lo < hi) {
    const u64 mid = lo + (hi - lo) / 2;
    if (__ldg(row_end + mid) <= k - mid - 1)
      lo = mid + 1;
    else
      hi = mid;
  }
  out_i = lo;
  out_j = k - lo;
}

__global__ void merge_search_kernel(const u64* __restrict__ row_ptr, u64 m, u64 nnz,
                                    const u64* __restrict__ diag, u64 n_diag,
                                    u64* __restrict__ out_i, u64* __restrict__ out_j) {
  const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_diag) return;
  u64 i, j;
  merge_search_dev(row_ptr, m, nnz, diag[t], i, j);
  out_i[t] = i;
  out_j[t] = j;
}

// split_merge, src/partition.cpp:69-84: diagonal ceil(t*(m+nnz)/T); keep .i (row-snapped).
// With snapped == 0 the diagonal itself is returned instead (true merge-path split).
__global__ void merge_boundaries_kernel(const u64* __restrict__ row_ptr, u64 m, u64 nnz,
                                        unsigned parts, int snapped, u64* __restrict__ out) {
  const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > parts) return;
  if (t == 0) { out[0] = 0; return; }
  if (t == parts) { out[t] = snapped ? m : m + nnz; return; }
  const u64 k = (t * (m + nnz) + parts - 1) / parts;  // partition.cpp:76
  if (!snapped) { out[t] = k; return; }
  u64 i, j;
  merge_search_dev(row_ptr, m, nnz, k, i, j);
  out[t] = i;
}

// RowRange list from T+1 boundaries: out[2t] = bnd[t], out[2t+1] = bnd[t+1].
__global__ void ranges_from_boundaries_kernel(const u64* __restrict__ bnd, unsigned parts,
                                              u64* __restrict__ out) {
  const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= parts) return;
  out[2 * t] = bnd[t];
  out[2 * t + 1] = bnd[t + 1];
}

// Row boundary b -> the merge-path diagonal through (b, row_ptr[b]).
__global__ void boundaries_to_diagonals_kernel(const u64* __restrict__ row_ptr,
                                               const u64* __restrict__ bnd, u64 count,
                                               u64* __restrict__ diag) {
  const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const u64 b = bnd[t];
  diag[t] = b + __ldg(row_ptr + b);
}

// Work-list refinement: a strategy range of `items` merge items becomes
// max(1, ceil(items / chunk_items)) chunks.
__global__ void count_chunks_kernel(const u64* __restrict__ diag, u64 parts, u64 chunk_items,
                                    u64 taper2, u64 taper4, u64* __restrict__ cnt) {
  const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= parts) return;
  const u64 items = diag[t + 1] - diag[t];
  // the ranges launched last are cut finer (half- and quarter-size chunks from diagonals
  // taper2 and taper4 on): the grid's tail then ends on short pieces
  if (diag[t] >= taper4) chunk_items = max(chunk_items / 4, (u64)32);
  else if (diag[t] >= taper2) chunk_items = max(chunk_items / 2, (u64)32);
  const u64 c = (items + chunk_items - 1) / chunk_items;
  cnt[t] = c ? c : 1;
}

// Exclusive scan of cnt[0..n) into off[0..n], off[n] = total. One CTA; n is at most a
// few million and this runs once per plan, outside any timed region.
__global__ void exclusive_scan_kernel(const u64* __restrict__ cnt, u64 n, u64* __restrict__ off) {
  __shared__ u64 part[1024];
  const u64 per = (n + blockDim.x - 1) / blockDim.x;
  const u64 lo = min((u64)threadIdx.x * per, n), hi = min(lo + per, n);
  u64 s = 0;
  for (u64 i = lo; i < hi; ++i) s += cnt[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 run = 0;
    for (unsigned i = 0; i < blockDim.x; ++i) {
      const u64 v = part[i];
      part[i] = run;
      run += v;
    }
    off[n] = run;
  }
  __syncthreads();
  u64 run = part[threadIdx.x];
  for (u64 i = lo; i < hi; ++i) {
    off[i] = run;
    run += cnt[i];
  }
}

// Work-list coordinates. Chunk c belongs to range t = upper_bound(off, c) - 1 and is its
// s-th piece; its starting diagonal is diag[t] + floor(s * items / cnt) (even split of the
// range), located on the merge path with the reference's own search. s == 0 is the
// strategy's boundary and is kept exactly. An interior boundary that falls inside a row
// shorter than snap_len is moved back to the start of that row: short rows are then never
// cut (they stay one fmaf chain, bitwise equal to the reference, and need no carry), only
// long rows are shared between chunks.
__global__ void chunk_coords_kernel(const u64* __restrict__ row_ptr, u64 m, u64 nnz,
                                    const u64* __restrict__ diag, const u64* __restrict__ off,
                                    u64 parts, u64 n_chunks, u64 snap_len,
                                    u64* __restrict__ out_row, u64* __restrict__ out_nnz) {
  const u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (c > n_chunks) return;
  u64 k, range_start = 0;
  bool interior = false;
  if (c == n_chunks) {
    k = diag[parts];
  } else {
    u64 lo = 0, hi = parts;  // last t with off[t] <= c
    while (lo + 1 < hi) {
      const u64 mid = lo + (hi - lo) / 2;
      if (off[mid] <= c) lo = mid; else hi = mid;
    }
    const u64 t = lo, s = c - off[t], cnt = off[t + 1] - off[t];
    const u64 items = diag[t + 1] - diag[t];
    // s < cnt <= items/chunk+1: s*items fits u64 for any realistic size
    k = diag[t] + (s * items) / cnt;
    interior = s != 0;
    range_start = diag[t];
  }
  u64 i, j;
  merge_search_dev(row_ptr, m, nnz, k, i, j);
  if (interior && i < m) {
    const u64 rs = __ldg(row_ptr + i);
    // (never back past the range's own first boundary: a merge cut may already sit in this row)
    if (j > rs && __ldg(row_ptr + i + 1) - rs < snap_len && i + rs >= range_start) j = rs;
  }
  out_row[c] = i;
  out_nnz[c] = j;
}

// Launch-order work list. The lane groups of a warp run their pieces in lockstep, so a warp
// is as slow as its longest piece: within tiles of kSortTile consecutive chunks the chunks are
// ordered by nonzero count (ties by chunk index: deterministic), so that the 32/G pieces a
// warp takes are of nearly equal length. Tiles keep the order local (X and Y locality, and
// the host pipeline's row blocks are runs of whole tiles). One CTA of kSortTile threads per
// tile, bitonic sort in shared memory.
#ifndef SPMX_SORT_TILE
#define SPMX_SORT_TILE 256
#endif
constexpr int kSortTile = SPMX_SORT_TILE;

// long_min > 0 (exact-order plans): a chunk that is exactly one row of long_min nonzeros or more
// is taken out of this list (its work item becomes an empty piece) and appended to long_rows,
// the work list of spmm_long_row_kernel.
template <typename Item, typename Long>
__global__ void __launch_bounds__(kSortTile)
work_items_kernel(const u64* __restrict__ chunk_row, const u64* __restrict__ chunk_nnz,
                  u64 n_chunks, Item* __restrict__ work, u64 long_min, Long* __restrict__ long_rows,
                  unsigned* __restrict__ long_count) {
  __shared__ u64 key[kSortTile];
  const u64 base = (u64)blockIdx.x * kSortTile;
  const u64 c = base + threadIdx.x;
  u64 k = ~0ull;  // padding sorts last
  if (c < n_chunks) {
    u64 span = chunk_nnz[c + 1] - chunk_nnz[c];
    if (long_min && span >= long_min && chunk_row[c + 1] == chunk_row[c] + 1) {
      Long lr;
      lr.row = chunk_row[c]; lr.j0 = chunk_nnz[c]; lr.j1 = chunk_nnz[c + 1];
      long_rows[atomicAdd(long_count, 1u)] = lr;
      span = 0;
    }
    k = (min(span, 0xffffffffull) << 32) | threadIdx.x;
  }
  key[threadIdx.x] = k;
  __syncthreads();
  for (int size = 2; size <= kSortTile; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const int i = threadIdx.x, j = i ^ stride;
      if (j > i) {
        const u64 a = key[i], b = key[j];
        const bool up = (i & size) == 0;
        if ((a > b) == up) { key[i] = b; key[j] = a; }
      }
      __syncthreads();
    }
  }
  const u64 slot = base + threadIdx.x;
  if (slot < n_chunks) {
    const u64 src = base + (key[threadIdx.x] & 0xffffffffull);
    Item it;
    it.r0 = chunk_row[src]; it.j0 = chunk_nnz[src];
    it.r1 = chunk_row[src + 1]; it.j1 = chunk_nnz[src + 1];
    if ((key[threadIdx.x] >> 32) == 0 && it.j1 != it.j0) { it.r1 = it.r0; it.j1 = it.j0; }  // a long row: not ours
    it.chunk = src;
    it.pad_ = 0;
    work[slot] = it;
  }
}

// Rows of long_min nonzeros or more, in no particular order (exact-order plans: these rows get
// work-list boundaries of their own and run in spmm_long_row_kernel).
__global__ void long_rows_kernel(const u64* __restrict__ row_ptr, u64 m, u64 long_min,
                                 u64* __restrict__ list, unsigned* __restrict__ count) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += stride)
    if (__ldg(row_ptr + r + 1) - __ldg(row_ptr + r) >= long_min) list[atomicAdd(count, 1u)] = r;
}

// Largest nonzero span of a chunk (the kernel keeps nonzero offsets inside a chunk in 32 bits).
__global__ void max_chunk_span_kernel(const u64* __restrict__ chunk_nnz, u64 n_chunks,
                                      u64* __restrict__ out) {
  const u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_chunks) return;
  atomicMax(out, chunk_nnz[c + 1] - chunk_nnz[c]);
}

// validate_csr, src/csr.cpp:18-42, on the device. err receives the largest code seen:
// 2 row_ptr[0] != 0, 3 row_ptr[m] != nnz, 4 row_ptr decreasing, 5 column out of range.
__global__ void validate_row_ptr_kernel(const u64* __restrict__ row_ptr, u64 m, u64 nnz, int* err) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  int e = 0;
  if (tid == 0) {
    if (row_ptr[0] != 0) e = 2;
    if (row_ptr[m] != nnz) e = max(e, 3);
  }
  for (u64 i = tid; i < m; i += stride)
    if (row_ptr[i + 1] < row_ptr[i] || row_ptr[i + 1] > nnz) e = max(e, 4);
  if (e) atomicMax(err, e);
}

__global__ void validate_cols_kernel(const unsigned* __restrict__ col, u64 count, u64 n, int* err) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  int e = 0;
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride)
    if ((u64)col[k] >= n) e = 5;
  if (e) atomicMax(err, e);
}

// next_batch, src/partition.cpp:29-33, one claim per thread on a shared device counter.
__global__ void next_batch_claims_kernel(u64* counter, u64 batch, u64 m, u64 n_claims,
                                         u64* __restrict__ out) {
  const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_claims) return;
  const u64 v = atomicAdd(counter, batch);
  if (v >= m) {
    out[2 * t] = out[2 * t + 1] = ~0ull;
  } else {
    out[2 * t] = v;
    out[2 * t + 1] = v + batch < m ? v + batch : m;
  }
}

}  // namespace spmx_dev
