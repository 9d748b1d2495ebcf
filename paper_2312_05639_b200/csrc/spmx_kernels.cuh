// spmx_kernels.cuh — sm_100a SpMM kernels (Y = A*X, CSR fp32 x dense fp32).
//
// GPU counterpart of the reference's JIT'd row kernel (src/jit.cpp:42-134): per
// output row, keep all d accumulators in registers, walk the row's nonzeros in
// CSR order, acc[j] = fma(v, X[k][j], acc[j]) with single rounding
// (src/interp.cpp:36-51 defines the bitwise result), store the row once.
//
// Mapping: a "group" of G lanes owns one output row at a time; each lane holds
// NT x VEC consecutive-column accumulators (d = 32/64/128 -> G = 8/16/32, VEC = 4,
// NT = 1: one float4 per lane). A warp holds 32/G groups and owns one "chunk" of
// the work list (spmx_plan): the contiguous piece of the merge path between two
// (row, nnz) coordinates. Rows that lie wholly inside a chunk are accumulated by
// a single group in CSR order (bitwise equal to the reference). A row cut by a
// chunk boundary leaves a partial in carry_out[chunk], added in CSR order by
// carry_fixup_kernel. Long row segments are shared by all groups of the warp and
// combined with warp shuffles.
//
// No tensor cores: the path is an irregular gather-reduce (2 flop per 4..8 bytes
// gathered), bounded by L2->SM / L1 gather bandwidth, not by math.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace spmx_dev {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kWarpsPerCta = 8;

// ---- cache-policy-aware loads/stores ---------------------------------------------------
// X rows are the only data with reuse: read-only path, default (allocating) L1 policy.
// col/val/row_ptr stream through once: evict-first. Y is written once: streaming store.
template <int VEC>
struct VecT;
template <>
struct VecT<1> {
  float v[1];
};
template <>
struct VecT<2> {
  float v[2];
};
template <>
struct VecT<4> {
  float v[4];
};

template <int VEC>
__device__ __forceinline__ VecT<VEC> ld_x(const float* p) {
  VecT<VEC> r;
  if constexpr (VEC == 4) {
    float4 t = __ldg(reinterpret_cast<const float4*>(p));
    r.v[0] = t.x; r.v[1] = t.y; r.v[2] = t.z; r.v[3] = t.w;
  } else if constexpr (VEC == 2) {
    float2 t = __ldg(reinterpret_cast<const float2*>(p));
    r.v[0] = t.x; r.v[1] = t.y;
  } else {
    r.v[0] = __ldg(p);
  }
  return r;
}

template <int VEC>
__device__ __forceinline__ void st_y(float* p, const float* a) {
  if constexpr (VEC == 4) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(a[0], a[1], a[2], a[3]));
  } else if constexpr (VEC == 2) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(a[0], a[1]));
  } else {
    __stcs(p, a[0]);
  }
}

struct SpmmArgs {
  const u64* __restrict__ row_ptr;
  const u32* __restrict__ col;
  const float* __restrict__ vals;
  const float* __restrict__ x;   // N x ldx
  float* __restrict__ y;         // M x ldx
  float* __restrict__ carry_out; // n_chunks x ldx (rows cut by a chunk end), may be null in exact mode
  const u64* __restrict__ chunk_row;  // n_chunks + 1
  const u64* __restrict__ chunk_nnz;  // n_chunks + 1
  u64 n_chunks;
  u64 m;
  int ldx;     // row stride of X, Y and carry_out in floats (= d)
  int c0;      // first column of the slab this launch computes
  int dw;      // slab width in columns (<= G*VEC*NT)
  u32 long_seg;  // row segments at least this long take the cooperative path (0 = never)
  // dynamic row dispatch (persistent CTAs claim `batch` rows at a time)
  u64* counter;
  u64 batch;
};

// One warp-synchronous accumulation step. Group g of the warp adds the next n (0..G)
// nonzeros of ITS row, starting at `cur`, into its accumulators in CSR order. n may
// differ per group; the trip count is warp-uniform (the largest n sets it) so the
// shuffles run under the full mask. Lane lg of a group fetches nonzero cur+lg
// (coalesced, streaming); column index and value are then broadcast inside the group.
template <int D_CT, int G, int VEC, int NT, bool RAGGED>
__device__ __forceinline__ void accumulate_step(const SpmmArgs& a, u64 cur, int n, int lg,
                                                float (&acc)[NT][VEC]) {
  constexpr int U = (NT >= 4) ? 2 : (NT == 2 ? 4 : 8);  // X rows in flight per lane
  const int nmax = __reduce_max_sync(kFullMask, n);
  if (nmax == 0) return;
  const int ldx = D_CT ? D_CT : a.ldx;
  const float* __restrict__ xbase = a.x + a.c0 + lg * VEC;
  u32 my_c = 0;
  float my_v = 0.0f;
  if (lg < n) {
    my_c = __ldcs(a.col + cur + lg);
    my_v = __ldcs(a.vals + cur + lg);
  }
#pragma unroll 1
  for (int t0 = 0; t0 < nmax; t0 += U) {
    u32 kk[U];
    float vv[U];
    VecT<VEC> xv[U][NT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      kk[u] = __shfl_sync(kFullMask, my_c, t0 + u, G);
      vv[u] = __shfl_sync(kFullMask, my_v, t0 + u, G);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (t0 + u < n) {
        const float* xr = xbase + (size_t)kk[u] * (size_t)ldx;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (!RAGGED || (t * G + lg) * VEC < a.dw) xv[u][t] = ld_x<VEC>(xr + t * G * VEC);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (t0 + u < n) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (!RAGGED || (t * G + lg) * VEC < a.dw) {
#pragma unroll
            for (int e = 0; e < VEC; ++e)
              acc[t][e] = __fmaf_rn(vv[u], xv[u][t].v[e], acc[t][e]);
          }
        }
      }
    }
  }
}

template <int G, int VEC, int NT, bool RAGGED>
__device__ __forceinline__ void store_row(const SpmmArgs& a, float* dst_row, int lg,
                                          const float (&acc)[NT][VEC]) {
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int c = (t * G + lg) * VEC;
    if (!RAGGED || c < a.dw) st_y<VEC>(dst_row + a.c0 + c, acc[t]);
  }
}

// Processes the piece of the merge path between (r0, j0) and (r1, j1) with one warp.
// Rows [r0, r1) end inside the piece and are stored to Y; when the piece ends in the
// middle of row r1 (has_carry) the partial sum of its nonzeros [.., j1) goes to
// carry_row. A row whose head lies in an earlier piece is stored like any other
// row; carry_fixup_kernel adds the earlier partials afterwards.
template <int D_CT, int G, int VEC, int NT, bool RAGGED>
__device__ __forceinline__ void process_piece(const SpmmArgs& a, u64 r0, u64 j0, u64 r1, u64 j1,
                                              bool has_carry, float* carry_row, int lane) {
  constexpr int NGW = 32 / G;
  const int g = lane / G, lg = lane % G;
  const int ldx = D_CT ? D_CT : a.ldx;
  const u64 row_lim = r1 + (has_carry ? 1 : 0);
  float acc[NT][VEC];

  const bool coop = (NGW > 1) && a.long_seg != 0;
  // ---- phase A: long row segments, all groups of the warp on one row ------------------
  if (coop) {
    for (u64 base = r0; base < row_lim; base += 32) {
      const u64 r = base + lane;
      u64 s = 0, e = 0;
      if (r < row_lim) {
        s = max((u64)__ldg(a.row_ptr + r), j0);
        e = min((u64)__ldg(a.row_ptr + r + 1), j1);
      }
      unsigned longmask = __ballot_sync(kFullMask, e - s >= (u64)a.long_seg);
      while (longmask) {
        const int src = __ffs(longmask) - 1;
        longmask &= longmask - 1;
        const u64 rs = __shfl_sync(kFullMask, s, src);
        const u64 re = __shfl_sync(kFullMask, e, src);
        const u64 rr = base + src;
        const u64 len = re - rs;
        u64 piece = (len + NGW - 1) / NGW;
        piece = (piece + G - 1) / G * G;
        const u64 ps = min(rs + (u64)g * piece, re);
        const u64 pe = min(ps + piece, re);
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int v = 0; v < VEC; ++v) acc[t][v] = 0.0f;
        for (u64 cur = ps; __any_sync(kFullMask, cur < pe);) {
          const int n = (int)min((u64)G, pe - cur);
          accumulate_step<D_CT, G, VEC, NT, RAGGED>(a, cur, n, lg, acc);
          cur += n;
        }
        // butterfly over the group index: fixed order, same value in every group
#pragma unroll
        for (int off = G; off < 32; off <<= 1)
#pragma unroll
          for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int v = 0; v < VEC; ++v)
              acc[t][v] += __shfl_xor_sync(kFullMask, acc[t][v], off);
        if (g == 0) {
          float* dst = (rr < r1) ? a.y + (size_t)rr * (size_t)ldx : carry_row;
          store_row<G, VEC, NT, RAGGED>(a, dst, lg, acc);
        }
      }
    }
  }

  // ---- phase B: every group walks its own rows r0+g, r0+g+NGW, ... ---------------------
  u64 r = r0 + g;
  u64 cur = 0, end = 0;
  bool have = false;  // a row is loaded and not yet stored
  for (;;) {
    // advance to the next row that still needs work (skipping rows done in phase A)
    if (!have && r < row_lim) {
      cur = max((u64)__ldg(a.row_ptr + r), j0);
      end = min((u64)__ldg(a.row_ptr + r + 1), j1);
      if (coop && end - cur >= (u64)a.long_seg) {
        r += NGW;  // done cooperatively
        cur = end = 0;
      } else {
        have = true;
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int v = 0; v < VEC; ++v) acc[t][v] = 0.0f;
      }
    }
    if (!__any_sync(kFullMask, have || r < row_lim)) break;
    const int n = have ? (int)min((u64)G, end - cur) : 0;
    accumulate_step<D_CT, G, VEC, NT, RAGGED>(a, cur, n, lg, acc);
    cur += n;
    if (have && cur == end) {
      float* dst = (r < r1) ? a.y + (size_t)r * (size_t)ldx : carry_row;
      store_row<G, VEC, NT, RAGGED>(a, dst, lg, acc);
      have = false;
      r += NGW;
    }
  }
}

// Static work list: warp w of the grid owns chunk w.
template <int D_CT, int G, int VEC, int NT, bool RAGGED>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
spmm_chunk_kernel(const SpmmArgs a) {
  const int lane = threadIdx.x & 31;
  const u64 chunk = (u64)blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (chunk >= a.n_chunks) return;
  const u64 r0 = a.chunk_row[chunk], j0 = a.chunk_nnz[chunk];
  const u64 r1 = a.chunk_row[chunk + 1], j1 = a.chunk_nnz[chunk + 1];
  const bool has_carry = (r1 < a.m) && (j1 > (u64)__ldg(a.row_ptr + r1));
  const int ldx = D_CT ? D_CT : a.ldx;
  float* carry_row = a.carry_out ? a.carry_out + (size_t)chunk * (size_t)ldx : nullptr;
  process_piece<D_CT, G, VEC, NT, RAGGED>(a, r0, j0, r1, j1, has_carry, carry_row, lane);
}

// Dynamic row dispatch (row-split only): persistent warps claim `batch` rows at a time
// from a device counter — next_batch(), src/partition.cpp:29-33; the JIT'd `lock xadd`
// driver, src/jit.cpp:106-121. One claim per warp keeps the claimed ranges disjoint and
// covering [0, m) exactly as the reference's dispatcher does.
template <int D_CT, int G, int VEC, int NT, bool RAGGED>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
spmm_dynamic_kernel(const SpmmArgs a) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    u64 v = 0;
    if (lane == 0) v = atomicAdd(a.counter, a.batch);
    v = __shfl_sync(kFullMask, v, 0);
    if (v >= a.m) return;
    const u64 hi = min(v + a.batch, a.m);
    const u64 j0 = __ldg(a.row_ptr + v), j1 = __ldg(a.row_ptr + hi);
    process_piece<D_CT, G, VEC, NT, RAGGED>(a, v, j0, hi, j1, false, nullptr, lane);
  }
}

// Adds the partial sums of rows cut by chunk boundaries, in CSR order of the pieces:
// Y[r] = carry_out[u0] + ... + carry_out[t] + (tail already stored in Y[r]).
// One CTA per chunk; only the last chunk of each chain of carries does work.
__global__ void carry_fixup_kernel(const u64* __restrict__ row_ptr,
                                   const u64* __restrict__ chunk_row,
                                   const u64* __restrict__ chunk_nnz, u64 n_chunks, u64 m,
                                   const float* __restrict__ carry_out, float* __restrict__ y,
                                   int ldx, int c0, int dw) {
  const u64 t = blockIdx.x;
  if (t + 1 >= n_chunks) return;  // the last chunk ends at (m, nnz): no carry
  const u64 r = chunk_row[t + 1];
  if (r >= m) return;
  const u64 rp = row_ptr[r];
  if (!(chunk_nnz[t + 1] > rp)) return;     // boundary t+1 is not inside row r
  if (chunk_row[t + 2] == r) return;        // chunk t+1 carries the same row on: not last
  u64 u0 = t;
  while (u0 > 0 && chunk_row[u0] == r && chunk_nnz[u0] > rp) --u0;
  for (int c = threadIdx.x; c < dw; c += blockDim.x) {
    float s = carry_out[(size_t)u0 * ldx + c0 + c];
    for (u64 u = u0 + 1; u <= t; ++u) s += carry_out[(size_t)u * ldx + c0 + c];
    float* dst = y + (size_t)r * ldx + c0 + c;
    *dst = s + *dst;
  }
}

}  // namespace spmx_dev
