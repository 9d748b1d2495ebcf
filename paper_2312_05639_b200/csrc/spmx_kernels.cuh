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

#include <type_traits>

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

template <int G, int VEC, int NT, bool RAGGED>
__device__ __forceinline__ void store_row(const SpmmArgs& a, float* dst_row, int lg,
                                          const float (&acc)[NT][VEC]) {
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int c = (t * G + lg) * VEC;
    if (!RAGGED || c < a.dw) st_y<VEC>(dst_row + a.c0 + c, acc[t]);
  }
}

template <int NT, int VEC>
__device__ __forceinline__ void zero_acc(float (&acc)[NT][VEC]) {
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[t][v] = 0.0f;
}

constexpr int kWindowRows = 128;  // rows whose bounds a warp stages at a time

#ifndef SPMX_U
#define SPMX_U 16  // LDG.128 gathers in flight per lane (measured best with 2 CTAs/SM)
#endif

// Per-warp shared memory.
template <int G>
struct WarpScratch {
  u32 row_idx[kWindowRows];  // k-th non-empty row of the window (window-local index)
  u32 row_end[kWindowRows];  // its end, as an offset from the piece's first nonzero
};

// Processes the piece of the merge path between (r0, j0) and (r1, j1) with one warp.
// Rows [r0, r1) end inside the piece and are stored to Y; when the piece ends in the
// middle of row r1 (has_carry) the partial sum of its nonzeros [.., j1) goes to
// carry_row. A row whose head lies in an earlier piece is stored like any other row;
// carry_fixup_kernel adds the earlier partials afterwards.
//
// Load phase and reduce phase are decoupled. Rows are staged kWindowRows at a time
// (bounds clipped to the piece, empty rows zeroed on the spot, the others compacted
// into shared memory). The staged rows are then consumed as a sequence of segments:
//   * a run of ordinary rows: its nonzero range is cut into 32/G contiguous sub-streams,
//     one per group of G lanes, cuts moved back to row starts, so every row is summed by
//     one group as one fmaf chain in CSR order (bitwise equal to the reference);
//   * one long row (>= long_seg nonzeros, or the row the piece ends in): cut evenly
//     between the groups, partial sums added in CSR order of the cuts by shuffles.
// A group walks its sub-stream through a rotating U-deep register pipeline: the X-row
// gather for nonzero q+U is issued as soon as nonzero q has been consumed, whatever the
// row structure. Column indices, values and the "row ends here" marks are produced a batch
// of G positions ahead (coalesced streaming loads; marks scattered through shared memory)
// and broadcast by shuffles, so the reduce step is: fma; if marked, store the row, zero.
// The piece must span fewer than 2^32 nonzeros (the plan guarantees it).
template <int D_CT, int G, int VEC, int NT, bool RAGGED>
__device__ __forceinline__ void process_piece(const SpmmArgs& a, u64 r0, u64 j0, u64 r1, u64 j1,
                                              bool has_carry, float* carry_row, int lane,
                                              WarpScratch<G>& sm) {
  constexpr int NGW = 32 / G;
  constexpr int UMAX = (SPMX_U / NT) > 0 ? (SPMX_U / NT) : 1;
  constexpr int U = UMAX < G ? UMAX : G;  // gathers in flight per lane; divides G
  const int g = lane / G, lg = lane % G;
  const int ldx = D_CT ? D_CT : a.ldx;
  const u64 row_lim = r1 + (has_carry ? 1 : 0);
  const u32* __restrict__ colp = a.col + j0;
  const float* __restrict__ valp = a.vals + j0;
  const float* __restrict__ xbase = a.x + a.c0 + lg * VEC;
  const u32 span = (u32)(j1 - j0);
  const u32 long_seg = (NGW > 1 && a.long_seg != 0) ? a.long_seg : 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  float acc[NT][VEC];

  u32 ws = 0;  // nonzero offset where the current window starts
  for (u64 wbase = r0; wbase < row_lim; wbase += kWindowRows) {
    const int nw = (int)min((u64)kWindowRows, row_lim - wbase);
    // ---- stage the window: clipped row ends, compacted over non-empty rows ----------------
    int count = 0;
    __syncwarp();
    zero_acc(acc);
#pragma unroll 1
    for (int q0 = 0; q0 < nw; q0 += 32) {
      const int li = q0 + lane;
      u32 s = 0, e = 0;
      const bool valid = li < nw;
      if (valid) {
        const u64 lo = __ldg(a.row_ptr + wbase + li), hi = __ldg(a.row_ptr + wbase + li + 1);
        s = lo > j0 ? (u32)min(lo - j0, (u64)span) : 0u;
        e = hi > j0 ? (u32)min(hi - j0, (u64)span) : 0u;
      }
      const unsigned ne = __ballot_sync(kFullMask, valid && e != s);
      if (valid && e != s) {
        const int pos = count + __popc(ne & lt_mask);
        sm.row_idx[pos] = (u32)li;
        sm.row_end[pos] = e;
      }
      count += __popc(ne);
      // empty rows: zeros, NGW rows per store instruction
      unsigned em = __ballot_sync(kFullMask, valid && e == s);
      while (em) {
        int src = -1;
#pragma unroll
        for (int q = 0; q < NGW; ++q) {
          const int bit = em ? __ffs(em) - 1 : -1;
          if (q == g) src = bit;
          if (em) em &= em - 1;
        }
        if (src >= 0) {
          const u64 rr = wbase + q0 + src;
          float* dst = (rr < r1) ? a.y + (size_t)rr * (size_t)ldx : carry_row;
          store_row<G, VEC, NT, RAGGED>(a, dst, lg, acc);
        }
      }
    }
    __syncwarp();
    if (count == 0) continue;
    const u32 we = sm.row_end[count - 1];
    float* __restrict__ ybase = a.y + (size_t)wbase * (size_t)ldx;

    // ---- which staged rows are "long" (shared by all groups) ------------------------------
    unsigned longm[kWindowRows / 32];
#pragma unroll
    for (int q = 0; q < kWindowRows / 32; ++q) {
      const int kk = q * 32 + lane;
      bool is_long = false;
      if (kk < count) {
        const u32 rs = kk > 0 ? sm.row_end[kk - 1] : ws;
        is_long = (sm.row_end[kk] - rs >= long_seg) ||
                  (has_carry && wbase + sm.row_idx[kk] == r1);
      }
      longm[q] = __ballot_sync(kFullMask, is_long);
    }

    // ---- consume the window as segments: [run of ordinary rows] [long row] ... --------------
    int seg_k = 0;
    for (;;) {
      // next long row at or after seg_k
      int kl = count;
#pragma unroll
      for (int q = kWindowRows / 32 - 1; q >= 0; --q) {
        unsigned mq = longm[q];
        if (seg_k > q * 32) mq = (seg_k >= (q + 1) * 32) ? 0u : (mq & ~((1u << (seg_k - q * 32)) - 1u));
        if (mq) kl = q * 32 + __ffs(mq) - 1;
      }
      bool is_long_seg;
      int ka, kb;  // rows [ka, kb) of this segment
      if (seg_k < kl) { is_long_seg = false; ka = seg_k; kb = kl; }
      else if (kl < count) { is_long_seg = true; ka = kl; kb = kl + 1; }
      else break;
      seg_k = kb;

      const u32 sa = ka > 0 ? sm.row_end[ka - 1] : ws;
      const u32 sb = sm.row_end[kb - 1];
      // ---- cut [sa, sb) into NGW sub-streams ------------------------------------------------
      u32 p0 = sa, pe = sb;
      int k0 = ka, k1 = kb;  // rows of this group (ordinary segment)
      if constexpr (NGW > 1) {
        const u32 len = sb - sa;
        const u32 q = (len + NGW - 1) / NGW;
        u32 cut[2];
        int kcut[2];
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          const int gg = g + side;
          u32 bnd = sa + min((u32)gg * q, len);
          int kk = gg >= NGW ? kb : ka;
          if (!is_long_seg && gg > 0 && gg < NGW) {
            int lo = ka, hi = kb;  // first row with end > bnd
            while (lo < hi) {
              const int mid_i = (lo + hi) >> 1;
              if (sm.row_end[mid_i] > bnd) hi = mid_i; else lo = mid_i + 1;
            }
            kk = lo;
            bnd = kk < kb ? (kk > ka ? sm.row_end[kk - 1] : sa) : sb;  // back to the row start
          }
          cut[side] = bnd;
          kcut[side] = kk;
        }
        p0 = cut[0];
        pe = cut[1];
        k0 = kcut[0];
        k1 = kcut[1];
      }
      const u32 L = pe - p0;  // this group's sub-stream length
      const u32 Lmax = __reduce_max_sync(kFullMask, L);
      int k = k0;  // current row of this group
      // nonzeros left in the current row; a long row's end is handled after the loop
      u32 left = (!is_long_seg && L > 0) ? sm.row_end[k] - p0 : 0x7fffffffu;

      u32 c0 = 0, c1 = 0;
      float v0 = 0.0f, v1 = 0.0f;
      if ((u32)lg < L) { c0 = __ldcs(colp + p0 + lg); v0 = __ldcs(valp + p0 + lg); }
      if ((u32)(G + lg) < L) { c1 = __ldcs(colp + p0 + G + lg); v1 = __ldcs(valp + p0 + G + lg); }
      VecT<VEC> xv[U][NT];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const u32 kq = __shfl_sync(kFullMask, c0, u, G);
        if ((u32)u < L) {
          const float* xr = xbase + (size_t)kq * (size_t)ldx;
#pragma unroll
          for (int t = 0; t < NT; ++t)
            if (!RAGGED || (t * G + lg) * VEC < a.dw) xv[u][t] = ld_x<VEC>(xr + t * G * VEC);
        }
      }
#pragma unroll 1
      for (u32 nb = 0; nb < Lmax; nb += G) {
        u32 c2 = 0;
        float v2 = 0.0f;
        if (nb + 2 * G + lg < L) {
          c2 = __ldcs(colp + p0 + nb + 2 * G + lg);
          v2 = __ldcs(valp + p0 + nb + 2 * G + lg);
        }
#pragma unroll
        for (int t = 0; t < G; ++t) {
          const int u = t % U;
          const float vq = __shfl_sync(kFullMask, v0, t, G);
          const u32 kq = (t + U < G) ? __shfl_sync(kFullMask, c0, t + U, G)
                                     : __shfl_sync(kFullMask, c1, t + U - G, G);
          if (nb + t < L) {
#pragma unroll
            for (int tt = 0; tt < NT; ++tt)
              if (!RAGGED || (tt * G + lg) * VEC < a.dw) {
#pragma unroll
                for (int e = 0; e < VEC; ++e)
                  acc[tt][e] = __fmaf_rn(vq, xv[u][tt].v[e], acc[tt][e]);
              }
          }
#ifdef SPMX_EXP_NOROWEND
          if (false) {
#else
          if (--left == 0) {  // row k ends here: store it, start the next one
#endif
#ifndef SPMX_EXP_NOSTORE
            store_row<G, VEC, NT, RAGGED>(a, ybase + (size_t)sm.row_idx[k] * (size_t)ldx, lg, acc);
#endif
            zero_acc(acc);
            ++k;
            left = (k < k1) ? sm.row_end[k] - sm.row_end[k - 1] : 0x7fffffffu;
          }
          if (nb + t + U < L) {
            const float* xr = xbase + (size_t)kq * (size_t)ldx;
#pragma unroll
            for (int tt = 0; tt < NT; ++tt)
              if (!RAGGED || (tt * G + lg) * VEC < a.dw) xv[u][tt] = ld_x<VEC>(xr + tt * G * VEC);
          }
        }
        c0 = c1; v0 = v1;
        c1 = c2; v1 = v2;
      }

      if (is_long_seg) {  // add the groups' partial sums in CSR order of the cuts, store once
        if constexpr (NGW > 1) {
          float tot[NT][VEC];
#pragma unroll
          for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              float sacc = __shfl_sync(kFullMask, acc[t][e], lg);
#pragma unroll
              for (int gg = 1; gg < NGW; ++gg) sacc += __shfl_sync(kFullMask, acc[t][e], gg * G + lg);
              tot[t][e] = sacc;
            }
#pragma unroll
          for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[t][e] = tot[t][e];
        }
        if (g == 0) {
          const u64 rr = wbase + sm.row_idx[ka];
          float* dst = (rr < r1) ? a.y + (size_t)rr * (size_t)ldx : carry_row;
          store_row<G, VEC, NT, RAGGED>(a, dst, lg, acc);
        }
        zero_acc(acc);
      }
    }
    ws = we;
  }
}

#ifndef SPMX_MIN_CTAS
#define SPMX_MIN_CTAS 2
#endif

// Static work list: warp w of the grid owns chunk w.
template <int D_CT, int G, int VEC, int NT, bool RAGGED>
__global__ void __launch_bounds__(kWarpsPerCta * 32, (NT <= 2 ? SPMX_MIN_CTAS : 1))
spmm_chunk_kernel(const SpmmArgs a) {
  __shared__ WarpScratch<G> scratch[kWarpsPerCta];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const u64 chunk = (u64)blockIdx.x * kWarpsPerCta + w;
  if (chunk >= a.n_chunks) return;
  const u64 r0 = a.chunk_row[chunk], j0 = a.chunk_nnz[chunk];
  const u64 r1 = a.chunk_row[chunk + 1], j1 = a.chunk_nnz[chunk + 1];
  const bool has_carry = (r1 < a.m) && (j1 > (u64)__ldg(a.row_ptr + r1));
  const int ldx = D_CT ? D_CT : a.ldx;
  float* carry_row = a.carry_out ? a.carry_out + (size_t)chunk * (size_t)ldx : nullptr;
  process_piece<D_CT, G, VEC, NT, RAGGED>(a, r0, j0, r1, j1, has_carry, carry_row, lane,
                                          scratch[w]);
}

// Dynamic row dispatch (row-split only): persistent warps claim `batch` rows at a time
// from a device counter — next_batch(), src/partition.cpp:29-33; the JIT'd `lock xadd`
// driver, src/jit.cpp:106-121. One claim per warp keeps the claimed ranges disjoint and
// covering [0, m) exactly as the reference's dispatcher does.
template <int D_CT, int G, int VEC, int NT, bool RAGGED>
__global__ void __launch_bounds__(kWarpsPerCta * 32, (NT <= 2 ? SPMX_MIN_CTAS : 1))
spmm_dynamic_kernel(const SpmmArgs a) {
  __shared__ WarpScratch<G> scratch[kWarpsPerCta];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (;;) {
    u64 v = 0;
    if (lane == 0) v = atomicAdd(a.counter, a.batch);
    v = __shfl_sync(kFullMask, v, 0);
    if (v >= a.m) return;
    const u64 hi = min(v + a.batch, a.m);
    const u64 j0 = __ldg(a.row_ptr + v), j1 = __ldg(a.row_ptr + hi);
    process_piece<D_CT, G, VEC, NT, RAGGED>(a, v, j0, hi, j1, false, nullptr, lane, scratch[w]);
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

// spmm_reference (src/reference.cpp:10-25, Alg. 1) for RunConfig.verify: one thread per
// output element, ret += v * x with separate multiply and add (two roundings), CSR order.
__global__ void spmm_unfused_reference_kernel(const u64* __restrict__ row_ptr,
                                              const u32* __restrict__ col,
                                              const float* __restrict__ vals,
                                              const float* __restrict__ x, float* __restrict__ y,
                                              u64 m, int d) {
  const u64 idx = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= m * (u64)d) return;
  const u64 i = idx / (u64)d;
  const int j = (int)(idx % (u64)d);
  float ret = 0.0f;
  for (u64 k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
    ret = __fadd_rn(ret, __fmul_rn(vals[k], x[(size_t)col[k] * d + j]));
  y[idx] = ret;
}

// max_relative_error (src/executor.cpp:27-34). The maximum of non-negative doubles is taken
// with an integer atomicMax on the bit pattern (order-preserving for non-negative values).
__global__ void max_rel_err_kernel(const float* __restrict__ y, const float* __restrict__ ref,
                                   u64 count, unsigned long long* out_bits) {
  double worst = 0.0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (u64)gridDim.x * blockDim.x) {
    const double r = (double)ref[i];
    const double denom = fmax(fabs(r), 1e-6);
    const double e = fabs((double)y[i] - r) / denom;
    worst = (e > worst || e != e) ? e : worst;
  }
  if (worst != worst) worst = __longlong_as_double(0x7ff0000000000000ll);  // NaN -> +inf
  atomicMax(out_bits, (unsigned long long)__double_as_longlong(worst));
}

}  // namespace spmx_dev
