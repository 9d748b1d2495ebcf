// spmx_kernels.cuh — sm_100a SpMM kernels (Y = A*X, CSR fp32 x dense fp32).
//
// GPU counterpart of the reference's JIT'd row kernel (src/jit.cpp:42-134): per
// output row, keep all d accumulators in registers, walk the row's nonzeros in
// CSR order, acc[j] = fma(v, X[k][j], acc[j]) with single rounding
// (src/interp.cpp:36-51 defines the bitwise result), store the row once.
//
// Mapping: a "group" of G lanes owns one "chunk" of the work list (spmx_plan) — the
// contiguous piece of the merge path between two (row, nnz) coordinates — and one output
// row at a time; each lane holds NT x VEC consecutive-column accumulators. G = 8 wherever a row
// can be spread over eight lanes (d = 8 -> VEC = 1; d = 16 -> VEC = 2; d = 32 -> VEC = 4;
// d = 64 -> NT = 2 float4 tiles; d = 128 -> NT = 4; see spmx_jit::choose_shape). The
// 32/G groups of a warp run the same instruction stream on different chunks. Rows that lie
// wholly inside a chunk are accumulated by a single group in CSR order (bitwise equal to
// the reference). A row cut by a chunk boundary leaves a partial in carry_out[chunk];
// carry_fixup_kernel adds the partials in an order fixed by the plan.
//
// No tensor cores: the path is an irregular gather-reduce (2 flop per 4..8 bytes
// gathered), bounded by L2->SM / L1 gather bandwidth, not by math.
#pragma once

#ifndef __CUDACC_RTC__  // NVRTC (runtime per-d instantiation) has the CUDA builtins predeclared
#include <cuda_runtime.h>
#include <stdint.h>
#endif

namespace spmx_dev {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr unsigned kFullMask = 0xffffffffu;

// Bounds self-check build (-DSPMX_DEBUG_BOUNDS=1, tools/bounds_check.py): compute-sanitizer is not
// available on the GPU pool, so every global and shared access of the SpMM kernels is checked
// against the extents passed in SpmmArgs and violations are counted per site. Off by default:
// the checks cost instructions in the hot loop.
#ifndef SPMX_DEBUG_BOUNDS
#define SPMX_DEBUG_BOUNDS 0
#endif
#if SPMX_DEBUG_BOUNDS
__device__ unsigned long long g_bounds_violations[16];
#define SPMX_CHECK(cond, site) do { if (!(cond)) atomicAdd(&g_bounds_violations[site], 1ull); } while (0)
#else
#define SPMX_CHECK(cond, site) do { } while (0)
#endif
#ifndef SPMX_WARPS_PER_CTA
#define SPMX_WARPS_PER_CTA 2  // small CTAs: a finished warp frees its slot at once (measured best)
#endif
constexpr int kWarpsPerCta = SPMX_WARPS_PER_CTA;

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
struct alignas(8) VecT<2> {
  float v[2];
};
template <>
struct alignas(16) VecT<4> {
  float v[4];
};

// Optional L2 eviction policies (createpolicy): evict_last for X rows, evict_first for the
// col/val stream and Y. Measured on c2/c3: no effect (X's L2 misses are not caused by the
// streams), so they are compiled out by default; -DSPMX_POL_X=1 etc. re-enable them.
#ifndef SPMX_POL_X
#define SPMX_POL_X 0
#endif
#ifndef SPMX_POL_STREAM
#define SPMX_POL_STREAM 0
#endif
#ifndef SPMX_POL_Y
#define SPMX_POL_Y 0
#endif
__device__ __forceinline__ u64 policy_evict_first() {
  u64 p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ u64 policy_evict_last() {
  u64 p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

template <int VEC>
__device__ __forceinline__ VecT<VEC> ld_x(const float* p, u64 pol) {
  VecT<VEC> r;
#if SPMX_POL_X
  if constexpr (VEC == 4) {
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
                 : "l"(p), "l"(pol));
  } else if constexpr (VEC == 2) {
    asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
                 : "=f"(r.v[0]), "=f"(r.v[1])
                 : "l"(p), "l"(pol));
  } else {
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r.v[0]) : "l"(p), "l"(pol));
  }
#else
  if constexpr (VEC == 4) {
    float4 t = __ldg(reinterpret_cast<const float4*>(p));
    r.v[0] = t.x; r.v[1] = t.y; r.v[2] = t.z; r.v[3] = t.w;
  } else if constexpr (VEC == 2) {
    float2 t = __ldg(reinterpret_cast<const float2*>(p));
    r.v[0] = t.x; r.v[1] = t.y;
  } else {
    r.v[0] = __ldg(p);
  }
#endif
  return r;
}

// software prefetch of the col/val stream (a line = 32 positions)
#ifndef SPMX_PF_STREAM
#define SPMX_PF_STREAM 0  // 0 off, 1 prefetch.global.L2, 2 prefetch.global.L1
#endif
#ifndef SPMX_PF_DIST
#define SPMX_PF_DIST 64  // positions ahead of the newest col/val batch
#endif
__device__ __forceinline__ void pf_stream(const void* p) {
#if SPMX_PF_STREAM == 1
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#elif SPMX_PF_STREAM == 2
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#endif
}

// streaming loads of the CSR arrays
__device__ __forceinline__ u32 ld_stream(const u32* p, u64 pol) {
#if SPMX_POL_STREAM
  u32 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
#else
  return __ldcs(p);
#endif
}
__device__ __forceinline__ float ld_stream(const float* p, u64 pol) {
#if SPMX_POL_STREAM
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
#else
  return __ldcs(p);
#endif
}

template <int VEC>
__device__ __forceinline__ void st_y(float* p, const float* a, u64 pol) {
#if SPMX_POL_Y
  if constexpr (VEC == 4) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(a[0]), "f"(a[1]),
                 "f"(a[2]), "f"(a[3]), "l"(pol)
                 : "memory");
  } else if constexpr (VEC == 2) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1,%2}, %3;" ::"l"(p), "f"(a[0]), "f"(a[1]), "l"(pol)
                 : "memory");
  } else {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(a[0]), "l"(pol) : "memory");
  }
#else
  if constexpr (VEC == 4) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(a[0], a[1], a[2], a[3]));
  } else if constexpr (VEC == 2) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(a[0], a[1]));
  } else {
    __stcs(p, a[0]);
  }
#endif
}

// One entry of the launch-order work list: chunk `chunk` of the plan, i.e. the piece of the
// merge path between (r0, j0) and (r1, j1).
struct alignas(16) WorkItem {
  u64 r0, j0, r1, j1;
  u64 chunk;
  u64 pad_;
};

struct SpmmArgs {
  const u64* __restrict__ row_ptr;
  const u32* __restrict__ col;
  const float* __restrict__ vals;
  const float* __restrict__ x;   // N x ldx
  float* __restrict__ y;         // M x ldx
  float* __restrict__ carry_out; // n_chunks x ldx (rows cut by a chunk end), may be null in exact mode
  const WorkItem* __restrict__ work;  // n_chunks work items in launch order (see work_items_kernel)
  u64 n_chunks;     // size of the whole work list
  u64 chunk_begin;  // this launch processes chunks [chunk_begin, chunk_end)
  u64 chunk_end;
  const int* abort_flag;  // when non-null and set (invalid input found on the device): do nothing
  u64 m;
  u64 n_x, nnz;  // rows of X and nonzeros of A (read by the bounds self-check build only)
  int ldx;     // row stride of X, Y and carry_out in floats (= d)
  int c0;      // first column of the slab this launch computes
  int dw;      // slab width in columns (<= G*VEC*NT)
  // dynamic row dispatch (persistent CTAs claim `batch` rows at a time)
  u64* counter;
  u64 batch;
};

// acc[e] = fma(v, x[e], acc[e]) with one rounding per element (src/interp.cpp:43). Blackwell's
// packed FFMA2 (fma.rn.f32x2: two independent IEEE fp32 FMAs per instruction, bitwise equal
// to two scalar FMAs) halves the instruction count of the reduce step.
#ifndef SPMX_FFMA2
#define SPMX_FFMA2 1
#endif
__device__ __forceinline__ void fma2(float v, float x0, float x1, float& a0, float& a1) {
#if SPMX_FFMA2
  unsigned long long vv, xx, aa;
  asm("mov.b64 %0, {%1, %1};" : "=l"(vv) : "f"(v));
  asm("mov.b64 %0, {%1, %2};" : "=l"(xx) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(aa) : "f"(a0), "f"(a1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(aa) : "l"(vv), "l"(xx));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(aa));
#else
  a0 = __fmaf_rn(v, x0, a0);
  a1 = __fmaf_rn(v, x1, a1);
#endif
}
template <int VEC, bool PACK>
__device__ __forceinline__ void fma_tile(float v, const VecT<VEC>& x, float (&acc)[VEC]) {
  if constexpr (!PACK) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = __fmaf_rn(v, x.v[e], acc[e]);
  } else if constexpr (VEC == 4) {
    fma2(v, x.v[0], x.v[1], acc[0], acc[1]);
    fma2(v, x.v[2], x.v[3], acc[2], acc[3]);
  } else if constexpr (VEC == 2) {
    fma2(v, x.v[0], x.v[1], acc[0], acc[1]);
  } else {
    acc[0] = __fmaf_rn(v, x.v[0], acc[0]);
  }
}

template <int NT, int VEC>
__device__ __forceinline__ void zero_acc(float (&acc)[NT][VEC]) {
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[t][v] = 0.0f;
}
// The same inside the row-end branch, from a register that holds zero: ptxas otherwise
// materialises every constant zero there through a uniform register (two instructions per
// accumulator).
template <int NT, int VEC>
__device__ __forceinline__ void zero_acc_from(float (&acc)[NT][VEC], float zero) {
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[t][v] = zero;
}

#ifndef SPMX_U
#define SPMX_U 16  // LDG.128 gathers in flight per lane (measured best with 2 CTAs/SM)
#endif
#ifndef SPMX_MIN_CTAS
#define SPMX_MIN_CTAS 2
#endif
#ifndef SPMX_STAGE_BATCH
#define SPMX_STAGE_BATCH 4  // row_ptr loads in flight per lane while staging row bounds
#endif
constexpr int kStageBatch = SPMX_STAGE_BATCH;

// Per-shape tuning (measured on B200, tools/dev_bench.py): CTAs per SM the register budget is
// set for, and row gathers in flight per lane.
//   8 lanes x 1 tile  (d = 8, 16, 32 and every width of 5..8 vectors): one load per position and
//                     lane, so more resident warps (24 per SM) and a pipeline as deep as a batch;
//   8 lanes x 2..4 tiles (d = 64, 128, 33..128 in general): 16 loads in flight per lane, 16 warps;
//   wider groups / more tiles (runtime-d slabs): as measured in round 1.
template <int D_CT, int G, int NT>
struct Tune {
#ifdef SPMX_MIN_CTAS_RAW
  static constexpr int kMinCtas = SPMX_MIN_CTAS_RAW;
#else
  static constexpr int kMinCtas =
      ((G == 8 && NT == 1) ? 3 : (NT <= 2 || (G == 8 && NT <= 4)) ? SPMX_MIN_CTAS : 1) * (8 / kWarpsPerCta);
#endif
  static constexpr int kInFlight = (G == 8 && NT == 1) ? 8 : SPMX_U;
};

__host__ __device__ constexpr int pipeline_depth(int want, int g) {
  int u = 1;
  while (u * 2 <= want && u * 2 <= g) u *= 2;
  return u;
}

#ifndef SPMX_REFILL_FIRST
#define SPMX_REFILL_FIRST (-1)  // -1: per width
#endif
#ifndef SPMX_EARLY_FILL
#define SPMX_EARLY_FILL 1
#endif
#ifndef SPMX_SHFL_AHEAD
#define SPMX_SHFL_AHEAD 1
#endif
#ifndef SPMX_WINDOW_ROWS
#define SPMX_WINDOW_ROWS 64
#endif
// Non-empty rows one group stages at a time (shared memory: 8 bytes per record and group).
template <int G>
struct Window {
  static constexpr int NGW = 32 / G;
  static constexpr int kRows = (512 / NGW) > SPMX_WINDOW_ROWS ? SPMX_WINDOW_ROWS : (512 / NGW);
};

// Per-warp shared memory: one region per group. One record per non-empty row of the window:
// x = end of the row (offset from the piece's first nonzero, clipped to the piece), y = its
// window-local row index (kCarryIdx for the row the piece ends in: its partial goes to carry_out).
constexpr u32 kCarryIdx = 0xffffffffu;
// Column indices and values reach the lanes of a group through shared memory where a group is
// 8 lanes and the gather pipeline is as deep as a batch (U == G: d = 32 and 64): every lane
// publishes the pair (column of position t + U, value of position t) of its position once per
// batch, and each position is one LDS.64 — half the instructions and L1 data-pipe wavefronts
// of two shuffles per position (shuffles go through the same pipe as the gathers: at d = 32
// they were a third of its load). With U < G (d = 128) the column belongs to a gather issued
// G - U positions later; the variant with that column queue ran 6 % slower (registers), so
// those kernels keep the shuffles.
#ifndef SPMX_SMEM_BCAST
#define SPMX_SMEM_BCAST 1
#endif
template <int G>
struct WarpScratch {
  uint2 rec[Window<G>::NGW][Window<G>::kRows + 2];  // + the two records read ahead at a row end
  uint2 bc[2][G][Window<G>::NGW];  // [batch parity][position][group]: conflict-free both ways
};

// One piece of the merge path per GROUP of G lanes: the nonzeros and row ends between the
// coordinates (r0, j0) and (r1, j1). Rows [r0, r1) end inside the piece and are stored to Y;
// when the piece ends in the middle of row r1 (r1 < m) the partial sum of that row's
// nonzeros [.., j1) goes to carry_row. A row whose head lies in an earlier piece is stored
// like any other row; carry_fixup_kernel adds the earlier partials afterwards, in CSR order.
// The 32/G groups of a warp run the same instruction stream on different pieces (all loop
// trip counts are made warp-uniform; pieces hold the same number of merge items, so the
// groups finish together).
//
// Load phase and reduce phase are decoupled. A group stages the bounds of its next rows
// (clipped to the piece) in shared memory — empty rows are zeroed on the spot, the others
// compacted — and then streams the nonzeros of those rows through a rotating U-deep register
// pipeline: the X-row gather for nonzero q+U is issued as soon as nonzero q has been
// consumed, whatever the row structure. Column indices and values are fetched a batch of G
// positions ahead (coalesced streaming loads) and broadcast inside the group by shuffles.
// The reduce step is acc = fmaf(v, x, acc) plus a countdown to the row end; at a row end the
// row is stored and the accumulators are zeroed. Every row that lies wholly inside a piece
// is therefore ONE fmaf chain in CSR order: bitwise equal to the reference.
// A piece must span fewer than 2^32 nonzeros (the plan guarantees it).
// Does tile t of lane lg hold columns of the slab? Always, unless the slab is narrower than
// G * NT * VEC (RAGGED). With a compile-time width the test folds away for every tile that lies
// wholly inside (or outside) the row: only the one tile the row ends in keeps a lane predicate.
template <int D_CT, int G, int VEC, bool RAGGED>
__device__ __forceinline__ bool tile_on(const SpmmArgs& a, int t, int lg) {
  if constexpr (!RAGGED) {
    return true;
  } else if constexpr (D_CT > 0) {
    if ((t * G + G - 1) * VEC < D_CT) return true;
    if (t * G * VEC >= D_CT) return false;
    return (t * G + lg) * VEC < D_CT;
  } else {
    return (t * G + lg) * VEC < a.dw;
  }
}

template <int D_CT, int G, int VEC, int NT, bool RAGGED>
__device__ __forceinline__ void store_lane(const SpmmArgs& a, float* dst_lane, int lg,
                                           const float (&acc)[NT][VEC], u64 pol) {
#pragma unroll
  for (int t = 0; t < NT; ++t)
    if (tile_on<D_CT, G, VEC, RAGGED>(a, t, lg)) st_y<VEC>(dst_lane + t * G * VEC, acc[t], pol);
}

template <int D_CT, int G, int VEC, int NT, bool RAGGED>
__device__ __forceinline__ void process_piece(const SpmmArgs& a, bool active, u64 r0, u64 j0,
                                              u64 r1, u64 j1, float* carry_row,
                                              int lane, WarpScratch<G>& sm) {
  constexpr int W = Window<G>::kRows;  // staged records (non-empty rows) per window
  constexpr int kScan = 512;           // rows scanned per window
  // packed FFMA2 where it was measured not to lose (three and six tiles per lane run 6-12 %
  // slower with it: d = 96 465 vs 522 us, d = 192 873 vs 925 us; four tiles 5 % faster)
  constexpr bool kPackFma = (NT == 1 || NT == 2 || NT == 4);
  constexpr bool kRefillFirst = SPMX_REFILL_FIRST >= 0 ? (SPMX_REFILL_FIRST != 0) : (NT <= 2);
  // positions in flight per lane: the largest power of two with U * NT <= kInFlight, at most G
  // (so that U divides G and a position keeps its pipeline slot from batch to batch)
  constexpr int U = pipeline_depth(Tune<D_CT, G, NT>::kInFlight / NT, G);
  const int g = lane / G, lg = lane % G;
  const int ldx = D_CT ? D_CT : a.ldx;
  // row r1 is staged too: clipped to the piece it is empty unless the piece ends inside it
  const u64 row_lim = active ? r1 + (r1 < a.m ? 1 : 0) : r0;
  const u32* __restrict__ colp = a.col + j0;
  const float* __restrict__ valp = a.vals + j0;
  const int lane_col = (D_CT ? 0 : a.c0) + lg * VEC;  // first column this lane owns
  const float* __restrict__ xbase = a.x + lane_col;
  float* const carry_lane = carry_row ? carry_row + lane_col : nullptr;
  const u32 span = active ? (u32)(j1 - j0) : 0u;
  const unsigned grp_mask = (G == 32) ? kFullMask : (((1u << G) - 1u) << (g * G));
  const unsigned lt_mask = grp_mask & ((1u << lane) - 1u);
  uint2* __restrict__ s_rec = sm.rec[g];
  float acc[NT][VEC];
  const float zero_f = __int_as_float(a.dw >> 31);  // 0.0f (dw >= 0), opaque to the compiler
  const u64 pol_first = policy_evict_first(), pol_last = policy_evict_last();

  // A piece without nonzeros that ends inside row r1 (duplicate diagonals: more parts than
  // merge items) still owns a slot of that row's carry chain: its partial is zero. Without
  // this store carry_fixup_kernel would add whatever the buffer held before.
  if (carry_lane != nullptr && active && span == 0u && r1 < a.m) {
    float z[NT][VEC];
    zero_acc(z);
    store_lane<D_CT, G, VEC, NT, RAGGED>(a, carry_lane, lg, z, pol_first);
  }

  u32 ws = 0;  // nonzero offset where the current window starts
  int adv = 0;  // rows the previous window covered
  for (u64 wbase = r0; __any_sync(kFullMask, wbase < row_lim); wbase += adv) {
    // A window holds at most W non-empty rows (the staged records) out of at most kScan rows:
    // it ends where the rows of the piece end, or where the records run out.
    const int nw = wbase < row_lim ? (int)min((u64)kScan, row_lim - wbase) : 0;
    float* const ywin = a.y + (size_t)wbase * (size_t)ldx + lane_col;  // this lane's columns of row wbase
    // The window's first two column/value batches and its first U gathers do not depend on the
    // row bounds: they are issued first, so that the row_ptr loads, the staging below and the
    // gather round trip overlap.
    const u32 p0 = ws;
    u32 c0 = 0, c1 = 0;
    float v0 = 0.0f, v1 = 0.0f;
    if (p0 + lg < span) { SPMX_CHECK(j0 + p0 + lg < a.nnz, 0); c0 = ld_stream(colp + p0 + lg, pol_first); v0 = ld_stream(valp + p0 + lg, pol_first); }
    if (p0 + G + lg < span) { SPMX_CHECK(j0 + p0 + G + lg < a.nnz, 0); c1 = ld_stream(colp + p0 + G + lg, pol_first); v1 = ld_stream(valp + p0 + G + lg, pol_first); }
#if SPMX_PF_STREAM
    {  // the lines that hold positions [p0 + 2G, p0 + 2G + SPMX_PF_DIST): one line per lane and array
      const u32 q = p0 + 2 * G + 32 * (u32)lg;
      if (32 * lg < SPMX_PF_DIST && q < span) { pf_stream(colp + q); pf_stream(valp + q); }
    }
#endif
    const int nw_max = __reduce_max_sync(kFullMask, nw);
    u32 eb[kStageBatch];
    auto load_bounds = [&](int qb) {
#pragma unroll
      for (int i = 0; i < kStageBatch; ++i) {
        const int li = qb + i * G + lg;
        eb[i] = 0;
        if (li < nw) {
          SPMX_CHECK(wbase + li + 1 <= a.m, 2);
          const u64 hi = __ldg(a.row_ptr + wbase + li + 1);
          eb[i] = hi > j0 ? (u32)min(hi - j0, (u64)span) : 0u;
        }
      }
    };
    load_bounds(0);
    VecT<VEC> xv[U][NT];
    auto fill = [&]() {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const u32 kq = __shfl_sync(kFullMask, c0, u, G);
        if (p0 + (u32)u < span) {
          SPMX_CHECK((u64)kq < a.n_x, 3);
          const float* xr = xbase + (size_t)kq * (size_t)ldx;
#pragma unroll
          for (int t = 0; t < NT; ++t)
            if (tile_on<D_CT, G, VEC, RAGGED>(a, t, lg)) xv[u][t] = ld_x<VEC>(xr + t * G * VEC, pol_last);
        }
      }
    };
    if (SPMX_EARLY_FILL) fill();
    // ---- stage the window: clipped row ends, compacted over non-empty rows ----------------
    // Row ends are loaded kStageBatch * G rows at a time (all loads of a batch in flight
    // together); a row starts where the previous one ends.
    int count = 0;
    u32 prev_e = ws;
    bool open = true;  // group-uniform: the record buffer still has room for G more rows
    adv = nw;
    __syncwarp();
    zero_acc(acc);
#pragma unroll 1
    for (int qb = 0; qb < nw_max; qb += kStageBatch * G) {
      if (qb > 0) {
        if (!__any_sync(kFullMask, open && qb < nw)) break;
        load_bounds(qb);
      }
#pragma unroll
      for (int i = 0; i < kStageBatch; ++i) {
        const int q0 = qb + i * G;
        if (q0 >= nw_max) break;  // warp-uniform
        if (open && q0 < nw && count + G > W) {  // out of records: the window ends before row q0
          open = false;
          adv = q0;
        }
        const int li = q0 + lg;
        const bool valid = open && li < nw;
        const u32 e = eb[i];
        const u32 up = __shfl_up_sync(kFullMask, e, 1, G);
        const u32 s = lg == 0 ? prev_e : up;
        prev_e = __shfl_sync(kFullMask, e, G - 1, G);
        const unsigned ne = __ballot_sync(kFullMask, valid && e != s) & grp_mask;
        SPMX_CHECK(!(valid && e != s) || count + __popc(ne & lt_mask) < W, 5);
        if (valid && e != s)
          s_rec[count + __popc(ne & lt_mask)] = make_uint2(e, wbase + li < r1 ? (u32)li : kCarryIdx);
        count += __popc(ne);
        // empty rows that end inside the piece: the whole group writes one row of zeros at a time
        unsigned em = __ballot_sync(kFullMask, valid && e == s && wbase + li < r1) & grp_mask;
        while (em) {
          const int src = (__ffs(em) - 1) - g * G;
          em &= em - 1;
          SPMX_CHECK(wbase + q0 + src < a.m, 8);
          store_lane<D_CT, G, VEC, NT, RAGGED>(a, ywin + (size_t)(q0 + src) * (size_t)ldx, lg, acc, pol_first);
        }
      }
    }
    __syncwarp();
    const u32 we = count > 0 ? s_rec[count - 1].x : ws;
    const u32 L = we - ws;  // nonzeros of this window in this group's piece
    const u32 Lmax = __reduce_max_sync(kFullMask, L);
    if (Lmax == 0) continue;  // warp-uniform
    if (!SPMX_EARLY_FILL) fill();
    int k = 0;  // current row = k-th non-empty row of the window
    // the record of the current row and of the one after it are kept in registers, so that a
    // row end costs no shared-memory round trip
    uint2 cur = s_rec[0], nxt = s_rec[1];
    // position (relative to the current batch) of the last nonzero of the current row
    constexpr int kNoRowEnd = 0x3fffffff;
    int e_rel = (L > 0) ? (int)min(cur.x - p0 - 1u, (u32)kNoRowEnd) : kNoRowEnd;

    // ---- walk the window's nonzeros ---------------------------------------------------------
    constexpr bool kSmemBc = SPMX_SMEM_BCAST && G == 8 && U == G && SPMX_SHFL_AHEAD;
    int par = 0;
#pragma unroll 1
    for (u32 nb = 0; nb < Lmax; nb += G) {
      const int rem = (int)min(L > nb ? L - nb : 0u, 0x7fffffffu);  // positions this group has left
      u32 c2 = 0;
      float v2 = 0.0f;
      if (nb + 2 * G + lg < L) {
        SPMX_CHECK(j0 + p0 + nb + 2 * G + lg < a.nnz, 1);
        c2 = ld_stream(colp + p0 + nb + 2 * G + lg, pol_first);
        v2 = ld_stream(valp + p0 + nb + 2 * G + lg, pol_first);
      }
#if SPMX_PF_STREAM
      if ((nb & 31u) == 0) {  // warp-uniform: once per line
        const u32 q = p0 + nb + 2 * G + SPMX_PF_DIST;
        if (lg == 0 && q < span) pf_stream(colp + q);
        if (lg == 1 && q < span) pf_stream(valp + q);
      }
#endif

      // The broadcasts of position t + 1 are issued before position t is consumed, so that the
      // shuffle latency is off the per-position critical path.
      float vq = 0.0f;
      u32 kq = 0;
      uint2 (*slot)[Window<G>::NGW] = sm.bc[par];
      if constexpr (kSmemBc) {
        par ^= 1;
        slot[lg][g] = make_uint2(c1, __float_as_uint(v0));  // U == G: position t + U is in the next batch
        __syncwarp();
        const uint2 pr = slot[0][g];
        kq = pr.x;
        vq = __uint_as_float(pr.y);
      } else if (SPMX_SHFL_AHEAD) {
        vq = __shfl_sync(kFullMask, v0, 0, G);
        kq = (U < G) ? __shfl_sync(kFullMask, c0, U % G, G) : __shfl_sync(kFullMask, c1, 0, G);
      }
#pragma unroll
      for (int t = 0; t < G; ++t) {
        const int u = t % U;
        float vq_n = 0.0f;
        u32 kq_n = 0;
        if (!SPMX_SHFL_AHEAD) {
          vq = __shfl_sync(kFullMask, v0, t, G);
          kq = (t + U < G) ? __shfl_sync(kFullMask, c0, t + U, G) : __shfl_sync(kFullMask, c1, t + U - G, G);
        } else if (kSmemBc) {
          if (t + 1 < G) {
            const uint2 pr = slot[t + 1][g];
            kq_n = pr.x;
            vq_n = __uint_as_float(pr.y);
          }
        } else if (t + 1 < G) {
          vq_n = __shfl_sync(kFullMask, v0, t + 1, G);
          kq_n = (t + 1 + U < G) ? __shfl_sync(kFullMask, c0, t + 1 + U, G)
                                 : __shfl_sync(kFullMask, c1, t + 1 + U - G, G);
        }
        if (t < rem) {
#pragma unroll
          for (int tt = 0; tt < NT; ++tt)
            if (tile_on<D_CT, G, VEC, RAGGED>(a, tt, lg)) {
              fma_tile<VEC, kPackFma>(vq, xv[u][tt], acc[tt]);
            }
        }
        // the slot is free again: refill it before any row-end work (with four tiles per lane
        // the compiler turns this order into three branches per position: refill afterwards)
        if (kRefillFirst && t + U < rem) {
          SPMX_CHECK((u64)kq < a.n_x, 4);
          const float* xr = xbase + (size_t)kq * (size_t)ldx;
#pragma unroll
          for (int tt = 0; tt < NT; ++tt)
            if (tile_on<D_CT, G, VEC, RAGGED>(a, tt, lg)) xv[u][tt] = ld_x<VEC>(xr + tt * G * VEC, pol_last);
        }
        if (t == e_rel) {  // row k ends here: store it, start the next one
          SPMX_CHECK(cur.y == kCarryIdx ? carry_lane != nullptr : wbase + cur.y < a.m, 7);
          float* dst = (cur.y != kCarryIdx) ? ywin + (size_t)cur.y * (size_t)ldx : carry_lane;
          store_lane<D_CT, G, VEC, NT, RAGGED>(a, dst, lg, acc, pol_first);
          zero_acc_from(acc, zero_f);
          ++k;
          e_rel = (k < count) ? (int)min((u32)e_rel + (nxt.x - cur.x), (u32)kNoRowEnd) : kNoRowEnd;
          // (the copies are pinned inside the branch: the compiler otherwise hoists them in
          // front of every position's row-end test)
          asm volatile("mov.b32 %0, %2;\n\tmov.b32 %1, %3;" : "=r"(cur.x), "=r"(cur.y) : "r"(nxt.x), "r"(nxt.y));
          SPMX_CHECK(k + 1 < W + 2, 6);
          nxt = s_rec[k + 1];
        }
        if (!kRefillFirst && t + U < rem) {
          SPMX_CHECK((u64)kq < a.n_x, 4);
          const float* xr = xbase + (size_t)kq * (size_t)ldx;
#pragma unroll
          for (int tt = 0; tt < NT; ++tt)
            if (tile_on<D_CT, G, VEC, RAGGED>(a, tt, lg)) xv[u][tt] = ld_x<VEC>(xr + tt * G * VEC, pol_last);
        }
        vq = vq_n;
        kq = kq_n;
      }
      c0 = c1; v0 = v1;
      c1 = c2; v1 = v2;
      if (e_rel < kNoRowEnd) e_rel -= G;
    }
    ws = we;
  }
}

// Static work list: group s of the grid (G lanes) owns chunk s.
template <int D_CT, int G, int VEC, int NT, bool RAGGED>
__global__ void __launch_bounds__(kWarpsPerCta * 32, Tune<D_CT, G, NT>::kMinCtas)
spmm_chunk_kernel(const SpmmArgs a) {
  constexpr int NGW = 32 / G;
  __shared__ WarpScratch<G> scratch[kWarpsPerCta];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const u64 warp = (u64)blockIdx.x * kWarpsPerCta + w;
  // the fix-up kernel is launched with programmatic stream serialisation: let its CTAs take
  // the SM slots this grid frees in its tail (they wait for this grid's completion before
  // they touch the carries)
  asm volatile("griddepcontrol.launch_dependents;");
  if (a.chunk_begin + warp * NGW >= a.chunk_end) return;  // whole warp idle
  if (a.abort_flag && *(volatile const int*)a.abort_flag) return;
  const u64 slot = a.chunk_begin + warp * NGW + lane / G;
  const bool active = slot < a.chunk_end;
  u64 r0 = 0, j0 = 0, r1 = 0, j1 = 0, chunk = 0;
  if (active) {
    const WorkItem it = a.work[slot];
    r0 = it.r0; j0 = it.j0; r1 = it.r1; j1 = it.j1; chunk = it.chunk;
  }
  const int ldx = D_CT ? D_CT : a.ldx;
  float* carry_row = (a.carry_out && active) ? a.carry_out + (size_t)chunk * (size_t)ldx : nullptr;
  process_piece<D_CT, G, VEC, NT, RAGGED>(a, active, r0, j0, r1, j1, carry_row, lane,
                                          scratch[w]);
}

// Dynamic row dispatch (row-split only): persistent warps claim `batch` rows at a time
// from a device counter — next_batch(), src/partition.cpp:29-33; the JIT'd `lock xadd`
// driver, src/jit.cpp:106-121. One claim per warp keeps the claimed ranges disjoint and
// covering [0, m) exactly as the reference's dispatcher does; the claimed rows are dealt
// to the warp's groups in contiguous runs of about equal nonzero count (rows are never split).
template <int D_CT, int G, int VEC, int NT, bool RAGGED>
__global__ void __launch_bounds__(kWarpsPerCta * 32, Tune<D_CT, G, NT>::kMinCtas)
spmm_dynamic_kernel(const SpmmArgs a) {
  constexpr int NGW = 32 / G;
  __shared__ WarpScratch<G> scratch[kWarpsPerCta];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane / G;
  // invalid input found by the validation kernels ahead of this launch: gather nothing
  if (a.abort_flag && *(volatile const int*)a.abort_flag) return;
  u64 v = 0;
  if (lane == 0) v = atomicAdd(a.counter, a.batch);
  v = __shfl_sync(kFullMask, v, 0);
  while (v < a.m) {
    // the next claim is issued now, so that its round trip overlaps this batch's work (a warp
    // over-claims once at the end, which next_batch() answers with "nothing left" as well)
    u64 vnext = 0;
    if (lane == 0) vnext = atomicAdd(a.counter, a.batch);
    const u64 hi = min(v + a.batch, a.m);
    // the claimed rows are dealt to the groups in contiguous runs of about equal nonzero count
    const u64 jl = __ldg(a.row_ptr + v), jh = __ldg(a.row_ptr + hi);
    u64 bnd[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int q = g + s;
      u64 r = q == 0 ? v : hi;
      if (q > 0 && q < NGW) {
        const u64 target = jl + (jh - jl) * (u64)q / NGW;
        u64 lo = v, up = hi;  // first row in [v, hi] whose start is >= target
        while (lo < up) {
          const u64 mid = lo + (up - lo) / 2;
          if (__ldg(a.row_ptr + mid) < target) lo = mid + 1; else up = mid;
        }
        r = lo;
      }
      bnd[s] = r;
    }
    const u64 b = bnd[0], e = bnd[1];
    const u64 j0 = __ldg(a.row_ptr + b), j1 = __ldg(a.row_ptr + e);
    process_piece<D_CT, G, VEC, NT, RAGGED>(a, b < e, b, j0, e, j1, nullptr, lane,
                                            scratch[w]);
    v = __shfl_sync(kFullMask, vnext, 0);
  }
}

// Long rows in exact-order mode. Every output element of a row is ONE fmaf chain over the row's
// nonzeros in CSR order (src/interp.cpp:36-51), serial by definition — but only the chain is:
// the gathers are not. One lane group walking a 39 542-nonzero row alone spends ~118 cycles per
// position (dependent issue latency of a lone warp: column -> address -> gather -> fma), so the
// plan hands rows of SPMX_LONG_ROW nonzeros or more to this kernel instead: one CTA of 8 warps
// per row. All 256 threads gather the X rows of the NEXT TWO tiles of positions into registers
// (2 x kLongK loads of PIECE floats per thread in flight: 64 KB per CTA with float4 pieces) while
// the consumer warps walk the current tile in shared memory in order, one column per thread:
// per position a broadcast LDS for the value (amortised over four positions), one conflict-free
// LDS for the X element and one dependent FFMA (~10-30 cycles per position instead of ~118);
// then the registers are stored to the other buffer. (cp.async would need no registers, but a warp sustains far
// fewer LDGSTS than LDG in flight: the same kernel with cp.async ran at ~74 cycles per position.)
// The result is bitwise the reference's: same operands, same order, one rounding per step.
struct LongRow {
  u64 row, j0, j1;
};
__device__ __forceinline__ float lds_f32(unsigned addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void lds_v4(unsigned addr, float& a, float& b, float& c, float& d) {
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(addr) : "memory");
}
__device__ __forceinline__ u32 lds_u32(unsigned addr) {
  u32 v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
template <int PIECE>
__device__ __forceinline__ void sts_piece(unsigned addr, const VecT<PIECE>& p) {
  if constexpr (PIECE == 4)
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(p.v[0]), "f"(p.v[1]), "f"(p.v[2]), "f"(p.v[3]) : "memory");
  else
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(p.v[0]) : "memory");
}
constexpr int kLongThreads = 256;
constexpr int kLongK = 8;  // loads per thread and tile; two tiles are in flight (two register sets)

// positions per tile for a slab of dw columns moved in pieces of `piece` floats
constexpr int kLongMaxTile = 1024;
__host__ __device__ constexpr int long_row_tile(int dw, int piece) {
  return kLongThreads * kLongK * piece / dw < kLongMaxTile ? kLongThreads * kLongK * piece / dw : kLongMaxTile;
}
__host__ __device__ constexpr size_t long_row_smem_bytes(int dw, int piece) {
  return 2 * (size_t)kLongThreads * kLongK * piece * 4 + 4 * (size_t)((long_row_tile(dw, piece) + 7) & ~3) * 8;
}

// PIECE: floats per load (4 when X rows are 16-byte aligned and the slab width is a multiple of
// 4, else 1). DW: the slab width when it is known at compile time (32, 64, 128: the element
// offsets of the consumer's loads become immediates), 0 = a.dw. The slab is at most 128 columns
// wide: warp w (w < ceil(dw / 32)) runs the chains of columns 32 w .. 32 w + 31, one per lane —
// the columns are independent chains, and a lone warp issues only one dependent instruction
// every few cycles, so four consumers are four times as fast as one lane holding four columns.
//
// Pipeline, iteration t (tile = TP positions): the gathers of tile t + 2 are issued into the
// register set that tile t's data has just left; tile t is consumed from shared memory by the
// consumer warps; tile t + 1 — issued one iteration ago, so it has had a whole iteration to
// arrive — is stored from the other register set to the other buffer; one barrier. Column
// indices and values run two tiles further ahead (registers, then a four-slot ring) under the
// same rule. Everything that does not change from tile to tile (which position and which columns
// a thread's k-th load belongs to, its shared-memory offsets) is computed once: a warp that has
// few instructions to issue per tile is what keeps the consumers, which share the SM's issue
// slots with the seven other warps, near the latency of their chain.
// Measured split on c4 (d = 32, longest row 184 124 nonzeros, 2.29 ms): 1.27 ms without the
// consumer, 1.83 ms without the gathers — the two add up instead of overlapping, because ptxas
// puts the gathers of both register sets and the consumer's LDS results on scoreboards that a
// consumer warp has to drain together (the counter semantics of DESIGN.md 7.5). Dedicated
// producer warps, split in two groups with one tile in flight each, would take the loads off the
// consumers' scoreboards; not done.
template <int PIECE, int DW>
__global__ void __launch_bounds__(kLongThreads, 2)  // 128 registers: two rows per SM
spmm_long_row_kernel(const SpmmArgs a, const LongRow* __restrict__ rows) {
  extern __shared__ float4 long_smem4[];
  const int dw = DW ? DW : a.dw, ldx = a.ldx, tid = threadIdx.x;
  const int my_col = tid;                       // consumer threads: tid < dw rounded up to a warp
  const bool consumer = (tid >> 5) < (dw + 31) / 32;
  const int ppr = dw / PIECE;                             // pieces per X row slab
  const int TP = long_row_tile(dw, PIECE);                // whole positions per tile
  const int cvs = (TP + 7) & ~3;                          // stride of the column/value rings (16-byte rows)
  const int tile_floats = kLongThreads * kLongK * PIECE;  // buffer stride (>= TP * dw)
  float* xbuf = reinterpret_cast<float*>(long_smem4);     // [2][tile_floats]
  u32* cbuf = reinterpret_cast<u32*>(xbuf + 2 * (size_t)tile_floats);  // [4][cvs]
  float* vbuf = reinterpret_cast<float*>(cbuf + 4 * cvs);                 // [4][cvs]
  const unsigned xbuf_s = (unsigned)__cvta_generic_to_shared(xbuf);
  const unsigned cbuf_s = (unsigned)__cvta_generic_to_shared(cbuf);
  const unsigned vbuf_s = (unsigned)__cvta_generic_to_shared(vbuf);
  const unsigned colb = (unsigned)min(my_col, dw - 1) * 4u;  // byte offset of this thread's column (clamped)
  if (a.abort_flag && *(volatile const int*)a.abort_flag) return;
  const LongRow lr = rows[blockIdx.x];
  const u64 len = lr.j1 - lr.j0;
  const u64 n_tiles = (len + TP - 1) / TP;
  const u32* __restrict__ colp = a.col + lr.j0;
  const float* __restrict__ valp = a.vals + lr.j0;

  // piece q = k * kLongThreads + tid of a tile: position pos[k] of the tile, columns
  // off .. off + PIECE - 1 of the slab. Kept as the byte offset of the position's column index
  // in a ring slot (cpos), the piece's byte offset in a tile buffer (soff) and the address of the
  // piece in X row 0 (xcol); `live` has bit k set when the piece exists (pos[k] < TP).
  unsigned cpos[kLongK], soff[kLongK], live = 0;
  const float* xcol[kLongK];
#pragma unroll
  for (int k = 0; k < kLongK; ++k) {
    const int q = k * kLongThreads + tid;
    const int pos = q / ppr, off = (q % ppr) * PIECE;
    cpos[k] = (unsigned)pos * 4u;
    soff[k] = (unsigned)(pos * dw + off) * 4u;
    xcol[k] = a.x + a.c0 + off;
    if (pos < TP) live |= 1u << k;
  }
  typedef VecT<PIECE> Piece;
  Piece set0[kLongK], set1[kLongK];

  // column indices and values of a tile: loaded into registers (fetch_cv), stored to ring slot
  // t % 4 later (store_cv), so that nobody waits for them between the two
  constexpr int kCv = (kLongMaxTile + kLongThreads - 1) / kLongThreads;
  const int n_cv = (TP + kLongThreads - 1) / kLongThreads;  // 1 for slabs of 32 columns and more
  u32 cv_c[kCv];
  float cv_v[kCv];
  auto fetch_cv = [&](u64 t) {
#pragma unroll
    for (int k = 0; k < kCv; ++k) {
      if (k >= n_cv) break;
      const int i = tid + k * kLongThreads;
      const u64 p = t * TP + i;
      cv_c[k] = 0;
      cv_v[k] = 0.0f;
      if (i < TP && p < len) { SPMX_CHECK(lr.j0 + p < a.nnz, 9); cv_c[k] = __ldcs(colp + p); cv_v[k] = __ldcs(valp + p); }
    }
  };
  auto store_cv = [&](u64 t) {
#pragma unroll
    for (int k = 0; k < kCv; ++k) {
      if (k >= n_cv) break;
      const int i = tid + k * kLongThreads;
      if (i < TP) {
        cbuf[(t & 3) * cvs + i] = cv_c[k];
        vbuf[(t & 3) * cvs + i] = cv_v[k];
      }
    }
  };
  auto gather = [&](u64 t, Piece (&r)[kLongK]) {  // X rows of tile t -> a register set
    const unsigned cs = cbuf_s + (unsigned)(t & 3) * (unsigned)cvs * 4u;
    const u64 left = t < n_tiles ? len - t * TP : 0;
    if (left >= (u64)TP && live == (1u << kLongK) - 1u) {  // a whole tile, every piece exists
#pragma unroll
      for (int k = 0; k < kLongK; ++k) {
        SPMX_CHECK((u64)lds_u32(cs + cpos[k]) < a.n_x, 10);
        r[k] = ld_x<PIECE>(xcol[k] + (size_t)lds_u32(cs + cpos[k]) * (size_t)ldx, 0);
      }
    } else {
#pragma unroll
      for (int k = 0; k < kLongK; ++k)
        if ((live >> k & 1u) && (u64)(cpos[k] >> 2) < left) {
          SPMX_CHECK((u64)lds_u32(cs + cpos[k]) < a.n_x, 10);
          r[k] = ld_x<PIECE>(xcol[k] + (size_t)lds_u32(cs + cpos[k]) * (size_t)ldx, 0);
        }
    }
  };
  auto stash = [&](u64 t, const Piece (&r)[kLongK]) {  // a register set -> buffer t & 1
    const unsigned dst = xbuf_s + (unsigned)(t & 1) * (unsigned)tile_floats * 4u;
#pragma unroll
    for (int k = 0; k < kLongK; ++k)
      if (live >> k & 1u) sts_piece<PIECE>(dst + soff[k], r[k]);
  };

  float acc = 0.0f;
  auto consume = [&](u64 t) {
    // Loads first, then the chain: 8 positions' values and X elements are in registers before
    // the first of their FFMAs issues. Threads beyond the slab width read the last column again
    // (no predicates in the loop; their sums are never stored).
    unsigned xb = xbuf_s + (unsigned)(t & 1) * (unsigned)tile_floats * 4u + colb;
    unsigned vb = vbuf_s + (unsigned)(t & 3) * (unsigned)cvs * 4u;
    const int npos = (int)min((u64)TP, len - t * TP);
    const unsigned row_bytes = (unsigned)dw * 4u;
    int i = 0;
    for (; i + 8 <= npos; i += 8) {
      float v[8], xe[8];
      lds_v4(vb, v[0], v[1], v[2], v[3]);
      lds_v4(vb + 16u, v[4], v[5], v[6], v[7]);
#pragma unroll
      for (int e = 0; e < 8; ++e) xe[e] = lds_f32(xb + (unsigned)e * row_bytes);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = __fmaf_rn(v[e], xe[e], acc);
      vb += 32u;
      xb += 8u * row_bytes;
    }
    for (; i < npos; ++i) {
      acc = __fmaf_rn(lds_f32(vb), lds_f32(xb), acc);
      vb += 4u;
      xb += row_bytes;
    }
  };

  for (u64 t = 0; t < 3; ++t) { fetch_cv(t); store_cv(t); }
  __syncthreads();
  gather(0, set0);
  stash(0, set0);
  gather(1, set1);
  fetch_cv(3);
  __syncthreads();

  // Every load is issued a whole iteration before its data is stored to shared memory: nobody
  // waits for memory between two barriers except for what the previous iteration left in flight.
  for (u64 t = 0; t < n_tiles; t += 2) {
    // even tile t: its data left set0 (stored before the last barrier); tile t + 1 is in set1
    store_cv(t + 3);      // fetched during the previous iteration; slot last read as tile t - 1
    fetch_cv(t + 4);
    gather(t + 2, set0);
    if (consumer) consume(t);
    stash(t + 1, set1);   // buffer (t + 1) & 1: last read as tile t - 1
    __syncthreads();
    if (t + 1 >= n_tiles) break;  // CTA-uniform
    // odd tile t + 1: tile t + 2 is in set0
    store_cv(t + 4);
    fetch_cv(t + 5);
    gather(t + 3, set1);
    if (consumer) consume(t + 1);
    stash(t + 2, set0);
    __syncthreads();
  }
  SPMX_CHECK(lr.row < a.m && lr.j1 <= a.nnz, 11);
  if (my_col < dw) __stcs(a.y + (size_t)lr.row * (size_t)ldx + a.c0 + my_col, acc);
}

// Carry fix-up. A row cut by chunk boundaries is summed from the partials of the chunks that
// hold its pieces, in CSR order: y[r] (the row's tail, stored by the chunk in which the row
// ends) += carry[first] + carry[first+1] + ... + carry[last]. Which boundaries close such a
// chain, and where the chain starts, depends only on the plan: chain_first_kernel records it
// once per plan (kNoChain where boundary t+1 closes nothing), so that the fix-up itself is one
// coalesced load per boundary followed by the chain's loads.
constexpr u32 kNoChain = 0xffffffffu;

// first[t], t in [0, n_chunks - 1): boundary t+1 (between chunks t and t+1) lies inside row
// r = chunk_row[t+1] and chunk t+1 ends that row -> the chunk holding the row's first nonzero.
// Boundaries that close a chain are also appended to a list — long_list for chains of more
// than kLongChain partials, short_list for the others (in no particular order; the chains
// are independent of each other) — so that the fix-up grid is sized by the number of chains,
// not by the number of boundaries.
constexpr u32 kLongChain = 16;

__global__ void chain_first_kernel(const u64* __restrict__ row_ptr, const u64* __restrict__ chunk_row,
                                   const u64* __restrict__ chunk_nnz, u64 n_chunks, u64 m,
                                   u32* __restrict__ first, u32* __restrict__ long_list,
                                   u32* __restrict__ long_count, u32* __restrict__ short_list,
                                   u32* __restrict__ short_count) {
  const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_chunks) return;
  u32 out = kNoChain;
  if (t + 1 < n_chunks) {  // the last chunk ends at (m, nnz)
    const u64 r = chunk_row[t + 1];
    if (r < m) {
      const u64 rp = __ldg(row_ptr + r);
      if (chunk_nnz[t + 1] > rp && chunk_row[t + 2] != r) {
        u64 lo = 0, hi = t;  // last chunk u with chunk_nnz[u] <= rp
        while (lo < hi) {
          const u64 mid = lo + (hi - lo + 1) / 2;
          if (chunk_nnz[mid] <= rp) lo = mid; else hi = mid - 1;
        }
        out = (u32)lo;
        if (t - lo + 1 > kLongChain) long_list[atomicAdd(long_count, 1u)] = (u32)t;
        else short_list[atomicAdd(short_count, 1u)] = (u32)t;
      }
    }
  }
  first[t] = out;
}

// Sum of the partials carry[ub .. ue) of one column vector, in order; the loads of a batch are
// independent and overlap.
template <int VEC>
__device__ __forceinline__ VecT<VEC> chain_sum(const float* __restrict__ src_c, int ldx, u64 ub, u64 ue) {
  constexpr int kBatch = 8;
  VecT<VEC> s;
#pragma unroll
  for (int e = 0; e < VEC; ++e) s.v[e] = 0.0f;
  u64 u = ub;
  for (; u + kBatch <= ue; u += kBatch) {
    VecT<VEC> part[kBatch];
#pragma unroll
    for (int q = 0; q < kBatch; ++q)
      part[q] = *reinterpret_cast<const VecT<VEC>*>(src_c + (size_t)(u + q) * ldx);
#pragma unroll
    for (int q = 0; q < kBatch; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) s.v[e] += part[q].v[e];
  }
  for (; u < ue; ++u) {
    const VecT<VEC> part = *reinterpret_cast<const VecT<VEC>*>(src_c + (size_t)u * ldx);
#pragma unroll
    for (int e = 0; e < VEC; ++e) s.v[e] += part.v[e];
  }
  return s;
}

// The first n_long CTAs take one long chain each (more than kLongChain partials): the chain is
// cut into blockDim/lpc consecutive segments, one per group of lpc lanes, each summed in CSR
// order; the segment sums are then added in order. The other CTAs give one group of `lpc`
// lanes (a power of two, <= 32) to every entry of short_list: lane lg sums columns lg*VEC ..
// of the short chain closed by that boundary, in CSR order. Both orders are fixed by the
// plan, so the result is deterministic. Only chains closed by a boundary t+1 with t in
// [t_begin, t_end) and starting in a chunk in [first_lo, first_hi) are handled: the host
// pipeline runs the fix-up block by block, and defers the one chain per block whose first
// partials belong to a block it has not computed yet.
constexpr int kFixupThreads = 256;

template <int VEC>
__global__ void __launch_bounds__(kFixupThreads)
carry_fixup_kernel(const u32* __restrict__ chain_first, const u64* __restrict__ chunk_row,
                   const u32* __restrict__ long_list, u32 n_long,
                   const u32* __restrict__ short_list, u32 n_short, u64 t_begin, u64 t_end,
                   u64 first_lo, u64 first_hi,
                   const float* __restrict__ carry_out, float* __restrict__ y, int ldx, int c0,
                   int dw, int lpc) {
  // Launched with programmatic stream serialisation: EVERY thread executes griddepcontrol.wait
  // before it retires, also the ones with nothing to do — a grid in which nobody waits could
  // complete while the SpMM grid before it is still running, and whatever follows on the
  // stream (the Y download of the host pipeline, the next block's kernels) is ordered after
  // this grid only. Plan data is read above the wait, SpMM results below it.
  if (blockIdx.x < n_long) {
    __shared__ VecT<VEC> seg_sum[kFixupThreads];
    const u64 last = long_list[blockIdx.x];
    const bool mine = last >= t_begin && last < t_end;  // CTA-uniform
    u64 first = 0, rr = 0;
    if (mine) { first = __ldg(chain_first + last); rr = __ldg(chunk_row + last + 1); }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (!mine || first < first_lo || first >= first_hi) return;  // CTA-uniform
    const int nseg = kFixupThreads / lpc, seg = threadIdx.x / lpc, lg = threadIdx.x % lpc;
    const u64 per = (last - first + nseg) / nseg;  // ceil(len / nseg)
    const u64 ub = min(first + (u64)seg * per, last + 1), ue = min(ub + per, last + 1);
    for (int cb = 0; cb < dw; cb += lpc * VEC) {  // CTA-uniform trip count
      const int c = cb + lg * VEC;
      if (c < dw) seg_sum[threadIdx.x] = chain_sum<VEC>(carry_out + c0 + c, ldx, ub, ue);
      __syncthreads();
      if (seg == 0 && c < dw) {
        float* dst = y + (size_t)rr * ldx + c0 + c;
        VecT<VEC> s = seg_sum[lg];
        for (int q = 1; q < nseg; ++q) {
          const VecT<VEC> part = seg_sum[q * lpc + lg];
#pragma unroll
          for (int e = 0; e < VEC; ++e) s.v[e] += part.v[e];
        }
        const VecT<VEC> tail = *reinterpret_cast<const VecT<VEC>*>(dst);
#pragma unroll
        for (int e = 0; e < VEC; ++e) s.v[e] += tail.v[e];
        *reinterpret_cast<VecT<VEC>*>(dst) = s;
      }
      __syncthreads();
    }
    return;
  }
  const u64 tid = (u64)(blockIdx.x - n_long) * kFixupThreads + threadIdx.x;
  const u64 entry = tid / (unsigned)lpc;
  const int lg = (int)(tid % (unsigned)lpc);
  // chunk whose END boundary closes this chain
  u64 last = 0, rr = 0;
  u32 u0 = 0;
  bool mine = entry < n_short;
  if (mine) {
    last = __ldg(short_list + entry);
    mine = last >= t_begin && last < t_end;
  }
  if (mine) {
    u0 = __ldg(chain_first + last);
    rr = __ldg(chunk_row + last + 1);
    mine = u0 >= first_lo && u0 < first_hi;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (!mine) return;
  for (int c = lg * VEC; c < dw; c += lpc * VEC) {
    float* dst = y + (size_t)rr * ldx + c0 + c;
    const VecT<VEC> tail = *reinterpret_cast<const VecT<VEC>*>(dst);
    VecT<VEC> s = chain_sum<VEC>(carry_out + c0 + c, ldx, u0, last + 1);
#pragma unroll
    for (int e = 0; e < VEC; ++e) s.v[e] += tail.v[e];
    *reinterpret_cast<VecT<VEC>*>(dst) = s;
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
