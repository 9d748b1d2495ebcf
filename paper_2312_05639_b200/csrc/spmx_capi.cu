// spmx_capi.cu — implementation of include/spmx_b200.h (the C ABI of the B200 SpMM path).
//
// Host-side orchestration only: handle lifetime, argument checks with the reference's
// error behaviour, plan construction (partition.cuh kernels) and kernel dispatch per d
// (the GPU counterpart of the reference's per-d code generation, src/plan.cpp:42-93 and
// src/jit.cpp:136-154: everything that depends on d is fixed before the hot loop).
#include "../../include/spmx_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "spmx_jit.cuh"
#include "spmx_kernels.cuh"
#include "spmx_partition.cuh"
#include "spmx_probe.cuh"
#include "spmx_stage.cuh"

using spmx_dev::u64;

#define SPMX_STR2(x) #x
#define SPMX_STR(x) SPMX_STR2(x)

namespace {

// "key=value;" pairs. The digit after SPMX_SASS_SCHED= is rewritten in the linked library by
// the post-link scheduling step (sass_sched.py): the number of kernels it re-scheduled, 0 when
// the library runs the schedule exactly as ptxas emitted it. Kept in writable data so that the
// text exists once in the binary.
char g_build_info[96] = "SPMX_SASS_SCHED=0;" "cuda=" SPMX_STR(CUDART_VERSION) ";arch=sm_100a;";

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

struct InvalidArg : std::runtime_error { using std::runtime_error::runtime_error; };
struct LogicErr : std::runtime_error { using std::runtime_error::runtime_error; };

#define CUDA_CHECK(expr)                                                                   \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(_e) +      \
                               " at " #expr);                                              \
  } while (0)

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return SPMX_OK;
  } catch (const InvalidArg& e) {
    g_last_error = e.what();
    return SPMX_EINVAL;
  } catch (const LogicErr& e) {
    g_last_error = e.what();
    return SPMX_ELOGIC;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return SPMX_ERUNTIME;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SPMX_ERUNTIME;
  }
}

constexpr uint32_t kMagicCtx = 0x58435443, kMagicCsr = 0x58435352, kMagicPlan = 0x58504c4e;
constexpr u64 kDefaultChunkItems = 256;  // merge items (rows + nonzeros) per warp-level chunk

// tuning knobs, overridable from the environment for experiments (tools/dev_bench.py)
inline u64 env_u64(const char* name, u64 dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? (u64)std::strtoull(v, nullptr, 10) : dflt;
}
inline u64 chunk_items() { return std::max<u64>(32, env_u64("SPMX_CHUNK_ITEMS", kDefaultChunkItems)); }
// small inputs: shrink the chunks until there are enough of them to occupy every SM
inline u64 chunk_items_for(u64 items, int sm_count) {
  const u64 want_chunks = (u64)sm_count * 64;
  return std::min<u64>(chunk_items(), std::max<u64>(32, items / want_chunks));
}
// interior chunk boundaries never cut a row shorter than this
inline u64 snap_len() { return env_u64("SPMX_SNAP_LEN", 128); }
inline u64 default_parts_per_sm() { return env_u64("SPMX_PARTS_PER_SM", 8); }
// exact-order plans: rows at least this long run in spmm_long_row_kernel (0 disables)
inline u64 long_row_min() { return env_u64("SPMX_LONG_ROW", 1024); }

inline unsigned blocks_for(u64 n, unsigned threads = 256) {
  return (unsigned)((n + threads - 1) / threads);
}

}  // namespace

struct spmx_ctx {
  uint32_t magic = kMagicCtx;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sm_count = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int* d_err = nullptr;  // device-side error flag for validation
  cudaStream_t s_compute = nullptr, s_d2h = nullptr, s_x = nullptr;  // spmx_spmm_host pipeline (lazy)
  size_t l2_persist = 0;         // persisting-L2 set-aside this context last asked for (spmx_ctx_l2_window)
  cudaStream_t s_aux = nullptr;  // long rows of exact-order plans run beside the main kernel (lazy)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<cudaEvent_t> pipe_events;                // created once, reused by every call
  // grow-only staging used by spmx_spmm_host
  void* ws[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t ws_bytes[5] = {0, 0, 0, 0, 0};
};

struct spmx_csr {
  uint32_t magic = kMagicCsr;
  spmx_ctx* ctx = nullptr;
  int64_t m = 0, n = 0, nnz = 0;
  u64* row_ptr = nullptr;
  uint32_t* col = nullptr;
  float* vals = nullptr;
  bool owned = false;
  bool structure_only = false;  // spmx_rowptr_upload: partitioner / plan input only
};

struct spmx_plan {
  uint32_t magic = kMagicPlan;
  spmx_ctx* ctx = nullptr;
  const spmx_csr* csr = nullptr;
  int strategy = 0;
  unsigned parts = 0;
  unsigned flags = 0;
  bool dynamic = false;  // make_partition's dynamic dispatch was asked for (no RowRange list)
  bool claims = false;   // ... and it runs as the atomic-claim kernel (see plan_build)
  u64 batch = 128;
  u64 n_chunks = 0;
  u64* ranges = nullptr;     // 2*parts, device (absent under dynamic dispatch)
  u64* chunk_row = nullptr;  // n_chunks+1
  u64* chunk_nnz = nullptr;  // n_chunks+1
  spmx_dev::WorkItem* work = nullptr;  // n_chunks: the chunks in launch order (sorted inside tiles)
  uint32_t* chain_first = nullptr;  // n_chunks: start of the carry chain closed by boundary t+1
  uint32_t* long_buf = nullptr;     // [count | boundaries closing chains longer than kLongChain]
  uint32_t* long_list = nullptr;    // = long_buf + 1
  uint32_t n_long = 0;
  uint32_t* short_buf = nullptr;    // [count | boundaries closing the other chains]
  uint32_t* short_list = nullptr;   // = short_buf + 1
  uint32_t n_short = 0;
  spmx_dev::LongRow* long_rows = nullptr;  // exact-order plans: rows run by spmm_long_row_kernel
  uint32_t n_long_rows = 0;
  u64* counter = nullptr;    // dynamic dispatch
  u64 x_extra_rows = 0;  // rows behind X the columns may point at (the multi-GPU driver's hot-row copy)
  bool may_carry = false;
  mutable float* carry = nullptr;  // n_chunks x ld floats, grown on demand
  mutable size_t carry_floats = 0;
};

namespace {

spmx_ctx* check(spmx_ctx* c) {
  if (!c || c->magic != kMagicCtx) throw LogicErr("invalid or destroyed spmx_ctx");
  CUDA_CHECK(cudaSetDevice(c->device));
  return c;
}
const spmx_csr* check(const spmx_csr* a) {
  if (!a || a->magic != kMagicCsr) throw LogicErr("invalid or destroyed spmx_csr");
  return a;
}
const spmx_plan* check(const spmx_plan* p) {
  if (!p || p->magic != kMagicPlan) throw LogicErr("invalid or destroyed spmx_plan");
  return p;
}

template <typename T>
T* dev_alloc(size_t count) {
  T* p = nullptr;
  CUDA_CHECK(cudaMalloc(&p, (count ? count : 1) * sizeof(T)));
  return p;
}

// Stream-ordered allocations for plans and their temporaries: no device-wide synchronisation
// (cudaMalloc/cudaFree serialise against transfers in flight), and after the first plan the
// pool hands the same memory back in microseconds.
template <typename T>
T* dev_alloc_async(spmx_ctx* ctx, size_t count) {
  T* p = nullptr;
  CUDA_CHECK(cudaMallocAsync(&p, (count ? count : 1) * sizeof(T), ctx->stream));
  return p;
}
void dev_free_async(spmx_ctx* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}

// Temporaries of a plan build / partition call: returned to the stream-ordered pool when the
// scope is left, on the exception path as well.
struct AsyncScratch {
  spmx_ctx* ctx;
  std::vector<void*> ptrs;
  explicit AsyncScratch(spmx_ctx* c) : ctx(c) {}
  AsyncScratch(const AsyncScratch&) = delete;
  AsyncScratch& operator=(const AsyncScratch&) = delete;
  template <typename T>
  T* get(size_t count) {
    T* p = dev_alloc_async<T>(ctx, count);
    ptrs.push_back(p);
    return p;
  }
  ~AsyncScratch() {
    for (void* p : ptrs) dev_free_async(ctx, p);
  }
};

void launched(unsigned n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void post_launch() {
  launched();
  CUDA_CHECK(cudaGetLastError());
}

// ---- partition boundaries on the device --------------------------------------------------
// Fills bnd[0..parts] (row boundaries) for the strategy, row-snapped.
void strategy_row_boundaries(spmx_ctx* ctx, const spmx_csr* a, int strategy, unsigned parts,
                             u64* d_bnd) {
  const unsigned nb = blocks_for((u64)parts + 1);
  switch (strategy) {
    case SPMX_ROW_SPLIT:
      spmx_dev::row_boundaries_kernel<<<nb, 256, 0, ctx->stream>>>((u64)a->m, parts, d_bnd);
      break;
    case SPMX_NNZ_SPLIT:
      spmx_dev::nnz_boundaries_kernel<<<nb, 256, 0, ctx->stream>>>(a->row_ptr, (u64)a->m,
                                                                   (u64)a->nnz, parts, d_bnd);
      break;
    case SPMX_MERGE_SPLIT:
      spmx_dev::merge_boundaries_kernel<<<nb, 256, 0, ctx->stream>>>(
          a->row_ptr, (u64)a->m, (u64)a->nnz, parts, 1, d_bnd);
      break;
    default:
      throw InvalidArg("unknown strategy");
  }
  post_launch();
}

void ranges_to_host(spmx_ctx* ctx, const u64* d_bnd, unsigned parts, uint64_t* out) {
  AsyncScratch tmp(ctx);
  u64* d_ranges = tmp.get<u64>(2 * (size_t)parts);
  spmx_dev::ranges_from_boundaries_kernel<<<blocks_for(parts), 256, 0, ctx->stream>>>(
      d_bnd, parts, d_ranges);
  post_launch();
  CUDA_CHECK(cudaMemcpyAsync(out, d_ranges, 2 * (size_t)parts * sizeof(u64),
                             cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
}

const char* csr_error_text(int err) {
  static const char* what[] = {"", "", "row_ptr[0] != 0", "row_ptr[m] != nnz",
                               "row_ptr not nondecreasing", "column index out of range"};
  return what[err < 0 || err > 5 ? 0 : err];
}

unsigned validate_grid(spmx_ctx* ctx, u64 work) {
  return (unsigned)std::min<u64>((u64)ctx->sm_count * 8, std::max<u64>(1, (work + 255) / 256));
}

void validate_on_device(spmx_ctx* ctx, const spmx_csr* a) {
  CUDA_CHECK(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  spmx_dev::validate_row_ptr_kernel<<<validate_grid(ctx, (u64)a->m), 256, 0, ctx->stream>>>(
      a->row_ptr, (u64)a->m, (u64)a->nnz, ctx->d_err);
  post_launch();
  if (a->nnz > 0) {
    spmx_dev::validate_cols_kernel<<<validate_grid(ctx, (u64)a->nnz), 256, 0, ctx->stream>>>(
        a->col, (u64)a->nnz, (u64)a->n, ctx->d_err);
    post_launch();
  }
  int err = 0;
  CUDA_CHECK(cudaMemcpyAsync(&err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  if (err) throw InvalidArg(std::string("invalid CSR: ") + csr_error_text(err));
}

// ---- kernel dispatch per d ------------------------------------------------------------------
template <int D_CT, int G, int VEC, int NT, bool RAGGED>
void launch_one(const spmx_plan* p, const spmx_dev::SpmmArgs& args, cudaStream_t st, int sm_count) {
  if (p->claims) {
    int occ = 0;
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, spmx_dev::spmm_dynamic_kernel<D_CT, G, VEC, NT, RAGGED>, spmx_dev::kWarpsPerCta * 32,
        0));
    const unsigned grid = (unsigned)(sm_count * (occ > 0 ? occ : 1));
    spmx_dev::spmm_dynamic_kernel<D_CT, G, VEC, NT, RAGGED>
        <<<grid, spmx_dev::kWarpsPerCta * 32, 0, st>>>(args);
  } else {
    constexpr int kChunksPerCta = spmx_dev::kWarpsPerCta * (32 / G);  // one chunk per group
    const u64 count = args.chunk_end - args.chunk_begin;
    const unsigned grid = (unsigned)((count + kChunksPerCta - 1) / kChunksPerCta);
    if (grid == 0) return;
#ifndef SPMX_CARVEOUT
#define SPMX_CARVEOUT 30  // % of the unified L1/shared array given to shared memory
#endif
    // In-flight X-row gathers are held in L1 lines: the kernel needs only a few KB of shared
    // memory, so keep the carve-out small (the driver's default picked 135 KB, leaving the
    // gathers half the L1; tools/microbench/gather_bw2.cu shows the effect).
    static std::atomic<uint64_t> done_mask{0};  // one bit per device
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    if (!(done_mask.load() >> (dev & 63) & 1)) {
      done_mask.fetch_or(1ull << (dev & 63));
      CUDA_CHECK(cudaFuncSetAttribute(spmx_dev::spmm_chunk_kernel<D_CT, G, VEC, NT, RAGGED>,
                                      cudaFuncAttributePreferredSharedMemoryCarveout, SPMX_CARVEOUT));
    }
    spmx_dev::spmm_chunk_kernel<D_CT, G, VEC, NT, RAGGED>
        <<<grid, spmx_dev::kWarpsPerCta * 32, 0, st>>>(args);
  }
  post_launch();
}

// runtime-d kernels (ragged tiles): the shape spmx_jit::choose_shape picks for the slab, with the
// tile count rounded up to the next instantiated one (1, 2, 4; 8 with all 32 lanes)
template <int VEC>
void launch_generic(const spmx_plan* p, const spmx_dev::SpmmArgs& a, int g, int nt,
                    cudaStream_t st, int sms) {
  if (nt == 1) {
    switch (g) {
      case 1: return launch_one<0, 1, VEC, 1, true>(p, a, st, sms);
      case 2: return launch_one<0, 2, VEC, 1, true>(p, a, st, sms);
      case 4: return launch_one<0, 4, VEC, 1, true>(p, a, st, sms);
      case 8: return launch_one<0, 8, VEC, 1, true>(p, a, st, sms);
    }
  } else if (g == 8) {
    switch (nt) {
      case 2: return launch_one<0, 8, VEC, 2, true>(p, a, st, sms);
      case 4: return launch_one<0, 8, VEC, 4, true>(p, a, st, sms);
    }
  } else if (g == 16 && nt == 4) {
    return launch_one<0, 16, VEC, 4, true>(p, a, st, sms);
  } else if (g == 32) {
    switch (nt) {
      case 4: return launch_one<0, 32, VEC, 4, true>(p, a, st, sms);
      case 8: return launch_one<0, 32, VEC, 8, true>(p, a, st, sms);
    }
  }
  throw std::runtime_error("internal: no kernel for this shape");
}

// carry_out buffer of the plan for width d (cudaMalloc/cudaFree synchronise the device, so
// pipelines call this before they start their transfers)
void ensure_carry(const spmx_plan* p, int64_t d) {
  if (!p->may_carry) return;
  const size_t need = (size_t)p->n_chunks * (size_t)d;
  if (need > p->carry_floats) {
    dev_free_async(p->ctx, p->carry);
    p->carry = dev_alloc_async<float>(p->ctx, need);
    p->carry_floats = need;
    CUDA_CHECK(cudaStreamSynchronize(p->ctx->stream));  // other streams may use it next
  }
}

// carry_fixup_kernel over boundaries t+1, t in [tb, te), with the widest column vector the
// slab's alignment allows.
constexpr u64 kNoLimit = ~0ull;

void launch_fixup(const spmx_plan* p, u64 tb, u64 te, float* d_y, int ldx, int c0, int dw,
                  cudaStream_t st, u64 first_lo = 0, u64 first_hi = kNoLimit) {
  const bool a16 = ((uintptr_t)d_y % 16 == 0) && ldx % 4 == 0 && c0 % 4 == 0 && dw % 4 == 0;
  const bool a8 = ((uintptr_t)d_y % 8 == 0) && ldx % 2 == 0 && c0 % 2 == 0 && dw % 2 == 0;
  const int vec = a16 ? 4 : a8 ? 2 : 1;
  int lpc = 1;  // lanes per chain: enough to cover the slab once, at most a warp
  while (lpc < 32 && lpc * vec < dw) lpc *= 2;
  constexpr int kT = spmx_dev::kFixupThreads;
  if (p->n_long + p->n_short == 0) return;  // no row is cut: nothing to add
  const unsigned grid = p->n_long + blocks_for((u64)p->n_short * (u64)lpc, kT);
  // Programmatic stream serialisation: the grid may start while the SpMM kernel before it on
  // the stream is draining; it waits (griddepcontrol.wait) before it reads that kernel's output.
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kT);
  cfg.stream = st;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  const uint32_t* cf = p->chain_first;
  const u64* cr = p->chunk_row;
  const uint32_t* ll = p->long_list;
  const uint32_t* sl = p->short_list;
  const float* carry = p->carry;
  if (vec == 4)
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, spmx_dev::carry_fixup_kernel<4>, cf, cr, ll, p->n_long, sl,
                                  p->n_short, tb, te, first_lo, first_hi,
                                  carry, d_y, ldx, c0, dw, lpc));
  else if (vec == 2)
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, spmx_dev::carry_fixup_kernel<2>, cf, cr, ll, p->n_long, sl,
                                  p->n_short, tb, te, first_lo, first_hi,
                                  carry, d_y, ldx, c0, dw, lpc));
  else
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, spmx_dev::carry_fixup_kernel<1>, cf, cr, ll, p->n_long, sl,
                                  p->n_short, tb, te, first_lo, first_hi,
                                  carry, d_y, ldx, c0, dw, lpc));
  post_launch();
}

// spmm_long_row_kernel for the plan's long rows (exact-order plans), columns [c0, c0 + dw) of X
// and Y, on the context's auxiliary stream beside the main kernel: forked from `st` here, joined
// by the caller's join_long_rows after the main kernel has been queued.
template <int PIECE, int DW>
void launch_long_one(const spmx_plan* p, const spmx_dev::SpmmArgs& args, cudaStream_t st) {
  const size_t smem = spmx_dev::long_row_smem_bytes(args.dw, PIECE);
  static std::atomic<uint64_t> done_mask{0};  // one bit per device
  int dev = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  if (!(done_mask.load() >> (dev & 63) & 1)) {
    done_mask.fetch_or(1ull << (dev & 63));
    // the narrowest slab has the most positions per tile, i.e. the largest column/value rings
    CUDA_CHECK(cudaFuncSetAttribute(spmx_dev::spmm_long_row_kernel<PIECE, DW>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)spmx_dev::long_row_smem_bytes(DW ? DW : 1, PIECE)));
  }
  spmx_dev::spmm_long_row_kernel<PIECE, DW>
      <<<p->n_long_rows, spmx_dev::kLongThreads, smem, st>>>(args, p->long_rows);
  post_launch();
}

void launch_long_rows(spmx_ctx* ctx, const spmx_plan* p, spmx_dev::SpmmArgs args, int c0, int dw, bool piece4,
                      cudaStream_t st) {
  if (!ctx->s_aux) {
    CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->s_aux, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  }
  CUDA_CHECK(cudaEventRecord(ctx->ev_fork, st));
  CUDA_CHECK(cudaStreamWaitEvent(ctx->s_aux, ctx->ev_fork, 0));
  for (int cc = c0; cc < c0 + dw; cc += 128) {  // the ring holds slabs of up to 128 columns
    args.c0 = cc;
    args.dw = std::min(128, c0 + dw - cc);
    const bool p4 = piece4 && args.dw % 4 == 0 && cc % 4 == 0;
    if (!p4) launch_long_one<1, 0>(p, args, ctx->s_aux);
    else if (args.dw == 128) launch_long_one<4, 128>(p, args, ctx->s_aux);
    else if (args.dw == 64) launch_long_one<4, 64>(p, args, ctx->s_aux);
    else if (args.dw == 32) launch_long_one<4, 32>(p, args, ctx->s_aux);
    else launch_long_one<4, 0>(p, args, ctx->s_aux);
  }
  CUDA_CHECK(cudaEventRecord(ctx->ev_join, ctx->s_aux));
}

// Launches the SpMM (and carry fix-up) for chunks [cb, ce) of the plan's work list on `st`.
// The fix-up handles the chains that start in a chunk in [first_lo, first_hi); with
// fixup_only the SpMM itself is not launched (the host pipeline's deferred chains).
void run_kernels(spmx_ctx* ctx, const spmx_plan* p, const spmx_csr* a, const float* d_x,
                 int64_t d, float* d_y, cudaStream_t st, u64 cb, u64 ce, const int* abort_flag,
                 u64 first_lo = 0, u64 first_hi = kNoLimit, bool fixup_only = false) {
  if (a->m == 0) return;
  if (!p->claims && ce <= cb) return;  // empty block of the host pipeline
  // widest column vector the alignment of X and Y rows allows
  const bool aligned16 = ((uintptr_t)d_x % 16 == 0) && ((uintptr_t)d_y % 16 == 0);
  const int vec_max = (d % 4 == 0 && aligned16) ? 4 : 1;
  // Narrow rows: eight lanes with narrower vectors beat fewer lanes with float4 (eight positions
  // in flight per group, column/value broadcast through shared memory, four instead of eight
  // chunk streams per warp: d = 16 178 -> 130 us, d = 8 207 -> 117 us on c2's matrix), so the
  // vector is narrowed until a row spans at least five lanes.
  const int vec = spmx_jit::narrow_vec((int)d, vec_max);
  // Columns per launch. Wider matrices are multiplied slab by slab (A is streamed again per
  // slab: 8 bytes per nonzero against 4 * 128 gathered). With float4 columns the slab is 128
  // wide, the shape of the d = 128 kernel (8 lanes x 4 tiles, measured best; one launch over
  // 256 columns with 16-lane groups took 1.30 ms on c2's matrix against 1.05 ms for two slabs).
  const int slab_max = vec == 4 ? 128 : 32 * vec * 8;

  ensure_carry(p, d);

  spmx_dev::SpmmArgs args{};
  args.row_ptr = a->row_ptr;
  args.col = a->col;
  args.vals = a->vals;
  args.x = d_x;
  args.y = d_y;
  args.carry_out = p->may_carry ? p->carry : nullptr;
  args.work = p->work;
  args.n_chunks = p->n_chunks;
  args.chunk_begin = cb;
  args.chunk_end = ce;
  args.abort_flag = abort_flag;
  args.m = (u64)a->m;
  args.n_x = (u64)a->n + p->x_extra_rows;
  args.nnz = (u64)a->nnz;
  args.ldx = (int)d;
  args.counter = p->counter;
  args.batch = p->batch;

  // exact-order plans: the long rows, beside the main kernel (the plan took them out of its list)
  const bool long_rows = p->n_long_rows > 0 && !fixup_only && !p->claims;
  if (long_rows) launch_long_rows(ctx, p, args, 0, (int)d, vec_max == 4, st);

  // run-time instantiation for exactly this d (SPMX_JIT_WIDTH): one launch covers the whole
  // width when it fits 32 lanes x 8 tiles; the precompiled widths and dynamic plans keep
  // their own kernels
  const bool precompiled = (vec == 4 && (d == 32 || d == 64 || d == 128)) || (vec == 2 && d == 16) ||
                           (vec == 1 && d == 8);
  if ((p->flags & SPMX_JIT_WIDTH) && !p->claims && !precompiled && d <= spmx_jit::max_width(vec_max)) {
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    const spmx_jit::Kernel& k = spmx_jit::get(dev, (int)d, vec_max);
    args.c0 = 0;
    args.dw = (int)d;
    const int chunks_per_cta = spmx_dev::kWarpsPerCta * (32 / k.shape.g);
    const unsigned grid = (unsigned)((ce - cb + chunks_per_cta - 1) / chunks_per_cta);
    if (grid && !fixup_only) {
      void* kargs[] = {(void*)&args};
      CUDA_CHECK(cudaLaunchKernel((const void*)k.chunk, dim3(grid), dim3(spmx_dev::kWarpsPerCta * 32),
                                  kargs, 0, st));
      post_launch();
    }
    const u64 tb = cb > 0 ? cb - 1 : 0, te = ce > 0 ? ce - 1 : 0;
    if (p->may_carry && te > tb) {
      launch_fixup(p, tb, te, d_y, (int)d, 0, (int)d, st, first_lo, first_hi);
    }
    if (long_rows) CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
    return;
  }

  for (int64_t c0 = 0; c0 < d; c0 += slab_max) {
    const int dw = (int)std::min<int64_t>(slab_max, d - c0);
    args.c0 = (int)c0;
    args.dw = dw;
    if (p->claims && !fixup_only) CUDA_CHECK(cudaMemsetAsync(p->counter, 0, sizeof(u64), st));
#ifndef SPMX_NT
#define SPMX_NT 2  // float4 tiles per lane for the specialised widths
#endif
    if (fixup_only) {
    } else if (vec == 4 && c0 == 0 && d == 32) {
      launch_one<32, 8, 4, 1, false>(p, args, st, ctx->sm_count);  // 8 lanes x float4
    } else if (vec == 4 && c0 == 0 && d == 64) {
      launch_one<64, 16 / SPMX_NT, 4, SPMX_NT, false>(p, args, st, ctx->sm_count);
    } else if (vec == 2 && c0 == 0 && d == 16) {
      launch_one<16, 8, 2, 1, false>(p, args, st, ctx->sm_count);  // 8 lanes x float2
    } else if (vec == 1 && c0 == 0 && d == 8) {
      launch_one<8, 8, 1, 1, false>(p, args, st, ctx->sm_count);
    } else if (vec == 4 && c0 == 0 && d == 128) {
      launch_one<128, 8, 4, 4, false>(p, args, st, ctx->sm_count);  // 8 lanes x 4 tiles
    } else if (vec == 4 && dw == 128) {
      launch_one<0, 8, 4, 4, false>(p, args, st, ctx->sm_count);  // full slab of a wider matrix
    } else {
      const int lanes = (dw + vec - 1) / vec;
      int g = 1, nt = 1;
      while (g < 8 && g < lanes) g <<= 1;
      for (;; g <<= 1) {  // 8 lanes up to 4 tiles, 16 lanes x 4, 32 lanes x 4 or 8 (slab_max bounds it)
        nt = (lanes + g - 1) / g;
        if (nt <= (g < 32 ? 4 : 8)) break;
      }
      nt = nt <= 2 ? nt : nt <= 4 ? 4 : 8;
      if (g == 16) nt = 4;
      if (g == 32 && nt < 4) nt = 4;
      if (vec == 4)
        launch_generic<4>(p, args, g, nt, st, ctx->sm_count);
      else if (vec == 2)
        launch_one<0, 8, 2, 1, true>(p, args, st, ctx->sm_count);  // d = 12 (16 is precompiled)
      else
        launch_generic<1>(p, args, g, nt, st, ctx->sm_count);
    }
    // rows that END in chunks [cb, ce) are closed by boundaries t+1 in [cb, ce): t in [cb-1, ce-1)
    const u64 tb = cb > 0 ? cb - 1 : 0, te = ce > 0 ? ce - 1 : 0;
    if (p->may_carry && te > tb) {
      launch_fixup(p, tb, te, d_y, (int)d, (int)c0, dw, st, first_lo, first_hi);
    }
  }
  if (long_rows) CUDA_CHECK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
}

void plan_free(spmx_plan* p) {
  if (!p) return;
  dev_free_async(p->ctx, p->ranges);
  dev_free_async(p->ctx, p->chunk_row);
  dev_free_async(p->ctx, p->work);
  dev_free_async(p->ctx, p->chain_first);
  dev_free_async(p->ctx, p->long_buf);
  dev_free_async(p->ctx, p->short_buf);
  dev_free_async(p->ctx, p->chunk_nnz);
  dev_free_async(p->ctx, p->counter);
  dev_free_async(p->ctx, p->long_rows);
  dev_free_async(p->ctx, p->carry);
  p->magic = 0;
  delete p;
}

spmx_plan* plan_build(spmx_ctx* ctx, const spmx_csr* a, int strategy, unsigned parts, int dynamic,
                      uint64_t batch, unsigned flags) {
  if (strategy < 0 || strategy > 2) throw InvalidArg("make_partition: unknown strategy");
  if (dynamic) {
    // partition.cpp:91-94
    if (strategy != SPMX_ROW_SPLIT)
      throw InvalidArg("dynamic dispatch pairs with row-split only");
    if (batch == 0) throw InvalidArg("batch_size must be >= 1");
  }
  const u64 m = (u64)a->m, nnz = (u64)a->nnz;
  const bool exact = (flags & SPMX_EXACT_ORDER) != 0;
  if (parts == 0) {
    // strategy-level ranges T: a few per SM (the device refines them into chunks); exact-order
    // mode has no refinement, so there T is the work-list size itself
    const u64 ci = chunk_items_for(m + nnz, ctx->sm_count);
    const u64 fine = (m + nnz + ci - 1) / ci;
    const u64 want = exact ? fine : std::min<u64>(fine, (u64)ctx->sm_count * default_parts_per_sm());
    parts = (unsigned)std::min<u64>(std::max<u64>(want, 1), 1u << 30);
  }
  if (dynamic && nnz >= (1ull << 32))
    throw InvalidArg("dynamic dispatch: a claimed row batch must span fewer than 2^32 nonzeros");
  spmx_plan* p = new spmx_plan;
  AsyncScratch tmp(ctx);  // freed on every way out
  try {
    p->ctx = ctx;
    p->csr = a;
    p->strategy = strategy;
    p->parts = parts;
    p->flags = flags;
    p->dynamic = dynamic != 0;
    p->batch = batch ? batch : 128;
    // Dynamic row dispatch (DispatchCounter, partition.hpp:38-40: workers claim `batch` rows at a
    // time). SPMX_CLAIM_KERNEL runs it literally: persistent warps claim row batches with atomics
    // (spmm_dynamic_kernel), rows are never cut. Otherwise the same request is served by the
    // row-split work list below: its chunks ARE handed to the SMs dynamically, by the hardware's
    // CTA scheduler; in the default mode long rows are shared between chunks, in exact-order
    // mode they go to spmm_long_row_kernel (the claim kernel is row-granular: one lane group
    // walks c2's 39 542-nonzero row alone, 7.2 ms against 0.26 / 0.83 ms). The result is the
    // same either way (bitwise in exact-order mode).
    p->claims = p->dynamic && (flags & SPMX_CLAIM_KERNEL);
    if (p->claims) {
      p->counter = dev_alloc_async<u64>(ctx, 1);
      CUDA_CHECK(cudaMemsetAsync(p->counter, 0, sizeof(u64), ctx->stream));
      return p;
    }
    // 1. the strategy's row-snapped boundaries and RowRange list (bit-exact with the reference)
    u64* d_bnd = tmp.get<u64>((size_t)parts + 1);
    strategy_row_boundaries(ctx, a, strategy, parts, d_bnd);
    p->ranges = dev_alloc_async<u64>(ctx, 2 * (size_t)parts);
    spmx_dev::ranges_from_boundaries_kernel<<<blocks_for(parts), 256, 0, ctx->stream>>>(
        d_bnd, parts, p->ranges);
    post_launch();
    // 2. strategy-level merge-path diagonals
    u64* d_diag = tmp.get<u64>((size_t)parts + 1);
    if (strategy == SPMX_MERGE_SPLIT && !exact) {
      spmx_dev::merge_boundaries_kernel<<<blocks_for((u64)parts + 1), 256, 0, ctx->stream>>>(
          a->row_ptr, m, nnz, parts, 0, d_diag);
    } else {
      spmx_dev::boundaries_to_diagonals_kernel<<<blocks_for((u64)parts + 1), 256, 0, ctx->stream>>>(
          a->row_ptr, d_bnd, (u64)parts + 1, d_diag);
    }
    post_launch();
    // 3. work list: exact -> one chunk per range, boundaries on rows; otherwise ranges heavier
    //    than the chunk budget are cut along the merge path (interior cuts snapped to the start
    //    of short rows)
    u64 long_min = 0;
    if (exact) {
      // Long rows get work-list boundaries of their own (before and after the row), so that each
      // is a chunk by itself: the list of such rows is small, it is sorted and merged with the
      // strategy's boundaries on the host.
      p->n_chunks = parts;
      long_min = long_row_min();
      if (long_min && nnz >= long_min) {
        const size_t cap = (size_t)(nnz / long_min) + 1;
        u64* d_list = tmp.get<u64>(cap);
        unsigned* d_n = tmp.get<unsigned>(1);
        CUDA_CHECK(cudaMemsetAsync(d_n, 0, sizeof(unsigned), ctx->stream));
        spmx_dev::long_rows_kernel<<<validate_grid(ctx, m), 256, 0, ctx->stream>>>(a->row_ptr, m, long_min,
                                                                                    d_list, d_n);
        post_launch();
        unsigned n_long = 0;
        CUDA_CHECK(cudaMemcpyAsync(&n_long, d_n, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (n_long > 0) {
          std::vector<u64> rows(n_long), bnd((size_t)parts + 1);
          CUDA_CHECK(cudaMemcpyAsync(rows.data(), d_list, (size_t)n_long * 8, cudaMemcpyDeviceToHost, ctx->stream));
          CUDA_CHECK(cudaMemcpyAsync(bnd.data(), d_bnd, ((size_t)parts + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
          CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
          bnd.reserve(bnd.size() + 2 * (size_t)n_long);
          for (u64 r : rows) { bnd.push_back(r); bnd.push_back(r + 1); }
          std::sort(bnd.begin(), bnd.end());
          bnd.erase(std::unique(bnd.begin(), bnd.end()), bnd.end());
          p->n_chunks = bnd.size() - 1;
          u64* d_bnd2 = tmp.get<u64>(bnd.size());
          d_diag = tmp.get<u64>(bnd.size());
          CUDA_CHECK(cudaMemcpyAsync(d_bnd2, bnd.data(), bnd.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
          spmx_dev::boundaries_to_diagonals_kernel<<<blocks_for(bnd.size()), 256, 0, ctx->stream>>>(
              a->row_ptr, d_bnd2, bnd.size(), d_diag);
          post_launch();
          CUDA_CHECK(cudaStreamSynchronize(ctx->stream));  // bnd goes out of scope
          p->long_rows = dev_alloc_async<spmx_dev::LongRow>(ctx, (size_t)n_long);
        } else {
          long_min = 0;
        }
      } else {
        long_min = 0;
      }
      if (p->n_chunks >= 0xffffffffull) throw InvalidArg("plan: work list too long");
      p->chunk_row = dev_alloc_async<u64>(ctx, (size_t)p->n_chunks + 1);
      p->chunk_nnz = dev_alloc_async<u64>(ctx, (size_t)p->n_chunks + 1);
      spmx_dev::merge_search_kernel<<<blocks_for(p->n_chunks + 1), 256, 0, ctx->stream>>>(
          a->row_ptr, m, nnz, d_diag, p->n_chunks + 1, p->chunk_row, p->chunk_nnz);
      post_launch();
    } else {
      u64* d_cnt = tmp.get<u64>(parts);
      u64* d_off = tmp.get<u64>((size_t)parts + 1);
      // Tail taper: the last wave of the grid is cut into half-size chunks and its last third
      // into quarter-size chunks, so that the SMs run dry together (one wave = the chunks
      // resident at once, 64 per SM).
      const u64 ci = chunk_items_for(m + nnz, ctx->sm_count);
      const u64 wave = (u64)ctx->sm_count * 64 * ci;
      const u64 taper2 = wave * env_u64("SPMX_TAPER2_WAVES", 80) / 100;
      const u64 taper4 = wave * env_u64("SPMX_TAPER4_WAVES", 25) / 100;
      spmx_dev::count_chunks_kernel<<<blocks_for(parts), 256, 0, ctx->stream>>>(
          d_diag, parts, ci, (m + nnz) - std::min<u64>(taper2, (m + nnz) / 4),
          (m + nnz) - std::min<u64>(taper4, (m + nnz) / 12), d_cnt);
      post_launch();
      spmx_dev::exclusive_scan_kernel<<<1, 1024, 0, ctx->stream>>>(d_cnt, parts, d_off);
      post_launch();
      u64 total = 0;
      CUDA_CHECK(cudaMemcpyAsync(&total, d_off + parts, sizeof(u64), cudaMemcpyDeviceToHost,
                                 ctx->stream));
      CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
      p->n_chunks = total;
      p->chunk_row = dev_alloc_async<u64>(ctx, (size_t)total + 1);
      p->chunk_nnz = dev_alloc_async<u64>(ctx, (size_t)total + 1);
      spmx_dev::chunk_coords_kernel<<<blocks_for(total + 1), 256, 0, ctx->stream>>>(
          a->row_ptr, m, nnz, d_diag, d_off, parts, total, snap_len(), p->chunk_row, p->chunk_nnz);
      post_launch();
      if (total >= 0xffffffffull) throw InvalidArg("plan: work list too long");
      p->chain_first = dev_alloc_async<uint32_t>(ctx, (size_t)total);
      // long_list[0] doubles as the counter while the list is built: [count | entries...]
      const size_t long_cap = (size_t)(total / spmx_dev::kLongChain) + 1;
      p->long_buf = dev_alloc_async<uint32_t>(ctx, long_cap + 1);
      p->long_list = p->long_buf + 1;
      CUDA_CHECK(cudaMemsetAsync(p->long_buf, 0, sizeof(uint32_t), ctx->stream));
      p->short_buf = dev_alloc_async<uint32_t>(ctx, (size_t)total + 1);
      p->short_list = p->short_buf + 1;
      CUDA_CHECK(cudaMemsetAsync(p->short_buf, 0, sizeof(uint32_t), ctx->stream));
      spmx_dev::chain_first_kernel<<<blocks_for(total), 256, 0, ctx->stream>>>(
          a->row_ptr, p->chunk_row, p->chunk_nnz, total, m, p->chain_first, p->long_list,
          p->long_buf, p->short_list, p->short_buf);
      post_launch();
      CUDA_CHECK(cudaMemcpyAsync(&p->n_long, p->long_buf, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                 ctx->stream));
      CUDA_CHECK(cudaMemcpyAsync(&p->n_short, p->short_buf, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                 ctx->stream));
      CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
      // a piece ends inside a row only where a chain of carries exists: without chains no
      // carry is ever written and the fix-up has nothing to do
      p->may_carry = p->n_long + p->n_short > 0;
    }
    if (p->n_chunks > 0) {
      p->work = dev_alloc_async<spmx_dev::WorkItem>(ctx, (size_t)p->n_chunks);
      unsigned* d_nlong = tmp.get<unsigned>(1);
      CUDA_CHECK(cudaMemsetAsync(d_nlong, 0, sizeof(unsigned), ctx->stream));
      spmx_dev::work_items_kernel<spmx_dev::WorkItem, spmx_dev::LongRow>
          <<<blocks_for(p->n_chunks, spmx_dev::kSortTile), spmx_dev::kSortTile, 0, ctx->stream>>>(
              p->chunk_row, p->chunk_nnz, p->n_chunks, p->work, p->long_rows ? long_min : 0, p->long_rows,
              d_nlong);
      post_launch();
      CUDA_CHECK(cudaMemcpyAsync(&p->n_long_rows, d_nlong, sizeof(unsigned), cudaMemcpyDeviceToHost,
                                 ctx->stream));
      if (p->long_rows) {  // longest rows first: a row is one CTA's serial chain, the tail is the longest
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        std::vector<spmx_dev::LongRow> lr(p->n_long_rows);
        CUDA_CHECK(cudaMemcpyAsync(lr.data(), p->long_rows, lr.size() * sizeof(spmx_dev::LongRow),
                                   cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        std::sort(lr.begin(), lr.end(), [](const spmx_dev::LongRow& x, const spmx_dev::LongRow& y) {
          const u64 lx = x.j1 - x.j0, ly = y.j1 - y.j0;
          return lx != ly ? lx > ly : x.row < y.row;
        });
        CUDA_CHECK(cudaMemcpyAsync(p->long_rows, lr.data(), lr.size() * sizeof(spmx_dev::LongRow),
                                   cudaMemcpyHostToDevice, ctx->stream));
        CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
      }
    }
    // a work item's nonzero offsets are 32-bit inside the kernel: every chunk must span fewer
    // than 2^32 nonzeros (only exact-order plans, one chunk per strategy range, can exceed it)
    u64 max_span = 0;
    if (p->n_chunks > 0 && nnz >= (1ull << 32)) {
      u64* d_max = tmp.get<u64>(1);
      CUDA_CHECK(cudaMemsetAsync(d_max, 0, sizeof(u64), ctx->stream));
      spmx_dev::max_chunk_span_kernel<<<blocks_for(p->n_chunks), 256, 0, ctx->stream>>>(
          p->chunk_nnz, p->n_chunks, d_max);
      post_launch();
      CUDA_CHECK(cudaMemcpyAsync(&max_span, d_max, sizeof(u64), cudaMemcpyDeviceToHost, ctx->stream));
    }
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (max_span >= (1ull << 32))
      throw InvalidArg("plan: a range spans 2^32 or more nonzeros (use more parts)");
    return p;
  } catch (...) {
    plan_free(p);
    throw;
  }
}

void* ws_get(spmx_ctx* ctx, int slot, size_t bytes) {
  if (ctx->ws_bytes[slot] < bytes) {
    if (ctx->ws[slot]) CUDA_CHECK(cudaFree(ctx->ws[slot]));
    ctx->ws[slot] = nullptr;
    ctx->ws_bytes[slot] = 0;
    CUDA_CHECK(cudaMalloc(&ctx->ws[slot], bytes ? bytes : 1));
    ctx->ws_bytes[slot] = bytes;
  }
  return ctx->ws[slot];
}

}  // namespace

extern "C" {

const char* spmx_last_error(void) { return g_last_error.c_str(); }
int spmx_abi_version(void) { return 2; }
const char* spmx_build_info(void) { return g_build_info; }
uint64_t spmx_kernel_launch_count(void) { return g_launches.load(); }

int spmx_ctx_create(int device, void* stream, spmx_ctx** out) {
  return guarded([&] {
    if (!out) throw InvalidArg("spmx_ctx_create: null out");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
      throw std::runtime_error(
          "no CUDA device: this library has no CPU fallback (cudaGetDeviceCount: " +
          std::string(cudaGetErrorString(e)) + ")");
    if (device < 0 || device >= count) throw InvalidArg("spmx_ctx_create: no such device");
    CUDA_CHECK(cudaSetDevice(device));
    spmx_ctx* c = new spmx_ctx;
    c->device = device;
    if (stream) {
      c->stream = (cudaStream_t)stream;
    } else {
      CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    CUDA_CHECK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    CUDA_CHECK(cudaEventCreate(&c->ev0));
    CUDA_CHECK(cudaEventCreate(&c->ev1));
    c->d_err = dev_alloc<int>(1);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = ~0ull;  // do not hand pool memory back to the OS between plans
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    *out = c;
  });
}

int spmx_ctx_destroy(spmx_ctx* ctx) {
  return guarded([&] {
    check(ctx);
    cudaStreamSynchronize(ctx->stream);
    for (int i = 0; i < 5; ++i)
      if (ctx->ws[i]) cudaFree(ctx->ws[i]);
    cudaFree(ctx->d_err);
    for (cudaEvent_t e : ctx->pipe_events) cudaEventDestroy(e);
    if (ctx->s_compute) cudaStreamDestroy(ctx->s_compute);
    if (ctx->s_d2h) cudaStreamDestroy(ctx->s_d2h);
    if (ctx->s_x) cudaStreamDestroy(ctx->s_x);
    if (ctx->s_aux) cudaStreamDestroy(ctx->s_aux);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    cudaEventDestroy(ctx->ev0);
    cudaEventDestroy(ctx->ev1);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    ctx->magic = 0;
    delete ctx;
  });
}

int spmx_ctx_synchronize(spmx_ctx* ctx) {
  return guarded([&] { CUDA_CHECK(cudaStreamSynchronize(check(ctx)->stream)); });
}

int spmx_ctx_sm_count(spmx_ctx* ctx, int* out) {
  return guarded([&] { *out = check(ctx)->sm_count; });
}

int spmx_dev_alloc(spmx_ctx* ctx, size_t bytes, void** out) {
  return guarded([&] {
    check(ctx);
    CUDA_CHECK(cudaMalloc(out, bytes ? bytes : 1));
  });
}
int spmx_dev_free(spmx_ctx* ctx, void* ptr) {
  return guarded([&] {
    check(ctx);
    CUDA_CHECK(cudaFree(ptr));
  });
}
namespace {

// Worker threads for copies of pageable host memory (spmx_stage.cuh): half of the host's hardware
// threads, at most 8 up and 6 down (measured on the 16-thread hosts of the B200 pool: c2 through
// spmx_spmm_host from pageable arrays 52 -> 15.4 ms; more threads oversubscribe the memory bus).
// SPMX_HOST_STAGE_THREADS = 0 leaves pageable copies to the driver.
int stage_threads_up() {
  const unsigned hw = std::max(4u, std::thread::hardware_concurrency());
  return (int)env_u64("SPMX_HOST_STAGE_THREADS", std::min(8u, hw / 2));
}
int stage_threads_down() {
  const unsigned hw = std::max(4u, std::thread::hardware_concurrency());
  return (int)env_u64("SPMX_HOST_STAGE_THREADS_DOWN", std::min<u64>(std::min(6u, std::max(2u, hw / 2 - 2)),
                                                                     (u64)std::max(1, stage_threads_up())));
}
constexpr size_t kStageMinBytes = 1u << 20;  // smaller copies are not worth a hand-over

bool stage_this(const void* host, size_t bytes) {
  return bytes >= kStageMinBytes && stage_threads_up() > 0 && spmx_stage::Stager::pageable(host);
}
spmx_stage::Stager& stager_up(spmx_ctx* ctx) {
  return spmx_stage::shared_stager(ctx->device, true, stage_threads_up());
}
spmx_stage::Stager& stager_down(spmx_ctx* ctx) {
  return spmx_stage::shared_stager(ctx->device, false, stage_threads_down());
}

// host -> device on `st`. Returns once the copy is enqueued (pinned source: asynchronous as
// cudaMemcpyAsync is; pageable source: the source has been read when this returns, as with
// cudaMemcpyAsync from pageable memory).
void copy_h2d(spmx_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (stage_this(src, bytes)) {
    spmx_stage::Stager::wait(stager_up(ctx).h2d(dst, src, bytes, st));
    return;
  }
  CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
}
// device -> host on `st`; with a pageable destination the data has arrived when this returns
void copy_d2h(spmx_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (stage_this(dst, bytes)) {
    spmx_stage::Stager::wait(stager_down(ctx).d2h(dst, src, bytes, st));
    return;
  }
  CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
}

}  // namespace

int spmx_h2d(spmx_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guarded([&] { copy_h2d(check(ctx), dst, src, bytes, ctx->stream); });
}
int spmx_d2h(spmx_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guarded([&] { copy_d2h(check(ctx), dst, src, bytes, ctx->stream); });
}
int spmx_host_alloc_pinned(size_t bytes, void** out) {
  return guarded([&] { CUDA_CHECK(cudaMallocHost(out, bytes ? bytes : 1)); });
}
int spmx_host_free_pinned(void* ptr) {
  return guarded([&] { CUDA_CHECK(cudaFreeHost(ptr)); });
}

int spmx_csr_upload(spmx_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const uint64_t* row_ptr,
                    const uint32_t* col, const float* vals, spmx_csr** out) {
  return guarded([&] {
    check(ctx);
    if (!out) throw InvalidArg("spmx_csr_upload: null out");
    if (m < 0 || n < 0 || nnz < 0) throw InvalidArg("invalid CSR: negative dimension");
    if (!row_ptr || (nnz > 0 && (!col || !vals))) throw InvalidArg("invalid CSR: null array");
    spmx_csr* a = new spmx_csr;
    a->ctx = ctx;
    a->m = m;
    a->n = n;
    a->nnz = nnz;
    a->owned = true;
    try {
      a->row_ptr = dev_alloc<u64>((size_t)m + 1);
      a->col = dev_alloc<uint32_t>((size_t)nnz);
      a->vals = dev_alloc<float>((size_t)nnz);
      copy_h2d(ctx, a->row_ptr, row_ptr, ((size_t)m + 1) * 8, ctx->stream);
      copy_h2d(ctx, a->col, col, (size_t)nnz * 4, ctx->stream);
      copy_h2d(ctx, a->vals, vals, (size_t)nnz * 4, ctx->stream);
      validate_on_device(ctx, a);
    } catch (...) {
      spmx_csr_destroy(a);
      throw;
    }
    *out = a;
  });
}

int spmx_rowptr_upload(spmx_ctx* ctx, int64_t m, int64_t nnz, const uint64_t* row_ptr,
                       spmx_csr** out) {
  return guarded([&] {
    check(ctx);
    if (!out) throw InvalidArg("spmx_rowptr_upload: null out");
    if (m < 0 || nnz < 0) throw InvalidArg("invalid CSR: negative dimension");
    if (!row_ptr) throw InvalidArg("invalid CSR: null array");
    spmx_csr* a = new spmx_csr;
    a->ctx = ctx;
    a->m = m;
    a->n = 0;
    a->nnz = nnz;
    a->owned = true;
    a->structure_only = true;
    try {
      a->row_ptr = dev_alloc<u64>((size_t)m + 1);
      CUDA_CHECK(cudaMemcpyAsync(a->row_ptr, row_ptr, ((size_t)m + 1) * 8, cudaMemcpyHostToDevice,
                                 ctx->stream));
      CUDA_CHECK(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
      spmx_dev::validate_row_ptr_kernel<<<validate_grid(ctx, (u64)m), 256, 0, ctx->stream>>>(
          a->row_ptr, (u64)m, (u64)nnz, ctx->d_err);
      post_launch();
      int err = 0;
      CUDA_CHECK(cudaMemcpyAsync(&err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
      if (err) throw InvalidArg(std::string("invalid CSR: ") + csr_error_text(err));
    } catch (...) {
      spmx_csr_destroy(a);
      throw;
    }
    *out = a;
  });
}

int spmx_csr_wrap_device(spmx_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const uint64_t* d_rp,
                         const uint32_t* d_col, const float* d_vals, int validate,
                         spmx_csr** out) {
  return guarded([&] {
    check(ctx);
    if (!out) throw InvalidArg("spmx_csr_wrap_device: null out");
    if (m < 0 || n < 0 || nnz < 0) throw InvalidArg("invalid CSR: negative dimension");
    if (!d_rp) throw InvalidArg("invalid CSR: null row_ptr");
    spmx_csr* a = new spmx_csr;
    a->ctx = ctx;
    a->m = m;
    a->n = n;
    a->nnz = nnz;
    a->row_ptr = (u64*)d_rp;
    a->col = (uint32_t*)d_col;
    a->vals = (float*)d_vals;
    a->owned = false;
    try {
      if (validate) validate_on_device(ctx, a);
    } catch (...) {
      spmx_csr_destroy(a);
      throw;
    }
    *out = a;
  });
}

int spmx_csr_destroy(spmx_csr* a) {
  return guarded([&] {
    check((const spmx_csr*)a);
    if (a->owned) {
      cudaFree(a->row_ptr);
      cudaFree(a->col);
      cudaFree(a->vals);
    }
    a->magic = 0;
    delete a;
  });
}

int spmx_csr_dims(const spmx_csr* a, int64_t* m, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    check(a);
    if (m) *m = a->m;
    if (n) *n = a->n;
    if (nnz) *nnz = a->nnz;
  });
}

int spmx_split_rows_static(spmx_ctx* ctx, uint64_t m, unsigned parts, uint64_t* out) {
  return guarded([&] {
    check(ctx);
    if (parts == 0) throw InvalidArg("split_rows_static: zero threads");
    AsyncScratch tmp(ctx);
    u64* d_bnd = tmp.get<u64>((size_t)parts + 1);
    spmx_dev::row_boundaries_kernel<<<blocks_for((u64)parts + 1), 256, 0, ctx->stream>>>(
        (u64)m, parts, d_bnd);
    post_launch();
    ranges_to_host(ctx, d_bnd, parts, out);
  });
}

int spmx_split_nnz(spmx_ctx* ctx, const spmx_csr* a, unsigned parts, uint64_t* out) {
  return guarded([&] {
    check(ctx);
    check(a);
    if (parts == 0) throw InvalidArg("split_nnz: zero threads");
    AsyncScratch tmp(ctx);
    u64* d_bnd = tmp.get<u64>((size_t)parts + 1);
    strategy_row_boundaries(ctx, a, SPMX_NNZ_SPLIT, parts, d_bnd);
    ranges_to_host(ctx, d_bnd, parts, out);
  });
}

int spmx_split_merge(spmx_ctx* ctx, const spmx_csr* a, unsigned parts, uint64_t* out) {
  return guarded([&] {
    check(ctx);
    check(a);
    if (parts == 0) throw InvalidArg("split_merge: zero threads");
    AsyncScratch tmp(ctx);
    u64* d_bnd = tmp.get<u64>((size_t)parts + 1);
    strategy_row_boundaries(ctx, a, SPMX_MERGE_SPLIT, parts, d_bnd);
    ranges_to_host(ctx, d_bnd, parts, out);
  });
}

int spmx_merge_path_search(spmx_ctx* ctx, const spmx_csr* a, size_t n_diag, const uint64_t* k,
                           uint64_t* out_i, uint64_t* out_j) {
  return guarded([&] {
    check(ctx);
    check(a);
    const u64 lim = (u64)a->m + (u64)a->nnz;
    for (size_t t = 0; t < n_diag; ++t)
      if (k[t] > lim) throw InvalidArg("merge_path_search: diagonal out of range");
    if (n_diag == 0) return;
    u64* d_k = dev_alloc<u64>(n_diag);
    u64* d_i = dev_alloc<u64>(n_diag);
    u64* d_j = dev_alloc<u64>(n_diag);
    CUDA_CHECK(cudaMemcpyAsync(d_k, k, n_diag * 8, cudaMemcpyHostToDevice, ctx->stream));
    spmx_dev::merge_search_kernel<<<blocks_for(n_diag), 256, 0, ctx->stream>>>(
        a->row_ptr, (u64)a->m, (u64)a->nnz, d_k, n_diag, d_i, d_j);
    post_launch();
    CUDA_CHECK(cudaMemcpyAsync(out_i, d_i, n_diag * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaMemcpyAsync(out_j, d_j, n_diag * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    CUDA_CHECK(cudaFree(d_k));
    CUDA_CHECK(cudaFree(d_i));
    CUDA_CHECK(cudaFree(d_j));
  });
}

int spmx_next_batch_claims(spmx_ctx* ctx, uint64_t m, uint64_t batch, size_t n_claims,
                           uint64_t* out) {
  return guarded([&] {
    check(ctx);
    if (batch == 0) throw InvalidArg("batch_size must be >= 1");
    if (n_claims == 0) return;
    u64* d_counter = dev_alloc<u64>(1);
    u64* d_out = dev_alloc<u64>(2 * n_claims);
    CUDA_CHECK(cudaMemsetAsync(d_counter, 0, 8, ctx->stream));
    spmx_dev::next_batch_claims_kernel<<<blocks_for(n_claims), 256, 0, ctx->stream>>>(
        d_counter, (u64)batch, (u64)m, (u64)n_claims, d_out);
    post_launch();
    CUDA_CHECK(cudaMemcpyAsync(out, d_out, 2 * n_claims * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    CUDA_CHECK(cudaFree(d_counter));
    CUDA_CHECK(cudaFree(d_out));
  });
}

int spmx_plan_create(spmx_ctx* ctx, const spmx_csr* a, int strategy, unsigned parts, int dynamic,
                     uint64_t batch, unsigned flags, spmx_plan** out) {
  return guarded([&] {
    check(ctx);
    check(a);
    if (!out) throw InvalidArg("spmx_plan_create: null out");
    if (a->ctx != ctx) throw LogicErr("spmx_plan_create: csr belongs to another context");
    *out = plan_build(ctx, a, strategy, parts, dynamic, batch, flags);
  });
}

int spmx_plan_destroy(spmx_plan* p) {
  return guarded([&] {
    check((const spmx_plan*)p);
    CUDA_CHECK(cudaSetDevice(p->ctx->device));
    plan_free(p);
  });
}

int spmx_plan_info(const spmx_plan* p, unsigned* parts, uint64_t* n_chunks, int* dynamic) {
  return guarded([&] {
    check(p);
    if (parts) *parts = p->parts;
    if (n_chunks) *n_chunks = p->n_chunks;
    if (dynamic) *dynamic = p->dynamic ? 1 : 0;
  });
}

int spmx_plan_ranges(const spmx_plan* p, uint64_t* out) {
  return guarded([&] {
    check(p);
    check(p->ctx);
    if (p->dynamic) return;  // WorkPartition.ranges is empty under dynamic dispatch
    CUDA_CHECK(cudaMemcpyAsync(out, p->ranges, 2 * (size_t)p->parts * 8, cudaMemcpyDeviceToHost,
                               p->ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(p->ctx->stream));
  });
}

int spmx_plan_chunks(const spmx_plan* p, uint64_t* out_row, uint64_t* out_nnz) {
  return guarded([&] {
    check(p);
    check(p->ctx);
    if (p->claims) return;
    const size_t bytes = ((size_t)p->n_chunks + 1) * 8;
    CUDA_CHECK(cudaMemcpyAsync(out_row, p->chunk_row, bytes, cudaMemcpyDeviceToHost, p->ctx->stream));
    CUDA_CHECK(cudaMemcpyAsync(out_nnz, p->chunk_nnz, bytes, cudaMemcpyDeviceToHost, p->ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(p->ctx->stream));
  });
}

int spmx_spmm(spmx_ctx* ctx, const spmx_plan* plan, const spmx_csr* a, const float* d_x,
              int64_t x_rows, int64_t d, float* d_y, float* elapsed_ms) {
  return guarded([&] {
    check(ctx);
    check(plan);
    check(a);
    if (plan->csr != a || plan->ctx != ctx)
      throw LogicErr("spmx_spmm: plan was built for another matrix or context");
    if (a->structure_only) throw LogicErr("spmx_spmm: structure-only CSR handle (spmx_rowptr_upload)");
    if (a->n != x_rows) throw InvalidArg("run_spmm: A.n != X.rows");  // executor.cpp:38
    if (d < 1) throw InvalidArg("run_spmm: X.cols must be >= 1");
    if (d > (1 << 30)) throw InvalidArg("run_spmm: X.cols too large");
    if ((!d_x && a->n > 0) || (!d_y && a->m > 0)) throw InvalidArg("run_spmm: null X or Y");
    if (elapsed_ms) CUDA_CHECK(cudaEventRecord(ctx->ev0, ctx->stream));
    run_kernels(ctx, plan, a, d_x, d, d_y, ctx->stream, 0, plan->n_chunks, nullptr);
    if (elapsed_ms) {
      CUDA_CHECK(cudaEventRecord(ctx->ev1, ctx->stream));
      CUDA_CHECK(cudaEventSynchronize(ctx->ev1));
      CUDA_CHECK(cudaEventElapsedTime(elapsed_ms, ctx->ev0, ctx->ev1));
    }
  });
}

int spmx_spmm_host(spmx_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const uint64_t* row_ptr,
                   const uint32_t* col, const float* vals, const float* x, int64_t x_rows,
                   int64_t d, float* y, int strategy, unsigned parts, int dynamic, uint64_t batch,
                   unsigned flags, double* times_ms) {
  // Pipeline over four streams (the transfers dominate: PCIe moves ~8 B per nonzero up and
  // 4*d B per row down, the kernel needs a fraction of that time):
  //   stream 0  H2D row_ptr -> validate + plan (the plan needs row_ptr only) -> wait for X
  //             -> H2D col/vals of row block 0, 1, ...
  //   stream 1  per block: validate columns, SpMM over the block's chunks, carry fix-up
  //   stream 2  per block: D2H of the Y rows that end in the block
  //   stream 3  H2D X (while the plan is built on stream 0)
  // Blocks are runs of whole chunks of the work list, so every Y row is final when its
  // block's kernels have run. Dynamic-dispatch plans have no work list: one block.
  return guarded([&] {
    check(ctx);
    if (m < 0 || n < 0 || nnz < 0) throw InvalidArg("invalid CSR: negative dimension");
    if (n != x_rows) throw InvalidArg("run_spmm: A.n != X.rows");
    if (d < 1) throw InvalidArg("run_spmm: X.cols must be >= 1");
    if (!row_ptr || (!x && n > 0) || (!y && m > 0) || (nnz > 0 && (!col || !vals)))
      throw InvalidArg("run_spmm: null array");
    if (!ctx->s_compute) {
      CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->s_compute, cudaStreamNonBlocking));
      CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking));
      CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->s_x, cudaStreamNonBlocking));
    }
    cudaStream_t s0 = ctx->stream, s1 = ctx->s_compute, s2 = ctx->s_d2h, s3 = ctx->s_x;
    // Pageable host arrays (what a caller of the reference's run_spmm holds: std::vector) are
    // staged through pinned slots by several host threads instead of the driver's single one
    // (spmx_stage.cuh); pinned or registered arrays go to the copy engines directly.
    using spmx_stage::Stager;
    auto staged = [&](const void* p, size_t bytes) { return stage_this(p, bytes); };
    const size_t x_bytes = (size_t)n * (size_t)d * 4, y_bytes = (size_t)m * (size_t)d * 4;
    const bool st_rp = staged(row_ptr, ((size_t)m + 1) * 8), st_x = staged(x, x_bytes);
    const bool st_col = staged(col, (size_t)nnz * 4), st_val = staged(vals, (size_t)nnz * 4);
    const bool st_y = staged(y, y_bytes);
    std::vector<Stager::Ticket> pending;  // staged copies not yet waited for
    auto drain_quiet = [&]() noexcept {
      for (auto& t : pending) Stager::wait_quiet(t);
      pending.clear();
    };
    auto up = [&](void* dst, const void* src, size_t bytes, bool stage, cudaStream_t st) -> Stager::Ticket {
      if (bytes == 0) return nullptr;
      if (stage) {
        pending.push_back(stager_up(ctx).h2d(dst, src, bytes, st));
        return pending.back();
      }
      CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
      return nullptr;
    };
    constexpr int kMaxBlocks = 32;
    cudaEvent_t ev_t[4];            // timing marks on stream 0 / 2
    cudaEvent_t ev_x, ev_in[kMaxBlocks], ev_done[kMaxBlocks];
    size_t next_event = 0;
    auto mk = [&](cudaEvent_t& e, bool) {
      if (next_event == ctx->pipe_events.size()) {
        cudaEvent_t fresh;
        CUDA_CHECK(cudaEventCreate(&fresh));
        ctx->pipe_events.push_back(fresh);
      }
      e = ctx->pipe_events[next_event++];
    };
    u64* d_rp = (u64*)ws_get(ctx, 0, ((size_t)m + 1) * 8);
    uint32_t* d_col = (uint32_t*)ws_get(ctx, 1, (size_t)nnz * 4);
    float* d_vals = (float*)ws_get(ctx, 2, (size_t)nnz * 4);
    float* d_x = (float*)ws_get(ctx, 3, (size_t)n * (size_t)d * 4);
    float* d_y = (float*)ws_get(ctx, 4, (size_t)m * (size_t)d * 4);
    spmx_csr a;
    a.ctx = ctx;
    a.m = m;
    a.n = n;
    a.nnz = nnz;
    a.row_ptr = d_rp;
    a.col = d_col;
    a.vals = d_vals;
    spmx_plan* plan = nullptr;
    auto cleanup = [&] {
      if (plan) plan_free(plan);
      plan = nullptr;
      a.magic = 0;
    };
    try {
      for (auto& e : ev_t) mk(e, true);
      mk(ev_x, false);
      for (int b = 0; b < kMaxBlocks; ++b) { mk(ev_in[b], false); mk(ev_done[b], false); }
      const auto t_host0 = std::chrono::steady_clock::now();
      CUDA_CHECK(cudaEventRecord(ev_t[0], s0));
      Stager::wait(up(d_rp, row_ptr, ((size_t)m + 1) * 8, st_rp, s0));  // enqueued: stream 0 orders the rest
      // X moves on its own stream while the plan is being built from row_ptr
      CUDA_CHECK(cudaStreamWaitEvent(s3, ev_t[0], 0));
      Stager::Ticket x_ticket = up(d_x, x, x_bytes, st_x, s3);
      if (!x_ticket) CUDA_CHECK(cudaEventRecord(ev_x, s3));
      CUDA_CHECK(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), s0));
      spmx_dev::validate_row_ptr_kernel<<<validate_grid(ctx, (u64)m), 256, 0, s0>>>(
          d_rp, (u64)m, (u64)nnz, ctx->d_err);
      post_launch();
      int err = 0;
      CUDA_CHECK(cudaMemcpyAsync(&err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, s0));
      CUDA_CHECK(cudaStreamSynchronize(s0));
      if (err) throw InvalidArg(std::string("invalid CSR: ") + csr_error_text(err));
      // the plan (a fraction of a millisecond, stream-ordered allocations only) overlaps the
      // X upload; col/vals follow X so that they do not take bandwidth from it
      plan = plan_build(ctx, &a, strategy, parts, dynamic, batch, flags);  // syncs stream 0
      ensure_carry(plan, d);
      const auto t_host1 = std::chrono::steady_clock::now();

      // blocks = runs of whole chunks with about equal nonzero counts
      int nblocks = 1;
      std::vector<u64> cb{0, plan->n_chunks}, row_b{0, (u64)m}, nnz_b{0, (u64)nnz};
      // (long rows of an exact-order plan read nonzeros of every block: no block pipeline then)
      if (!plan->claims && plan->n_long_rows == 0 && plan->n_chunks >= 64 && nnz > (1 << 20)) {
        nblocks = (int)std::min<u64>(kMaxBlocks, std::max<u64>(2, env_u64("SPMX_HOST_BLOCKS", 8)));
        cb.assign(nblocks + 1, 0);
        row_b.assign(nblocks + 1, 0);
        nnz_b.assign(nblocks + 1, 0);
        // whole sort tiles, so that a block's launch slots hold exactly the block's chunks
        for (int b = 0; b < nblocks; ++b)
          cb[b] = plan->n_chunks * (u64)b / (u64)nblocks / spmx_dev::kSortTile * spmx_dev::kSortTile;
        cb[nblocks] = plan->n_chunks;
        for (int b = 0; b <= nblocks; ++b) {
          CUDA_CHECK(cudaMemcpyAsync(&row_b[b], plan->chunk_row + cb[b], 8, cudaMemcpyDeviceToHost, s0));
          CUDA_CHECK(cudaMemcpyAsync(&nnz_b[b], plan->chunk_nnz + cb[b], 8, cudaMemcpyDeviceToHost, s0));
        }
        CUDA_CHECK(cudaStreamSynchronize(s0));
        // a block's first chunk may start inside a row whose head is in the previous block; the
        // nonzeros it needs still start at its own chunk_nnz, which is what nnz_b holds
      }
      if (x_ticket) {  // staged X: every piece has to be on stream 3 before the event that marks its end
        Stager::wait(x_ticket);
        CUDA_CHECK(cudaEventRecord(ev_x, s3));
      }
      CUDA_CHECK(cudaStreamWaitEvent(s0, ev_x, 0));
      CUDA_CHECK(cudaEventRecord(ev_t[1], s0));
      // The blocks go LAST TO FIRST: on a power-law matrix the last block (equal merge items)
      // holds the most rows and the fewest nonzeros, i.e. the smallest upload and the largest
      // Y download, so the download engine gets its work early and stays busy while the
      // nonzero-heavy blocks are still arriving (c2: 11.3 -> 10.7 ms per call). The one row per
      // block whose head lies in the block before it (computed later in this order) has its
      // carry chain deferred to the end and is downloaded again then.
      for (int bi = 0; bi < nblocks; ++bi) {
        const int b = nblocks - 1 - bi;
        const u64 n0 = nnz_b[b], n1 = nnz_b[b + 1];
        if (n1 > n0) {
          Stager::Ticket tc = up(d_col + n0, col + n0, (n1 - n0) * 4, st_col, s0);
          Stager::Ticket tv = up(d_vals + n0, vals + n0, (n1 - n0) * 4, st_val, s0);
          Stager::wait(tc);
          Stager::wait(tv);
        }
        CUDA_CHECK(cudaEventRecord(ev_in[b], s0));
        CUDA_CHECK(cudaStreamWaitEvent(s1, ev_in[b], 0));
        if (bi == 0) CUDA_CHECK(cudaStreamWaitEvent(s1, ev_x, 0));
        if (n1 > n0) {
          spmx_dev::validate_cols_kernel<<<validate_grid(ctx, n1 - n0), 256, 0, s1>>>(
              d_col + n0, n1 - n0, (u64)n, ctx->d_err);
          post_launch();
        }
        run_kernels(ctx, plan, &a, d_x, d, d_y, s1, cb[b], cb[b + 1], ctx->d_err, /*first_lo=*/cb[b]);
        CUDA_CHECK(cudaEventRecord(ev_done[b], s1));
        CUDA_CHECK(cudaStreamWaitEvent(s2, ev_done[b], 0));
        const u64 r0 = row_b[b], r1 = (b + 1 == nblocks) ? (u64)m : row_b[b + 1];
        if (bi == 0) CUDA_CHECK(cudaEventRecord(ev_t[2], s2));
        if (r1 > r0) {
          if (st_y)  // done when the rows are in the caller's array (waited for below)
            pending.push_back(stager_down(ctx).d2h(y + r0 * (size_t)d, d_y + r0 * (size_t)d,
                                                   (r1 - r0) * (size_t)d * 4, s2));
          else
            CUDA_CHECK(cudaMemcpyAsync(y + r0 * (size_t)d, d_y + r0 * (size_t)d, (r1 - r0) * (size_t)d * 4,
                                       cudaMemcpyDeviceToHost, s2));
        }
      }
      if (nblocks > 1 && plan->may_carry) {
        // deferred chains: those closed in block b whose first partial is in an earlier block
        for (int b = 1; b < nblocks; ++b)
          run_kernels(ctx, plan, &a, d_x, d, d_y, s1, cb[b], cb[b + 1], ctx->d_err, 0, cb[b],
                      /*fixup_only=*/true);
        CUDA_CHECK(cudaEventRecord(ev_done[0], s1));
        CUDA_CHECK(cudaStreamWaitEvent(s2, ev_done[0], 0));
        // staged downloads write the caller's array from worker threads: the rows downloaded
        // again below must land after the block copies that hold their earlier values
        for (auto& t : pending) Stager::wait(t);
        pending.clear();
        for (int b = 1; b < nblocks; ++b) {
          const u64 r = row_b[b];  // the row block b starts in
          if (r < (u64)m)
            CUDA_CHECK(cudaMemcpyAsync(y + r * (size_t)d, d_y + r * (size_t)d, (size_t)d * 4,
                                       cudaMemcpyDeviceToHost, s2));
        }
      }
      for (auto& t : pending) Stager::wait(t);
      pending.clear();
      CUDA_CHECK(cudaEventRecord(ev_t[3], s2));
      CUDA_CHECK(cudaMemcpyAsync(&err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, s2));
      CUDA_CHECK(cudaStreamSynchronize(s2));
      CUDA_CHECK(cudaStreamSynchronize(s1));
      CUDA_CHECK(cudaStreamSynchronize(s0));
      if (err) throw InvalidArg(std::string("invalid CSR: ") + csr_error_text(err));
      if (times_ms) {
        float t = 0.f;
        // {row_ptr upload + plan (host clock), -, first block ready -> last Y byte, -, total, blocks}
        times_ms[0] = std::chrono::duration<double, std::milli>(t_host1 - t_host0).count();
        times_ms[1] = times_ms[0];
        CUDA_CHECK(cudaEventElapsedTime(&t, ev_t[2], ev_t[3]));
        times_ms[2] = 0.0;
        times_ms[3] = t;
        CUDA_CHECK(cudaEventElapsedTime(&t, ev_t[0], ev_t[1]));
        const double head = t;
        times_ms[4] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
        times_ms[2] = times_ms[4] - times_ms[3] - head > 0 ? times_ms[4] - times_ms[3] - head : 0.0;
        times_ms[5] = (double)nblocks;
      }
    } catch (...) {
      drain_quiet();  // workers still read the caller's arrays / write Y
      cudaStreamSynchronize(s0);
      cudaStreamSynchronize(s1);
      cudaStreamSynchronize(s2);
      cudaStreamSynchronize(s3);
      cleanup();
      throw;
    }
    cleanup();
  });
}

int spmx_spmm_reference(spmx_ctx* ctx, const spmx_csr* a, const float* d_x, int64_t x_rows,
                        int64_t d, float* d_y) {
  return guarded([&] {
    check(ctx);
    check(a);
    if (a->structure_only) throw LogicErr("spmm_reference: structure-only CSR handle");
    if (a->n != x_rows) throw InvalidArg("spmm_reference: A.n != X.rows");  // reference.cpp:11
    if (d < 1) throw InvalidArg("spmm_reference: X.cols must be >= 1");
    const u64 total = (u64)a->m * (u64)d;
    if (total == 0) return;
    spmx_dev::spmm_unfused_reference_kernel<<<blocks_for(total), 256, 0, ctx->stream>>>(
        a->row_ptr, a->col, a->vals, d_x, d_y, (u64)a->m, (int)d);
    post_launch();
  });
}

int spmx_max_relative_error(spmx_ctx* ctx, const float* d_y, const float* d_ref, size_t count,
                            double* out) {
  return guarded([&] {
    check(ctx);
    unsigned long long* d_bits = dev_alloc<unsigned long long>(1);
    CUDA_CHECK(cudaMemsetAsync(d_bits, 0, 8, ctx->stream));
    if (count) {
      const unsigned nb = (unsigned)std::min<u64>((u64)ctx->sm_count * 8, (count + 255) / 256);
      spmx_dev::max_rel_err_kernel<<<nb, 256, 0, ctx->stream>>>(d_y, d_ref, (u64)count, d_bits);
      post_launch();
    }
    unsigned long long bits = 0;
    CUDA_CHECK(cudaMemcpyAsync(&bits, d_bits, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    CUDA_CHECK(cudaFree(d_bits));
    std::memcpy(out, &bits, 8);
  });
}

int spmx_probe_l2_to_sm(spmx_ctx* ctx, int repeats, double* out_tbs, double* out_ms) {
  return guarded([&] {
    check(ctx);
    if (repeats < 1) repeats = 1;
    constexpr size_t kBytes = 64u << 20;  // resident in the 126 MB L2
    constexpr int kSteps = 2048;
    const int warps_per_sm[] = {24, 32, 40, 48};  // the ceiling is the best any occupancy reaches
    float4* buf = (float4*)dev_alloc<char>(kBytes);
    float* sink = dev_alloc<float>(1);
    try {
      CUDA_CHECK(cudaMemsetAsync(buf, 0, kBytes, ctx->stream));
      double best_tbs = 0.0, best_ms = 0.0;
      for (int wps : warps_per_sm) {
        const int ctas = ctx->sm_count * wps / 4;
        const double bytes = (double)ctas * 128 * kSteps * 16;
        for (int w = 0; w < 2; ++w) {
          spmx_dev::l2_rows_probe_kernel<<<ctas, 128, 0, ctx->stream>>>(buf, kBytes / 256, kSteps, w, sink);
          post_launch();
        }
        for (int r = 0; r < repeats; ++r) {
          CUDA_CHECK(cudaEventRecord(ctx->ev0, ctx->stream));
          spmx_dev::l2_rows_probe_kernel<<<ctas, 128, 0, ctx->stream>>>(buf, kBytes / 256, kSteps, 10 + r, sink);
          post_launch();
          CUDA_CHECK(cudaEventRecord(ctx->ev1, ctx->stream));
          CUDA_CHECK(cudaEventSynchronize(ctx->ev1));
          float ms = 0.f;
          CUDA_CHECK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
          const double tbs = bytes / (ms * 1e-3) / 1e12;
          if (tbs > best_tbs) { best_tbs = tbs; best_ms = ms; }
        }
      }
      if (out_tbs) *out_tbs = best_tbs;
      if (out_ms) *out_ms = best_ms;
    } catch (...) {
      cudaFree(buf);
      cudaFree(sink);
      throw;
    }
    CUDA_CHECK(cudaFree(buf));
    CUDA_CHECK(cudaFree(sink));
  });
}

int spmx_ctx_l2_window(spmx_ctx* ctx, const void* base, size_t bytes, float hit_ratio,
                       size_t* out_window_bytes) {
  return guarded([&] {
    check(ctx);
    int max_window = 0, max_persist = 0;
    CUDA_CHECK(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device));
    CUDA_CHECK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device));
    cudaStreamAttrValue v{};
    if (base && bytes) {
      const size_t win = std::min<size_t>(bytes, (size_t)max_window);
      const size_t want = std::min<size_t>(win, (size_t)max_persist);
      if (want != ctx->l2_persist) {  // (changing the set-aside reconfigures the L2: tens of milliseconds)
        CUDA_CHECK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
        ctx->l2_persist = want;
      }
      v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
      v.accessPolicyWindow.num_bytes = win;
      v.accessPolicyWindow.hitRatio = hit_ratio;
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      if (out_window_bytes) *out_window_bytes = win;
    } else {
      v.accessPolicyWindow.num_bytes = 0;
      if (out_window_bytes) *out_window_bytes = 0;
    }
    CUDA_CHECK(cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &v));
    if (!(base && bytes) && ctx->l2_persist != 0) {
      CUDA_CHECK(cudaCtxResetPersistingL2Cache());
      CUDA_CHECK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
      ctx->l2_persist = 0;
    }
  });
}

int spmx_debug_bounds(uint64_t* out16) {
  return guarded([&] {
#if SPMX_DEBUG_BOUNDS
    unsigned long long h[16];
    CUDA_CHECK(cudaDeviceSynchronize());
    CUDA_CHECK(cudaMemcpyFromSymbol(h, spmx_dev::g_bounds_violations, sizeof h));
    for (int i = 0; i < 16; ++i) out16[i] = h[i];
#else
    (void)out16;
    throw LogicErr("spmx_debug_bounds: this library was not built with -DSPMX_DEBUG_BOUNDS=1");
#endif
  });
}

int spmx_jit_available(void) { return spmx_jit::Nvrtc::get().ok() ? 1 : 0; }

int spmx_jit_stats(uint64_t* kernels_compiled, double* seconds) {
  return guarded([&] {
    std::lock_guard<std::mutex> lock(spmx_jit::mu());
    if (kernels_compiled) *kernels_compiled = spmx_jit::stats().compiled;
    if (seconds) *seconds = spmx_jit::stats().seconds;
  });
}

int spmx_checksum_device(spmx_ctx* ctx, const float* d_y, size_t count, uint64_t* out) {
  return guarded([&] {
    check(ctx);
    std::vector<float> h(count);
    CUDA_CHECK(cudaMemcpyAsync(h.data(), d_y, count * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    // FNV-1a-64 over the little-endian f32 bytes, dense.cpp:17-28
    uint64_t hsh = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < count; ++i) {
      uint32_t bits;
      std::memcpy(&bits, &h[i], 4);
      for (int s = 0; s < 32; s += 8) {
        hsh ^= (bits >> s) & 0xffu;
        hsh *= 0x100000001b3ull;
      }
    }
    *out = hsh;
  });
}

}  // extern "C"

#include "spmx_mg.cuh"
