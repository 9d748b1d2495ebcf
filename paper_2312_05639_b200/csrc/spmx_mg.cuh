// spmx_mg.cuh — the multi-GPU driver behind the spmx_mg_* entry points of include/spmx_b200.h.
// Included at the end of spmx_capi.cu (same translation unit: it drives the single-GPU
// machinery above — contexts, the device partitioner, plan_build, run_kernels).
//
// What it generalises: the reference runs ONE fork-join over contiguous row ranges of A, one
// range per worker (executor.cpp:66-99), the ranges coming from make_partition
// (partition.cpp:86-104). Here the workers of the outer level are GPUs: A is cut into row
// blocks ("shards") by the reference's own split_nnz(A, G) (partition.cpp:35-51) or
// split_merge(A, G) (partition.cpp:69-84), evaluated by the device partitioner (bit-exact);
// every shard is a CSR of its own with a rebased row_ptr on one GPU; X is replicated by one
// ncclBroadcast; every GPU runs its shards through its own plans; Y stays row-sharded. Rows have
// a single writer, so no collective sits on the data path. An all-gather-v of Y
// (one ncclBroadcast per shard in one group — shards have unequal row counts, nothing is padded)
// and small all-reduces for the timing statistics are the only other NCCL calls.
//
// NCCL is loaded with dlopen: no link-time dependency, and inside a process that already carries
// a libnccl.so.2 (torch) the same copy is used.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <thread>

namespace {

struct Nccl {
  void* handle = nullptr;
  decltype(&ncclGetVersion) GetVersion = nullptr;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommInitAll) CommInitAll = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  std::string tried;

  static Nccl& get() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
      std::vector<std::string> names;
      if (const char* e = std::getenv("SPMX_NCCL_LIB"))
        if (*e) names.push_back(e);
      names.push_back("libnccl.so.2");
      names.push_back("libnccl.so");
      for (const std::string& nm : names) {
        n.tried += (n.tried.empty() ? "" : ", ") + nm;
        if ((n.handle = dlopen(nm.c_str(), RTLD_NOW | RTLD_LOCAL))) break;
      }
      if (!n.handle) return;
#define SPMX_SYM(f) n.f = reinterpret_cast<decltype(n.f)>(dlsym(n.handle, "nccl" #f))
      SPMX_SYM(GetVersion); SPMX_SYM(GetUniqueId); SPMX_SYM(CommInitRank); SPMX_SYM(CommInitAll);
      SPMX_SYM(CommDestroy); SPMX_SYM(Broadcast); SPMX_SYM(AllReduce); SPMX_SYM(GroupStart);
      SPMX_SYM(GroupEnd); SPMX_SYM(GetErrorString);
#undef SPMX_SYM
    });
    return n;
  }
  bool ok() const {
    return handle && GetVersion && GetUniqueId && CommInitRank && CommInitAll && CommDestroy &&
           Broadcast && AllReduce && GroupStart && GroupEnd;
  }
  static Nccl& require() {
    Nccl& n = get();
    if (!n.ok())
      throw std::runtime_error("NCCL is not available (tried " + n.tried +
                               "): the multi-GPU driver has no other transport");
    return n;
  }
};

#define NCCL_CHECK(expr)                                                                      \
  do {                                                                                        \
    ncclResult_t _r = (expr);                                                                 \
    if (_r != ncclSuccess) {                                                                  \
      Nccl& _n = Nccl::get();                                                                 \
      throw std::runtime_error(std::string("NCCL error: ") +                                  \
                               (_n.GetErrorString ? _n.GetErrorString(_r) : "?") + " at " #expr); \
    }                                                                                         \
  } while (0)

constexpr uint32_t kMagicMg = 0x584d4721;

// row_ptr of a shard: the slice row_ptr[b .. e] of A minus row_ptr[b]
__global__ void rebase_row_ptr_kernel(u64* __restrict__ rp, u64 count, u64 base) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) rp[i] -= base;
}

// ---- hot X rows (L2 residency for matrices whose X is far larger than the L2) ---------------
// On a power-law matrix a few columns carry a large share of the nonzeros (c5: the 50 000
// hottest of 16.8 M columns 43.5 %), yet their X rows are scattered and get evicted by the
// stream of cold rows (L2 hit 28 %, DRAM traffic 4.9 x the algorithmic bytes). When the driver
// owns the X replicas it keeps a COMPACT COPY of each rank's hottest rows behind X (rows
// N .. N + H of the same buffer), points the shards' column indices of those columns at the
// copy (col' = N + slot: the kernels are unchanged, values and order too) and puts a persisting
// L2 access-policy window over it. Measured upper bound (tools/exp_hot_window.py, c5): DRAM reads
// 85.7 -> 75.2 GB, 14.0 -> 12.5 ms.
__global__ void col_degree_kernel(const uint32_t* __restrict__ col, u64 nnz, uint32_t* __restrict__ deg) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) atomicAdd(deg + col[k], 1u);
}
__global__ void count_ge_kernel(const uint32_t* __restrict__ deg, u64 n, uint32_t thr, unsigned long long* out) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  unsigned long long c = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) c += deg[i] >= thr;
  c = __reduce_add_sync(0xffffffffu, (unsigned)c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
// deg[c] becomes the slot of column c (kNotHot when it is not hot); hot_cols[slot] = c
constexpr uint32_t kNotHot = 0xffffffffu;
__global__ void assign_slots_kernel(uint32_t* __restrict__ deg, u64 n, uint32_t thr, uint32_t cap,
                                    uint32_t* __restrict__ hot_cols, uint32_t* __restrict__ counter) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint32_t slot = kNotHot;
    if (deg[i] >= thr) {
      slot = atomicAdd(counter, 1u);
      if (slot < cap) hot_cols[slot] = (uint32_t)i; else slot = kNotHot;
    }
    deg[i] = slot;
  }
}
__global__ void remap_cols_kernel(uint32_t* __restrict__ col, u64 nnz, const uint32_t* __restrict__ slot_of,
                                  uint32_t n) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    const uint32_t s = slot_of[col[k]];
    if (s != kNotHot) col[k] = n + s;
  }
}
__global__ void unmap_cols_kernel(uint32_t* __restrict__ col, u64 nnz, const uint32_t* __restrict__ hot_cols,
                                  uint32_t n) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride)
    if (col[k] >= n) col[k] = hot_cols[col[k] - n];
}
// xext[n + s] = x[hot_cols[s]] for every slot s: d floats per row, one thread per element
__global__ void compact_rows_kernel(float* __restrict__ x, const uint32_t* __restrict__ hot_cols, u64 n_hot,
                                    u64 n, int d) {
  const u64 idx = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_hot * (u64)d) return;
  const u64 s = idx / (u64)d;
  const int j = (int)(idx % (u64)d);
  x[(n + s) * (u64)d + j] = x[(u64)hot_cols[s] * (u64)d + j];
}

struct MgRank {  // one GPU driven by this process
  int rank = 0;  // global rank
  int device = 0;
  spmx_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  float* x = nullptr;  // replicated X (x_rows x d)
  bool x_owned = false;
  size_t x_floats = 0;
  float* y_full = nullptr;  // all-gather target (M x d)
  size_t y_full_floats = 0;
  double* red = nullptr;  // scratch of the statistics all-reduce
  uint32_t* hot_cols = nullptr;  // original column of every hot slot
  uint32_t* slot_of = nullptr;   // slot of every column (kNotHot), kept while the shards can be remapped
  uint32_t n_hot = 0;
  bool remapped = false;         // the rank's shards point their hot columns at rows N .. N + n_hot of X
  bool window = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  float ms = 0.f;
  size_t hot_cap = 0, slot_n = 0;  // element counts of hot_cols / slot_of
  // Device buffers of the shards that were last released, kept for the next sharding: a caller
  // that shards the same matrix again (every end-to-end call does) asks for exactly these sizes,
  // and cudaMalloc / cudaFree of gigabyte buffers cost 50 - 500 ms per call with a large spread.
  std::vector<std::pair<void*, size_t>> spare;
};

struct MgShard {
  int global = 0;      // index among all shards
  int local_rank = 0;  // index into spmx_mg::ranks
  u64 row_begin = 0, row_end = 0, nnz_begin = 0, nnz = 0;
  spmx_csr* csr = nullptr;  // owns the shard's arrays
  spmx_plan* plan = nullptr;
  float* y = nullptr;  // (row_end - row_begin) x d
  size_t y_floats = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

}  // namespace

struct spmx_mg {
  uint32_t magic = kMagicMg;
  int world = 1;
  int n_shards = 1;
  bool has_comm = false;
  int nccl_version = 0;
  std::vector<MgRank> ranks;    // local
  std::vector<MgShard> shards;  // local, ascending global index
  std::vector<u64> ranges;      // 2 * n_shards, all shards
  int64_t m = 0, n = 0, nnz = 0;  // of the whole A
  int64_t d = 0;                  // width of the X currently held
};

namespace {

spmx_mg* check(spmx_mg* g) {
  if (!g || g->magic != kMagicMg) throw LogicErr("invalid or destroyed spmx_mg");
  return g;
}
const spmx_mg* check(const spmx_mg* g) {
  if (!g || g->magic != kMagicMg) throw LogicErr("invalid or destroyed spmx_mg");
  return g;
}

int shard_owner(int n_shards, int world, int shard) {
  return (int)((int64_t)shard * world / n_shards);
}

// runs f(local rank index) for every local rank, one host thread per GPU when there are several
// (the reference's fork-join with GPUs for workers); the first exception is rethrown on the caller
template <typename F>
void for_each_rank(spmx_mg* g, F&& f) {
  const size_t nr = g->ranks.size();
  if (nr == 1) {
    CUDA_CHECK(cudaSetDevice(g->ranks[0].device));
    f(0);
    return;
  }
  std::vector<std::exception_ptr> errs(nr);
  std::vector<std::thread> th;
  th.reserve(nr);
  for (size_t r = 0; r < nr; ++r)
    th.emplace_back([&, r] {
      try {
        CUDA_CHECK(cudaSetDevice(g->ranks[r].device));
        f((int)r);
      } catch (...) {
        errs[r] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// (the rank's device is current)
void mg_drop_spare(MgRank& r) {
  for (auto& e : r.spare) cudaFree(e.first);
  r.spare.clear();
}
template <typename T>
T* mg_take(MgRank& r, size_t count) {
  const size_t bytes = (count ? count : 1) * sizeof(T);
  for (size_t i = 0; i < r.spare.size(); ++i)
    if (r.spare[i].second == bytes) {
      T* p = (T*)r.spare[i].first;
      r.spare.erase(r.spare.begin() + (long)i);
      return p;
    }
  mg_drop_spare(r);  // other sizes: another matrix, the old buffers are of no use
  T* p = nullptr;
  CUDA_CHECK(cudaMalloc(&p, bytes));
  return p;
}
template <typename T>
void mg_give(MgRank& r, T* p, size_t count) {
  if (!p) return;
  if (r.spare.size() >= 64) { cudaFree(p); return; }
  r.spare.emplace_back((void*)p, (count ? count : 1) * sizeof(T));
}

void mg_free_shards(spmx_mg* g) {
  for (MgShard& s : g->shards) {
    MgRank& r = g->ranks[s.local_rank];
    cudaSetDevice(r.device);
    cudaStreamSynchronize(r.ctx->stream);
    if (s.plan) plan_free(s.plan);
    if (s.csr) {  // the arrays belong to the driver (owned = false): kept for the next sharding
      mg_give(r, s.csr->row_ptr, (size_t)s.csr->m + 1);
      mg_give(r, s.csr->col, (size_t)s.csr->nnz);
      mg_give(r, s.csr->vals, (size_t)s.csr->nnz);
      spmx_csr_destroy(s.csr);
    }
    mg_give(r, s.y, s.y_floats);
    if (s.ev0) cudaEventDestroy(s.ev0);
    if (s.ev1) cudaEventDestroy(s.ev1);
  }
  g->shards.clear();
  g->ranges.clear();
  for (MgRank& r : g->ranks) {  // the hot-row tables describe the shards that just went away
    if (!r.ctx) continue;
    cudaSetDevice(r.device);
    mg_give(r, r.hot_cols, r.hot_cap);
    mg_give(r, r.slot_of, r.slot_n);
    r.hot_cols = r.slot_of = nullptr;
    r.hot_cap = r.slot_n = 0;
    r.n_hot = 0;
    r.remapped = false;
  }
}

void mg_free(spmx_mg* g) {
  if (!g) return;
  mg_free_shards(g);
  Nccl& nc = Nccl::get();
  for (MgRank& r : g->ranks) {
    if (!r.ctx) continue;  // creation failed before anything was allocated on this device
    cudaSetDevice(r.device);
    mg_drop_spare(r);
    cudaStreamSynchronize(r.ctx->stream);
    if (r.comm && nc.CommDestroy) nc.CommDestroy(r.comm);
    if (r.x && r.x_owned) cudaFree(r.x);
    if (r.y_full) cudaFree(r.y_full);
    if (r.red) cudaFree(r.red);
    if (r.hot_cols) cudaFree(r.hot_cols);
    if (r.slot_of) cudaFree(r.slot_of);
    if (r.ev0) cudaEventDestroy(r.ev0);
    if (r.ev1) cudaEventDestroy(r.ev1);
    if (r.ctx) spmx_ctx_destroy(r.ctx);
  }
  g->magic = 0;
  delete g;
}

void mg_add_rank(spmx_mg* g, int rank, int device, void* stream) {
  g->ranks.emplace_back();  // mg_free releases whatever has been created so far
  MgRank& r = g->ranks.back();
  r.rank = rank;
  r.device = device;
  const int rc = spmx_ctx_create(device, stream, &r.ctx);
  if (rc == SPMX_EINVAL) throw InvalidArg(g_last_error);
  if (rc != SPMX_OK) throw std::runtime_error(g_last_error);
  CUDA_CHECK(cudaSetDevice(device));
  CUDA_CHECK(cudaEventCreate(&r.ev0));
  CUDA_CHECK(cudaEventCreate(&r.ev1));
  r.red = dev_alloc<double>(16);
}

void mg_set_shards(spmx_mg* g, int n_shards) {
  if (n_shards < 0) throw InvalidArg("spmx_mg: negative shard count");
  g->n_shards = n_shards == 0 ? g->world : n_shards;
  if (g->n_shards < g->world)
    throw InvalidArg("spmx_mg: fewer shards than ranks (every GPU owns at least one row block)");
}

// Builds the local shards from the boundaries in g->ranges. `fetch(dst_dev_ptr, what, first,
// count, rank)` copies count elements starting at `first` of A's row_ptr (what = 0), col (1) or
// vals (2) into device memory of local rank `rank`, on that rank's stream. nnz_at(r) = row_ptr[r].
template <typename Fetch, typename NnzAt>
void mg_place(spmx_mg* g, Fetch&& fetch, NnzAt&& nnz_at) {
  for (int sh = 0; sh < g->n_shards; ++sh) {
    const int owner = shard_owner(g->n_shards, g->world, sh);
    int lr = -1;
    for (size_t i = 0; i < g->ranks.size(); ++i)
      if (g->ranks[i].rank == owner) lr = (int)i;
    if (lr < 0) continue;  // another process owns it
    MgRank& r = g->ranks[lr];
    CUDA_CHECK(cudaSetDevice(r.device));
    MgShard s;
    s.global = sh;
    s.local_rank = lr;
    s.row_begin = g->ranges[2 * sh];
    s.row_end = g->ranges[2 * sh + 1];
    s.nnz_begin = nnz_at(s.row_begin);
    s.nnz = nnz_at(s.row_end) - s.nnz_begin;
    const u64 rows = s.row_end - s.row_begin;
    spmx_csr* a = new spmx_csr;
    a->ctx = r.ctx;
    a->m = (int64_t)rows;
    a->n = g->n;
    a->nnz = (int64_t)s.nnz;
    a->owned = false;  // the arrays go back to the rank's spare list (mg_free_shards)
    s.csr = a;
    g->shards.push_back(s);  // from here on mg_free_shards releases it
    MgShard& t = g->shards.back();
    a->row_ptr = mg_take<u64>(r, (size_t)rows + 1);
    a->col = mg_take<uint32_t>(r, (size_t)s.nnz);
    a->vals = mg_take<float>(r, (size_t)s.nnz);
    CUDA_CHECK(cudaEventCreate(&t.ev0));
    CUDA_CHECK(cudaEventCreate(&t.ev1));
    fetch((void*)a->row_ptr, 0, s.row_begin, rows + 1, lr);
    if (s.nnz) {
      fetch((void*)a->col, 1, s.nnz_begin, s.nnz, lr);
      fetch((void*)a->vals, 2, s.nnz_begin, s.nnz, lr);
    }
    rebase_row_ptr_kernel<<<validate_grid(r.ctx, rows + 1), 256, 0, r.ctx->stream>>>(
        a->row_ptr, rows + 1, s.nnz_begin);
    post_launch();
  }
  // the invariants of validate_csr (csr.cpp:18-42) per shard, on the shard's own GPU
  for (MgShard& s : g->shards) {
    MgRank& r = g->ranks[s.local_rank];
    CUDA_CHECK(cudaSetDevice(r.device));
    validate_on_device(r.ctx, s.csr);
  }
}

// split_nnz / split_merge of the WHOLE matrix into n_shards ranges, on `ctx`'s device
void mg_split(spmx_mg* g, spmx_ctx* ctx, const u64* d_row_ptr, int shard_by) {
  spmx_csr tmp;
  tmp.ctx = ctx;
  tmp.m = g->m;
  tmp.n = g->n;
  tmp.nnz = g->nnz;
  tmp.row_ptr = (u64*)d_row_ptr;
  tmp.structure_only = true;
  CUDA_CHECK(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
  spmx_dev::validate_row_ptr_kernel<<<validate_grid(ctx, (u64)g->m), 256, 0, ctx->stream>>>(
      d_row_ptr, (u64)g->m, (u64)g->nnz, ctx->d_err);
  post_launch();
  int err = 0;
  CUDA_CHECK(cudaMemcpyAsync(&err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  if (err) throw InvalidArg(std::string("invalid CSR: ") + csr_error_text(err));
  AsyncScratch scratch(ctx);
  u64* d_bnd = scratch.get<u64>((size_t)g->n_shards + 1);
  const int strategy = shard_by == SPMX_SHARD_BY_MERGE ? SPMX_MERGE_SPLIT : SPMX_NNZ_SPLIT;
  strategy_row_boundaries(ctx, &tmp, strategy, (unsigned)g->n_shards, d_bnd);
  g->ranges.assign(2 * (size_t)g->n_shards, 0);
  ranges_to_host(ctx, d_bnd, (unsigned)g->n_shards, (uint64_t*)g->ranges.data());
}

void mg_check_shape(int64_t m, int64_t n, int64_t nnz, int shard_by) {
  if (m < 0 || n < 0 || nnz < 0) throw InvalidArg("invalid CSR: negative dimension");
  if (shard_by != SPMX_SHARD_BY_NNZ && shard_by != SPMX_SHARD_BY_MERGE)
    throw InvalidArg("spmx_mg_shard: shard_by must be SPMX_SHARD_BY_NNZ or SPMX_SHARD_BY_MERGE");
}

// knobs of the hot-row copy: rows kept per rank (0 disables), and how large X has to be before
// the persisting L2 window is worth its set-aside (it costs the rest of the L2 what it gives)
inline u64 mg_hot_rows() { return env_u64("SPMX_MG_HOT_ROWS", 50000); }
inline u64 mg_hot_min_x_mb() { return env_u64("SPMX_MG_HOT_MIN_MB", 1024); }

void mg_ensure_x(spmx_mg* g, int64_t x_rows, int64_t d) {
  // (room for the compact copy of the hot rows behind X, whatever the current shards need)
  const size_t need = ((size_t)x_rows + (size_t)mg_hot_rows()) * (size_t)d;
  for (MgRank& r : g->ranks) {
    CUDA_CHECK(cudaSetDevice(r.device));
    if (!r.x_owned) { r.x = nullptr; r.x_floats = 0; }
    if (r.x_floats < need) {
      if (r.x) CUDA_CHECK(cudaFree(r.x));
      r.x = nullptr;
      r.x = dev_alloc<float>(need);
      r.x_floats = need;
    }
    r.x_owned = true;
  }
}

// Per rank: the H columns with the most nonzeros in the rank's shards (degree histogram, then
// the smallest threshold that admits at most H columns), their slots, and the list of hot columns.
void mg_build_hot(spmx_mg* g) {
  const u64 cap = mg_hot_rows();
  if (cap == 0 || (u64)g->n < 8 * cap || g->n >= (int64_t)0x7fffffff - (int64_t)cap) return;
  for (size_t lr = 0; lr < g->ranks.size(); ++lr) {
    MgRank& r = g->ranks[lr];
    u64 nnz = 0;
    for (const MgShard& s : g->shards)
      if (s.local_rank == (int)lr) nnz += s.nnz;
    if (nnz == 0) continue;
    CUDA_CHECK(cudaSetDevice(r.device));
    cudaStream_t st = r.ctx->stream;
    const u64 n = (u64)g->n;
    r.slot_of = mg_take<uint32_t>(r, (size_t)n);
    r.slot_n = (size_t)n;
    r.hot_cols = mg_take<uint32_t>(r, (size_t)cap);
    r.hot_cap = (size_t)cap;
    CUDA_CHECK(cudaMemsetAsync(r.slot_of, 0, (size_t)n * 4, st));
    for (const MgShard& s : g->shards)
      if (s.local_rank == (int)lr && s.nnz) {
        col_degree_kernel<<<validate_grid(r.ctx, s.nnz), 256, 0, st>>>(s.csr->col, s.nnz, r.slot_of);
        post_launch();
      }
    unsigned long long* d_cnt = dev_alloc<unsigned long long>(1);
    uint32_t* d_n = dev_alloc<uint32_t>(1);
    try {
      auto count_ge = [&](uint32_t thr) {
        unsigned long long c = 0;
        CUDA_CHECK(cudaMemsetAsync(d_cnt, 0, 8, st));
        count_ge_kernel<<<validate_grid(r.ctx, n), 256, 0, st>>>(r.slot_of, n, thr, d_cnt);
        post_launch();
        CUDA_CHECK(cudaMemcpyAsync(&c, d_cnt, 8, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        return (u64)c;
      };
      uint32_t lo = 1, hi = 0x80000000u;  // smallest thr in [lo, hi] with count(deg >= thr) <= cap
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (count_ge(mid) <= cap) hi = mid; else lo = mid + 1;
      }
      CUDA_CHECK(cudaMemsetAsync(d_n, 0, 4, st));
      assign_slots_kernel<<<validate_grid(r.ctx, n), 256, 0, st>>>(r.slot_of, n, lo, (uint32_t)cap, r.hot_cols, d_n);
      post_launch();
      CUDA_CHECK(cudaMemcpyAsync(&r.n_hot, d_n, 4, cudaMemcpyDeviceToHost, st));
      CUDA_CHECK(cudaStreamSynchronize(st));
      r.n_hot = std::min<uint32_t>(r.n_hot, (uint32_t)cap);
    } catch (...) {
      cudaFree(d_cnt);
      cudaFree(d_n);
      throw;
    }
    CUDA_CHECK(cudaFree(d_cnt));
    CUDA_CHECK(cudaFree(d_n));
  }
}

// Points the hot columns of every local shard at the compact copy (on) or back at X (off).
void mg_set_remap(spmx_mg* g, bool on) {
  for (size_t lr = 0; lr < g->ranks.size(); ++lr) {
    MgRank& r = g->ranks[lr];
    if (r.n_hot == 0 || r.remapped == on) continue;
    CUDA_CHECK(cudaSetDevice(r.device));
    for (MgShard& s : g->shards) {
      if (s.local_rank != (int)lr || s.nnz == 0) continue;
      if (on)
        remap_cols_kernel<<<validate_grid(r.ctx, s.nnz), 256, 0, r.ctx->stream>>>(s.csr->col, s.nnz, r.slot_of,
                                                                                  (uint32_t)g->n);
      else
        unmap_cols_kernel<<<validate_grid(r.ctx, s.nnz), 256, 0, r.ctx->stream>>>(s.csr->col, s.nnz, r.hot_cols,
                                                                                  (uint32_t)g->n);
      post_launch();
    }
    r.remapped = on;
  }
}

void mg_clear_window(MgRank& r) {
  if (!r.window) return;
  CUDA_CHECK(cudaSetDevice(r.device));
  if (spmx_ctx_l2_window(r.ctx, nullptr, 0, 0.f, nullptr) != SPMX_OK) throw std::runtime_error(g_last_error);
  r.window = false;
}

// The driver owns X (x_rows x d at the front of every rank's buffer, just broadcast): refresh the
// compact copy of the hot rows behind it, point the shards at it, and protect it in L2 when X is
// large enough for that to pay.
void mg_refresh_hot(spmx_mg* g, int64_t x_rows, int64_t d) {
  mg_set_remap(g, true);
  const bool big = (u64)x_rows * (u64)d * 4 >= (mg_hot_min_x_mb() << 20);
  for (MgRank& r : g->ranks) {
    if (r.n_hot == 0) { mg_clear_window(r); continue; }
    CUDA_CHECK(cudaSetDevice(r.device));
    const u64 elems = (u64)r.n_hot * (u64)d;
    compact_rows_kernel<<<blocks_for(elems), 256, 0, r.ctx->stream>>>(r.x, r.hot_cols, r.n_hot, (u64)x_rows, (int)d);
    post_launch();
    if (big) {
      if (spmx_ctx_l2_window(r.ctx, r.x + (size_t)x_rows * (size_t)d, (size_t)elems * 4, 1.0f, nullptr) != SPMX_OK)
        throw std::runtime_error(g_last_error);
      r.window = true;
    } else {
      mg_clear_window(r);
    }
  }
}

// one ncclBroadcast of X from root_rank on every local rank's stream, timed per rank
void mg_broadcast(spmx_mg* g, int root_rank, size_t count, float* bcast_ms) {
  const float* root_buf = nullptr;
  for (MgRank& r : g->ranks)
    if (r.rank == root_rank) root_buf = r.x;
  for (MgRank& r : g->ranks) {
    CUDA_CHECK(cudaSetDevice(r.device));
    CUDA_CHECK(cudaEventRecord(r.ev0, r.ctx->stream));
  }
  if (g->has_comm) {
    Nccl& nc = Nccl::require();
    NCCL_CHECK(nc.GroupStart());
    for (MgRank& r : g->ranks) {
      // the send buffer is read on the root only; elsewhere NCCL ignores it
      const float* send = r.rank == root_rank ? r.x : (root_buf ? root_buf : r.x);
      NCCL_CHECK(nc.Broadcast(send, r.x, count, ncclFloat, root_rank, r.comm, r.ctx->stream));
    }
    NCCL_CHECK(nc.GroupEnd());
  } else if (g->world > 1) {
    throw std::runtime_error("spmx_mg_broadcast_x: this driver was built without a communicator");
  }
  float worst = 0.f;
  for (MgRank& r : g->ranks) {
    CUDA_CHECK(cudaSetDevice(r.device));
    CUDA_CHECK(cudaEventRecord(r.ev1, r.ctx->stream));
    CUDA_CHECK(cudaEventSynchronize(r.ev1));
    float t = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&t, r.ev0, r.ev1));
    worst = std::max(worst, t);
  }
  if (bcast_ms) *bcast_ms = worst;
}

void mg_require_x_shape(const spmx_mg* g, int root_rank, int64_t x_rows, int64_t d) {
  if (root_rank < 0 || root_rank >= g->world) throw InvalidArg("spmx_mg_broadcast_x: no such rank");
  if (d < 1) throw InvalidArg("run_spmm: X.cols must be >= 1");
  if (!g->ranges.empty() && x_rows != g->n) throw InvalidArg("run_spmm: A.n != X.rows");
}

}  // namespace

extern "C" {

int spmx_mg_shard_owner(int n_shards, int world, int shard) {
  if (n_shards < 1 || world < 1 || shard < 0 || shard >= n_shards) return -1;
  return shard_owner(n_shards, world, shard);
}

int spmx_mg_create(int n_devices, const int* devices, int n_shards, spmx_mg** out) {
  return guarded([&] {
    if (!out) throw InvalidArg("spmx_mg_create: null out");
    if (n_devices < 1 || !devices) throw InvalidArg("spmx_mg_create: no devices");
    for (int i = 0; i < n_devices; ++i)
      for (int j = 0; j < i; ++j)
        if (devices[i] == devices[j])
          throw InvalidArg("spmx_mg_create: a device is listed twice (several row blocks on one "
                           "GPU are n_shards > n_devices)");
    Nccl& nc = Nccl::require();
    spmx_mg* g = new spmx_mg;
    try {
      g->world = n_devices;
      mg_set_shards(g, n_shards);
      for (int i = 0; i < n_devices; ++i) mg_add_rank(g, i, devices[i], nullptr);
      std::vector<ncclComm_t> comms((size_t)n_devices, nullptr);
      NCCL_CHECK(nc.CommInitAll(comms.data(), n_devices, devices));
      for (int i = 0; i < n_devices; ++i) g->ranks[(size_t)i].comm = comms[(size_t)i];
      g->has_comm = true;
      NCCL_CHECK(nc.GetVersion(&g->nccl_version));
      // peer copies of shard_device go directly over NVLink where the topology allows it
      for (int i = 0; i < n_devices; ++i) {
        CUDA_CHECK(cudaSetDevice(devices[i]));
        for (int j = 0; j < n_devices; ++j) {
          int can = 0;
          if (i != j && cudaDeviceCanAccessPeer(&can, devices[i], devices[j]) == cudaSuccess && can)
            if (cudaDeviceEnablePeerAccess(devices[j], 0) != cudaSuccess) cudaGetLastError();
        }
      }
    } catch (...) {
      mg_free(g);
      throw;
    }
    *out = g;
  });
}

int spmx_mg_unique_id(void* out128) {
  return guarded([&] {
    if (!out128) throw InvalidArg("spmx_mg_unique_id: null out");
    static_assert(sizeof(ncclUniqueId) == 128, "the ABI hands the NCCL id over as 128 bytes");
    ncclUniqueId id;
    NCCL_CHECK(Nccl::require().GetUniqueId(&id));
    std::memcpy(out128, &id, sizeof id);
  });
}

int spmx_mg_create_rank(int device, void* stream, int rank, int world, int n_shards,
                        const void* id128, spmx_mg** out) {
  return guarded([&] {
    if (!out) throw InvalidArg("spmx_mg_create_rank: null out");
    if (world < 1 || rank < 0 || rank >= world) throw InvalidArg("spmx_mg_create_rank: bad rank/world");
    spmx_mg* g = new spmx_mg;
    try {
      g->world = world;
      mg_set_shards(g, n_shards);
      mg_add_rank(g, rank, device, stream);
      if (id128) {
        Nccl& nc = Nccl::require();
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof id);
        CUDA_CHECK(cudaSetDevice(device));
        NCCL_CHECK(nc.CommInitRank(&g->ranks[0].comm, world, id, rank));
        g->has_comm = true;
        NCCL_CHECK(nc.GetVersion(&g->nccl_version));
      }
    } catch (...) {
      mg_free(g);
      throw;
    }
    *out = g;
  });
}

int spmx_mg_destroy(spmx_mg* mg) {
  return guarded([&] {
    check(mg);
    mg_free(mg);
  });
}

int spmx_mg_info(const spmx_mg* mg, int* world, int* n_local_ranks, int* n_shards,
                 int* n_local_shards, int* nccl_version) {
  return guarded([&] {
    check(mg);
    if (world) *world = mg->world;
    if (n_local_ranks) *n_local_ranks = (int)mg->ranks.size();
    if (n_shards) *n_shards = mg->n_shards;
    if (n_local_shards) *n_local_shards = (int)mg->shards.size();
    if (nccl_version) *nccl_version = mg->has_comm ? mg->nccl_version : 0;
  });
}

int spmx_mg_shard_host(spmx_mg* mg, int64_t m, int64_t n, int64_t nnz, const uint64_t* row_ptr,
                       const uint32_t* col, const float* vals, int shard_by, uint64_t* out_ranges) {
  return guarded([&] {
    check(mg);
    mg_check_shape(m, n, nnz, shard_by);
    if (!row_ptr || (nnz > 0 && (!col || !vals))) throw InvalidArg("invalid CSR: null array");
    mg_free_shards(mg);
    mg->m = m; mg->n = n; mg->nnz = nnz;
    try {
      MgRank& r0 = mg->ranks[0];
      CUDA_CHECK(cudaSetDevice(r0.device));
      u64* d_rp = dev_alloc<u64>((size_t)m + 1);
      try {
        copy_h2d(r0.ctx, d_rp, row_ptr, ((size_t)m + 1) * 8, r0.ctx->stream);
        mg_split(mg, r0.ctx, d_rp, shard_by);
      } catch (...) {
        cudaFree(d_rp);
        throw;
      }
      CUDA_CHECK(cudaFree(d_rp));
      auto fetch = [&](void* dst, int what, u64 first, u64 count, int lr) {
        const MgRank& r = mg->ranks[(size_t)lr];
        const void* src = what == 0 ? (const void*)(row_ptr + first)
                        : what == 1 ? (const void*)(col + first) : (const void*)(vals + first);
        copy_h2d(r.ctx, dst, src, count * (what == 0 ? 8 : 4), r.ctx->stream);  // pageable arrays: staged by host threads
      };
      // the split has validated row_ptr, so these reads stay inside [0, nnz]
      mg_place(mg, fetch, [&](u64 r) { return (u64)row_ptr[r]; });
      mg_build_hot(mg);
      if (mg->d > 0 && mg->ranks[0].x_owned) mg_refresh_hot(mg, n, mg->d);  // X stays across a re-shard
    } catch (...) {
      mg_free_shards(mg);
      throw;
    }
    if (out_ranges) std::memcpy(out_ranges, mg->ranges.data(), mg->ranges.size() * 8);
  });
}

int spmx_mg_shard_device(spmx_mg* mg, int src_local_rank, int64_t m, int64_t n, int64_t nnz,
                         const uint64_t* d_row_ptr, const uint32_t* d_col, const float* d_vals,
                         int shard_by, uint64_t* out_ranges) {
  return guarded([&] {
    check(mg);
    mg_check_shape(m, n, nnz, shard_by);
    if (src_local_rank < 0 || src_local_rank >= (int)mg->ranks.size())
      throw InvalidArg("spmx_mg_shard_device: no such local rank");
    if (!d_row_ptr || (nnz > 0 && (!d_col || !d_vals))) throw InvalidArg("invalid CSR: null array");
    mg_free_shards(mg);
    mg->m = m; mg->n = n; mg->nnz = nnz;
    try {
      MgRank& src = mg->ranks[(size_t)src_local_rank];
      CUDA_CHECK(cudaSetDevice(src.device));
      mg_split(mg, src.ctx, (const u64*)d_row_ptr, shard_by);
      // row_ptr at the shard boundaries, read back once
      std::vector<u64> at((size_t)mg->n_shards + 1, 0);
      for (int sh = 0; sh <= mg->n_shards; ++sh) {
        const u64 row = sh < mg->n_shards ? mg->ranges[2 * (size_t)sh] : (u64)m;
        CUDA_CHECK(cudaMemcpyAsync(&at[(size_t)sh], d_row_ptr + row, 8, cudaMemcpyDeviceToHost,
                                   src.ctx->stream));
      }
      CUDA_CHECK(cudaStreamSynchronize(src.ctx->stream));
      auto nnz_at = [&](u64 row) {
        for (int sh = 0; sh < mg->n_shards; ++sh)
          if (mg->ranges[2 * (size_t)sh] == row) return at[(size_t)sh];
        return at[(size_t)mg->n_shards];  // row == m (ranges are contiguous and end at m)
      };
      auto fetch = [&](void* dst, int what, u64 first, u64 count, int lr) {
        const MgRank& r = mg->ranks[(size_t)lr];
        const void* from = what == 0 ? (const void*)(d_row_ptr + first)
                         : what == 1 ? (const void*)(d_col + first) : (const void*)(d_vals + first);
        const size_t bytes = count * (what == 0 ? 8 : 4);
        if (r.device == src.device)
          CUDA_CHECK(cudaMemcpyAsync(dst, from, bytes, cudaMemcpyDeviceToDevice, r.ctx->stream));
        else
          CUDA_CHECK(cudaMemcpyPeerAsync(dst, r.device, from, src.device, bytes, r.ctx->stream));
      };
      mg_place(mg, fetch, nnz_at);
      mg_build_hot(mg);
      if (mg->d > 0 && mg->ranks[0].x_owned) mg_refresh_hot(mg, n, mg->d);  // X stays across a re-shard
    } catch (...) {
      mg_free_shards(mg);
      throw;
    }
    if (out_ranges) std::memcpy(out_ranges, mg->ranges.data(), mg->ranges.size() * 8);
  });
}

int spmx_mg_shard_info(const spmx_mg* mg, int local_shard, int* global_shard, int* device,
                       uint64_t* row_begin, uint64_t* row_end, uint64_t* nnz) {
  return guarded([&] {
    check(mg);
    if (local_shard < 0 || local_shard >= (int)mg->shards.size())
      throw InvalidArg("spmx_mg_shard_info: no such local shard");
    const MgShard& s = mg->shards[(size_t)local_shard];
    if (global_shard) *global_shard = s.global;
    if (device) *device = mg->ranks[(size_t)s.local_rank].device;
    if (row_begin) *row_begin = s.row_begin;
    if (row_end) *row_end = s.row_end;
    if (nnz) *nnz = s.nnz;
  });
}

int spmx_mg_plan(spmx_mg* mg, int strategy, unsigned parts, int dynamic, uint64_t batch,
                 unsigned flags) {
  return guarded([&] {
    check(mg);
    if (mg->ranges.empty()) throw LogicErr("spmx_mg_plan: no matrix has been sharded yet");
    for_each_rank(mg, [&](int lr) {
      for (MgShard& s : mg->shards) {
        if (s.local_rank != lr) continue;
        if (s.plan) plan_free(s.plan);
        s.plan = nullptr;
        s.plan = plan_build(mg->ranks[(size_t)lr].ctx, s.csr, strategy, parts, dynamic, batch, flags);
      }
    });
  });
}

int spmx_mg_broadcast_x_host(spmx_mg* mg, const float* x_host, int root_rank, int64_t x_rows,
                             int64_t d, float* h2d_ms, float* bcast_ms) {
  return guarded([&] {
    check(mg);
    mg_require_x_shape(mg, root_rank, x_rows, d);
    mg_ensure_x(mg, x_rows, d);
    if (h2d_ms) *h2d_ms = 0.f;
    for (MgRank& r : mg->ranks) {
      if (r.rank != root_rank) continue;
      if (!x_host && x_rows > 0) throw InvalidArg("run_spmm: null X on the root rank");
      CUDA_CHECK(cudaSetDevice(r.device));
      CUDA_CHECK(cudaEventRecord(r.ev0, r.ctx->stream));
      copy_h2d(r.ctx, r.x, x_host, (size_t)x_rows * (size_t)d * 4, r.ctx->stream);
      CUDA_CHECK(cudaEventRecord(r.ev1, r.ctx->stream));
      CUDA_CHECK(cudaEventSynchronize(r.ev1));
      if (h2d_ms) CUDA_CHECK(cudaEventElapsedTime(h2d_ms, r.ev0, r.ev1));
    }
    mg_broadcast(mg, root_rank, (size_t)x_rows * (size_t)d, bcast_ms);
    mg->d = d;
    mg_refresh_hot(mg, x_rows, d);
  });
}

int spmx_mg_broadcast_x_from_device(spmx_mg* mg, const float* d_x_root, int root_rank, int64_t x_rows,
                                    int64_t d, float* copy_ms, float* bcast_ms) {
  return guarded([&] {
    check(mg);
    mg_require_x_shape(mg, root_rank, x_rows, d);
    mg_ensure_x(mg, x_rows, d);
    if (copy_ms) *copy_ms = 0.f;
    for (MgRank& r : mg->ranks) {
      if (r.rank != root_rank) continue;
      if (!d_x_root && x_rows > 0) throw InvalidArg("run_spmm: null X on the root rank");
      CUDA_CHECK(cudaSetDevice(r.device));
      CUDA_CHECK(cudaEventRecord(r.ev0, r.ctx->stream));
      CUDA_CHECK(cudaMemcpyAsync(r.x, d_x_root, (size_t)x_rows * (size_t)d * 4, cudaMemcpyDeviceToDevice,
                                 r.ctx->stream));
      CUDA_CHECK(cudaEventRecord(r.ev1, r.ctx->stream));
      CUDA_CHECK(cudaEventSynchronize(r.ev1));
      if (copy_ms) CUDA_CHECK(cudaEventElapsedTime(copy_ms, r.ev0, r.ev1));
    }
    mg_broadcast(mg, root_rank, (size_t)x_rows * (size_t)d, bcast_ms);
    mg->d = d;
    mg_refresh_hot(mg, x_rows, d);
  });
}

int spmx_mg_broadcast_x_device(spmx_mg* mg, float* const* d_x_local, int root_rank, int64_t x_rows,
                               int64_t d, float* bcast_ms) {
  return guarded([&] {
    check(mg);
    mg_require_x_shape(mg, root_rank, x_rows, d);
    if (!d_x_local) throw InvalidArg("spmx_mg_broadcast_x_device: null buffer list");
    mg_set_remap(mg, false);  // borrowed buffers have no room for the compact copy of the hot rows
    for (MgRank& r : mg->ranks) mg_clear_window(r);
    for (size_t i = 0; i < mg->ranks.size(); ++i) {
      MgRank& r = mg->ranks[i];
      if (!d_x_local[i] && x_rows > 0) throw InvalidArg("run_spmm: null X");
      if (r.x && r.x_owned) {
        CUDA_CHECK(cudaSetDevice(r.device));
        CUDA_CHECK(cudaFree(r.x));
      }
      r.x = d_x_local[i];
      r.x_owned = false;
      r.x_floats = (size_t)x_rows * (size_t)d;
    }
    mg_broadcast(mg, root_rank, (size_t)x_rows * (size_t)d, bcast_ms);
    mg->d = d;
  });
}

int spmx_mg_spmm(spmx_mg* mg, int steps, float* step_ms, float* ms_per_local_shard) {
  return guarded([&] {
    check(mg);
    if (steps < 1) throw InvalidArg("spmx_mg_spmm: steps must be >= 1");
    if (mg->ranges.empty()) throw LogicErr("spmx_mg_spmm: no matrix has been sharded yet");
    if (mg->d < 1) throw LogicErr("spmx_mg_spmm: X has not been broadcast yet");
    const int64_t d = mg->d;
    for (MgShard& s : mg->shards) {
      if (!s.plan) throw LogicErr("spmx_mg_spmm: spmx_mg_plan has not been called");
      const size_t need = (size_t)(s.row_end - s.row_begin) * (size_t)d;
      if (s.y_floats < need) {
        MgRank& ry = mg->ranks[(size_t)s.local_rank];
        CUDA_CHECK(cudaSetDevice(ry.device));
        if (s.y) CUDA_CHECK(cudaFree(s.y));
        s.y = nullptr;
        s.y_floats = 0;
        s.y = mg_take<float>(ry, need);
        s.y_floats = need;
      }
    }
    // the parallel region (executor.cpp:70-97): every GPU walks its own shards, nobody waits for
    // anybody; a rank's time is what its own stream measures
    for_each_rank(mg, [&](int lr) {
      MgRank& r = mg->ranks[(size_t)lr];
      cudaStream_t st = r.ctx->stream;
      CUDA_CHECK(cudaEventRecord(r.ev0, st));
      for (int step = 0; step < steps; ++step)
        for (MgShard& s : mg->shards) {
          if (s.local_rank != lr) continue;
          const bool mark = step + 1 == steps;
          if (mark) CUDA_CHECK(cudaEventRecord(s.ev0, st));
          s.plan->x_extra_rows = r.remapped ? r.n_hot : 0;
          run_kernels(r.ctx, s.plan, s.csr, r.x, d, s.y, st, 0, s.plan->n_chunks, nullptr);
          if (mark) CUDA_CHECK(cudaEventRecord(s.ev1, st));
        }
      CUDA_CHECK(cudaEventRecord(r.ev1, st));
      CUDA_CHECK(cudaEventSynchronize(r.ev1));
      CUDA_CHECK(cudaEventElapsedTime(&r.ms, r.ev0, r.ev1));
    });
    float worst = 0.f;
    for (const MgRank& r : mg->ranks) worst = std::max(worst, r.ms);
    if (step_ms) *step_ms = worst / (float)steps;
    if (ms_per_local_shard)
      for (size_t i = 0; i < mg->shards.size(); ++i) {
        CUDA_CHECK(cudaSetDevice(mg->ranks[(size_t)mg->shards[i].local_rank].device));
        CUDA_CHECK(cudaEventElapsedTime(&ms_per_local_shard[i], mg->shards[i].ev0, mg->shards[i].ev1));
      }
  });
}

int spmx_mg_y_shard(const spmx_mg* mg, int local_shard, float** d_y) {
  return guarded([&] {
    check(mg);
    if (local_shard < 0 || local_shard >= (int)mg->shards.size() || !d_y)
      throw InvalidArg("spmx_mg_y_shard: no such local shard");
    *d_y = mg->shards[(size_t)local_shard].y;
  });
}

int spmx_mg_download_y(spmx_mg* mg, float* y_host) {
  return guarded([&] {
    check(mg);
    if (!y_host && mg->m > 0) throw InvalidArg("spmx_mg_download_y: null Y");
    const size_t d = (size_t)mg->d;
    std::vector<spmx_stage::Stager::Ticket> tickets;
    for (MgShard& s : mg->shards)  // checked before the first copy: staged copies run on worker threads
      if (!s.y) throw LogicErr("spmx_mg_download_y: spmx_mg_spmm has not run");
    for (MgShard& s : mg->shards) {
      MgRank& r = mg->ranks[(size_t)s.local_rank];
      CUDA_CHECK(cudaSetDevice(r.device));
      const size_t rows = (size_t)(s.row_end - s.row_begin);
      if (!rows) continue;
      float* dst = y_host + (size_t)s.row_begin * d;
      if (stage_this(dst, rows * d * 4))  // pageable Y: the shards of all GPUs are staged side by side
        tickets.push_back(stager_down(r.ctx).d2h(dst, s.y, rows * d * 4, r.ctx->stream));
      else
        CUDA_CHECK(cudaMemcpyAsync(dst, s.y, rows * d * 4, cudaMemcpyDeviceToHost, r.ctx->stream));
    }
    for (auto& t : tickets) spmx_stage::Stager::wait_quiet(t);
    for (MgRank& r : mg->ranks) {
      CUDA_CHECK(cudaSetDevice(r.device));
      CUDA_CHECK(cudaStreamSynchronize(r.ctx->stream));
    }
    for (auto& t : tickets) spmx_stage::Stager::wait(t);  // rethrows a worker's error
  });
}

int spmx_mg_download_y_shards(spmx_mg* mg, float* const* host_per_local_shard) {
  return guarded([&] {
    check(mg);
    if (!host_per_local_shard && !mg->shards.empty()) throw InvalidArg("spmx_mg_download_y_shards: null list");
    const size_t d = (size_t)mg->d;
    std::vector<spmx_stage::Stager::Ticket> tickets;
    for (size_t i = 0; i < mg->shards.size(); ++i) {  // checked before the first copy
      if (!mg->shards[i].y) throw LogicErr("spmx_mg_download_y_shards: spmx_mg_spmm has not run");
      if (mg->shards[i].row_end > mg->shards[i].row_begin && !host_per_local_shard[i])
        throw InvalidArg("spmx_mg_download_y_shards: null Y block");
    }
    for (size_t i = 0; i < mg->shards.size(); ++i) {
      MgShard& s = mg->shards[i];
      MgRank& r = mg->ranks[(size_t)s.local_rank];
      const size_t rows = (size_t)(s.row_end - s.row_begin);
      if (!rows) continue;
      CUDA_CHECK(cudaSetDevice(r.device));
      if (stage_this(host_per_local_shard[i], rows * d * 4))
        tickets.push_back(stager_down(r.ctx).d2h(host_per_local_shard[i], s.y, rows * d * 4, r.ctx->stream));
      else
        CUDA_CHECK(cudaMemcpyAsync(host_per_local_shard[i], s.y, rows * d * 4, cudaMemcpyDeviceToHost,
                                   r.ctx->stream));
    }
    for (auto& t : tickets) spmx_stage::Stager::wait_quiet(t);
    for (MgRank& r : mg->ranks) {
      CUDA_CHECK(cudaSetDevice(r.device));
      CUDA_CHECK(cudaStreamSynchronize(r.ctx->stream));
    }
    for (auto& t : tickets) spmx_stage::Stager::wait(t);
  });
}

int spmx_mg_allgather_y(spmx_mg* mg, float* elapsed_ms) {
  return guarded([&] {
    check(mg);
    if (mg->ranges.empty() || mg->d < 1) throw LogicErr("spmx_mg_allgather_y: nothing to gather yet");
    if (!mg->has_comm) throw std::runtime_error("spmx_mg_allgather_y: this driver was built without a communicator");
    Nccl& nc = Nccl::require();
    const size_t d = (size_t)mg->d, need = (size_t)mg->m * d;
    for (MgRank& r : mg->ranks) {
      CUDA_CHECK(cudaSetDevice(r.device));
      if (r.y_full_floats < need) {
        if (r.y_full) CUDA_CHECK(cudaFree(r.y_full));
        r.y_full = nullptr;
        r.y_full = dev_alloc<float>(need);
        r.y_full_floats = need;
      }
      CUDA_CHECK(cudaEventRecord(r.ev0, r.ctx->stream));
    }
    for (const MgShard& s : mg->shards)
      if (!s.y) throw LogicErr("spmx_mg_allgather_y: spmx_mg_spmm has not run");
    // all-gather-v: shard g's rows go from their owner to everybody's rows [b_g, e_g)
    NCCL_CHECK(nc.GroupStart());
    for (int sh = 0; sh < mg->n_shards; ++sh) {
      const u64 b = mg->ranges[2 * (size_t)sh], e = mg->ranges[2 * (size_t)sh + 1];
      if (e == b) continue;
      const int root = shard_owner(mg->n_shards, mg->world, sh);
      for (MgRank& r : mg->ranks) {
        float* recv = r.y_full + (size_t)b * d;
        const float* send = recv;
        if (r.rank == root)
          for (const MgShard& s : mg->shards)
            if (s.global == sh) send = s.y;
        NCCL_CHECK(nc.Broadcast(send, recv, (size_t)(e - b) * d, ncclFloat, root, r.comm, r.ctx->stream));
      }
    }
    NCCL_CHECK(nc.GroupEnd());
    float worst = 0.f;
    for (MgRank& r : mg->ranks) {
      CUDA_CHECK(cudaSetDevice(r.device));
      CUDA_CHECK(cudaEventRecord(r.ev1, r.ctx->stream));
      CUDA_CHECK(cudaEventSynchronize(r.ev1));
      float t = 0.f;
      CUDA_CHECK(cudaEventElapsedTime(&t, r.ev0, r.ev1));
      worst = std::max(worst, t);
    }
    if (elapsed_ms) *elapsed_ms = worst;
  });
}

int spmx_mg_y_full(const spmx_mg* mg, int local_rank, float** d_y_full) {
  return guarded([&] {
    check(mg);
    if (local_rank < 0 || local_rank >= (int)mg->ranks.size() || !d_y_full)
      throw InvalidArg("spmx_mg_y_full: no such local rank");
    *d_y_full = mg->ranks[(size_t)local_rank].y_full;
  });
}

int spmx_mg_allreduce(spmx_mg* mg, double* values, int count, int op) {
  return guarded([&] {
    check(mg);
    if (count < 0 || count > 16 || (count > 0 && !values)) throw InvalidArg("spmx_mg_allreduce: count must be 0..16");
    if (op != SPMX_REDUCE_SUM && op != SPMX_REDUCE_MAX) throw InvalidArg("spmx_mg_allreduce: unknown op");
    if (count == 0) return;
    if (!mg->has_comm) {
      if (mg->world > 1) throw std::runtime_error("spmx_mg_allreduce: this driver was built without a communicator");
      return;  // one rank: the value is its own reduction
    }
    Nccl& nc = Nccl::require();
    // every local rank contributes the caller's values once: with several ranks in this process
    // the caller passes the per-process figure, and a sum counts it once (first local rank only)
    for (size_t i = 0; i < mg->ranks.size(); ++i) {
      MgRank& r = mg->ranks[i];
      CUDA_CHECK(cudaSetDevice(r.device));
      if (i == 0 || op == SPMX_REDUCE_MAX)
        CUDA_CHECK(cudaMemcpyAsync(r.red, values, (size_t)count * 8, cudaMemcpyHostToDevice, r.ctx->stream));
      else
        CUDA_CHECK(cudaMemsetAsync(r.red, 0, (size_t)count * 8, r.ctx->stream));
    }
    NCCL_CHECK(nc.GroupStart());
    for (MgRank& r : mg->ranks)
      NCCL_CHECK(nc.AllReduce(r.red, r.red, (size_t)count, ncclDouble, op == SPMX_REDUCE_MAX ? ncclMax : ncclSum,
                              r.comm, r.ctx->stream));
    NCCL_CHECK(nc.GroupEnd());
    MgRank& r0 = mg->ranks[0];
    CUDA_CHECK(cudaSetDevice(r0.device));
    CUDA_CHECK(cudaMemcpyAsync(values, r0.red, (size_t)count * 8, cudaMemcpyDeviceToHost, r0.ctx->stream));
    for (MgRank& r : mg->ranks) {
      CUDA_CHECK(cudaSetDevice(r.device));
      CUDA_CHECK(cudaStreamSynchronize(r.ctx->stream));
    }
  });
}

int spmx_mg_synchronize(spmx_mg* mg) {
  return guarded([&] {
    check(mg);
    for (MgRank& r : mg->ranks) {
      CUDA_CHECK(cudaSetDevice(r.device));
      CUDA_CHECK(cudaStreamSynchronize(r.ctx->stream));
    }
  });
}

}  // extern "C"
