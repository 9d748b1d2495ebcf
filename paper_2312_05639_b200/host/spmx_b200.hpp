// spmx_b200.hpp — C++ host mirror of the reference's public API for the SpMM path, over the
// C ABI of libspmx_b200.so (include/spmx_b200.h). Header-only; link with -lspmx_b200.
//
// Same names, argument meaning and error behaviour as the reference (namespace spmx,
// /root/reference/proj/include/spmx/{csr,dense,partition,executor}.hpp), so code written
// against the reference — including its tests — compiles against this header unchanged for
// the path in scope:
//     CsrMatrix, DenseMatrix, Strategy, RowRange, WorkPartition, MergeCoordinate,
//     split_rows_static, split_nnz, split_merge, merge_path_search, make_partition,
//     RunConfig, RunReport, run_spmm, max_relative_error, checksum, kVerifyTolerance.
// Differences, all forced by the device:
//   * the work runs on a B200 through hand-written CUDA kernels; there is no CPU fallback;
//   * RunConfig.threads is the number of partition ranges T (0 = a default that fills the
//     GPU), not OS threads; RunReport.threads echoes it;
//   * Backend::Native is the default device mode (ranges heavier than a chunk and the merge
//     strategy split rows at nonzero granularity; deterministic, within the reference's
//     1e-5 verify tolerance); Backend::Interp — the reference's bitwise oracle — selects
//     SPMX_EXACT_ORDER, whose result is bitwise equal to the reference's for every
//     strategy and T;
//   * codegen_s reports the plan construction (device partitioner + work list), the step
//     that — like the reference's code generation — happens once before the timed trials;
//   * tier_cap and collect_counters are accepted and ignored (x86-only concepts).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/spmx_b200.h"
#include "spmx_types.hpp"

namespace spmx {

enum class Strategy { RowSplit, NnzSplit, MergeSplit };
inline const char* strategy_name(Strategy s) {
  return s == Strategy::RowSplit ? "row" : s == Strategy::NnzSplit ? "nnz" : "merge";
}

struct RowRange {
  uint64_t begin = 0, end = 0;
  uint64_t size() const { return end - begin; }
  bool operator==(const RowRange&) const = default;
};
struct DispatchConfig {
  uint64_t batch_size = 128;
};
struct WorkPartition {
  Strategy strategy = Strategy::RowSplit;
  std::vector<RowRange> ranges;  // empty under dynamic dispatch
  std::optional<DispatchConfig> dynamic;
};
struct MergeCoordinate {
  uint64_t i = 0, j = 0;
};

namespace detail {

// status code -> the reference's exception type
inline void check(int rc) {
  if (rc == SPMX_OK) return;
  const std::string msg = spmx_last_error();
  if (rc == SPMX_EINVAL) throw std::invalid_argument(msg);
  if (rc == SPMX_ELOGIC) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}

inline int to_c(Strategy s) {
  return s == Strategy::RowSplit ? SPMX_ROW_SPLIT
                                 : s == Strategy::NnzSplit ? SPMX_NNZ_SPLIT : SPMX_MERGE_SPLIT;
}

// RAII over the opaque handles
struct Ctx {
  spmx_ctx* h = nullptr;
  explicit Ctx(int device = 0) { check(spmx_ctx_create(device, nullptr, &h)); }
  ~Ctx() { if (h) spmx_ctx_destroy(h); }
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
};
struct DevCsr {
  spmx_csr* h = nullptr;
  DevCsr(Ctx& c, const CsrMatrix& a) {
    if (a.row_ptr.size() != size_t(a.m) + 1)
      throw std::invalid_argument("invalid CSR: row_ptr length != m+1");
    if (a.col_indices.size() != size_t(a.nnz) || a.vals.size() != size_t(a.nnz))
      throw std::invalid_argument("invalid CSR: col_indices/vals length != nnz");
    check(spmx_csr_upload(c.h, a.m, a.n, a.nnz, a.row_ptr.data(), a.col_indices.data(),
                          a.vals.data(), &h));
  }
  // structure only (partition functions never read columns or values): row_ptr is all that
  // crosses the bus
  DevCsr(Ctx& c, int64_t m, int64_t nnz, const uint64_t* row_ptr) {
    check(spmx_rowptr_upload(c.h, m, nnz, row_ptr, &h));
  }
  ~DevCsr() { if (h) spmx_csr_destroy(h); }
  DevCsr(const DevCsr&) = delete;
  DevCsr& operator=(const DevCsr&) = delete;
};
struct DevBuf {
  Ctx& c;
  void* p = nullptr;
  DevBuf(Ctx& ctx, size_t bytes) : c(ctx) { check(spmx_dev_alloc(c.h, bytes, &p)); }
  ~DevBuf() { if (p) spmx_dev_free(c.h, p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};
struct Plan {
  spmx_plan* h = nullptr;
  ~Plan() { if (h) spmx_plan_destroy(h); }
};

inline std::vector<RowRange> to_ranges(const std::vector<uint64_t>& flat) {
  std::vector<RowRange> r(flat.size() / 2);
  for (size_t t = 0; t < r.size(); ++t) r[t] = {flat[2 * t], flat[2 * t + 1]};
  return r;
}

inline double now_s();

// One context per host thread and device, created on first use and kept for the thread's
// lifetime: the reference's entry points hold no global state and may be called concurrently
// (SPEC.md:342), a context belongs to one host thread at a time (include/spmx_b200.h).
inline Ctx& thread_ctx(int device = 0) {
  thread_local std::vector<std::unique_ptr<Ctx>> per_device;
  if (device < 0) throw std::invalid_argument("no such device");
  if (per_device.size() <= size_t(device)) per_device.resize(size_t(device) + 1);
  if (!per_device[size_t(device)]) per_device[size_t(device)] = std::make_unique<Ctx>(device);
  return *per_device[size_t(device)];
}

}  // namespace detail

// ---- partitioner (partition.hpp:44-68), computed on the device, bit-exact ----------------------
inline std::vector<RowRange> split_rows_static(uint64_t m, unsigned threads) {
  if (threads == 0) throw std::invalid_argument("split_rows_static: zero threads");
  detail::Ctx& c = detail::thread_ctx();
  std::vector<uint64_t> flat(2 * size_t(threads));
  detail::check(spmx_split_rows_static(c.h, m, threads, flat.data()));
  return detail::to_ranges(flat);
}

inline std::vector<RowRange> split_nnz(const CsrMatrix& a, unsigned threads) {
  if (threads == 0) throw std::invalid_argument("split_nnz: zero threads");
  detail::Ctx& c = detail::thread_ctx();
  detail::DevCsr d(c, a.m, a.nnz, a.row_ptr.data());
  std::vector<uint64_t> flat(2 * size_t(threads));
  detail::check(spmx_split_nnz(c.h, d.h, threads, flat.data()));
  return detail::to_ranges(flat);
}

inline std::vector<RowRange> split_merge(const CsrMatrix& a, unsigned threads) {
  if (threads == 0) throw std::invalid_argument("split_merge: zero threads");
  detail::Ctx& c = detail::thread_ctx();
  detail::DevCsr d(c, a.m, a.nnz, a.row_ptr.data());
  std::vector<uint64_t> flat(2 * size_t(threads));
  detail::check(spmx_split_merge(c.h, d.h, threads, flat.data()));
  return detail::to_ranges(flat);
}

// row_end[r] == row_ptr[r+1], exactly as the reference takes it (partition.hpp:56-58);
// row_end - 1 must therefore be the start of a row_ptr array of m+1 entries.
inline MergeCoordinate merge_path_search(uint64_t k, const uint64_t* row_end, uint64_t m,
                                         uint64_t nnz) {
  if (k > m + nnz) throw std::invalid_argument("merge_path_search: diagonal out of range");
  detail::Ctx& c = detail::thread_ctx();
  detail::DevCsr d(c, int64_t(m), int64_t(nnz), row_end - 1);
  MergeCoordinate out;
  detail::check(spmx_merge_path_search(c.h, d.h, 1, &k, &out.i, &out.j));
  return out;
}

// many diagonals at once (one upload): the efficient form of the call above
inline std::vector<MergeCoordinate> merge_path_search(const CsrMatrix& a,
                                                      const std::vector<uint64_t>& ks) {
  detail::Ctx& c = detail::thread_ctx();
  detail::DevCsr d(c, a.m, a.nnz, a.row_ptr.data());
  std::vector<uint64_t> oi(ks.size()), oj(ks.size());
  detail::check(spmx_merge_path_search(c.h, d.h, ks.size(), ks.data(), oi.data(), oj.data()));
  std::vector<MergeCoordinate> out(ks.size());
  for (size_t t = 0; t < ks.size(); ++t) out[t] = {oi[t], oj[t]};
  return out;
}

inline WorkPartition make_partition(const CsrMatrix& a, Strategy strategy, unsigned threads,
                                    bool dynamic_dispatch, uint64_t batch_size) {
  if (threads == 0) throw std::invalid_argument("make_partition: zero threads");
  WorkPartition p;
  p.strategy = strategy;
  if (dynamic_dispatch) {
    if (strategy != Strategy::RowSplit)
      throw std::invalid_argument("dynamic dispatch pairs with row-split only");
    if (batch_size == 0) throw std::invalid_argument("batch_size must be >= 1");
    p.dynamic = DispatchConfig{batch_size};
    return p;
  }
  switch (strategy) {
    case Strategy::RowSplit: p.ranges = split_rows_static(uint64_t(a.m), threads); break;
    case Strategy::NnzSplit: p.ranges = split_nnz(a, threads); break;
    case Strategy::MergeSplit: p.ranges = split_merge(a, threads); break;
  }
  return p;
}

// ---- executor (executor.hpp:20-50) ---------------------------------------------------------------------
enum class Backend { Native, Interp };
inline const char* backend_name(Backend b) { return b == Backend::Native ? "native" : "interp"; }
enum class SimdTier { Scalar, V256, V512 };  // kept for source compatibility; unused on the GPU

struct RunConfig {
  Strategy strategy = Strategy::RowSplit;
  bool dynamic_dispatch = true;  // RowSplit only
  unsigned threads = 0;          // partition ranges T; 0 = fill the GPU
  Backend backend = Backend::Native;
  std::optional<SimdTier> tier_cap;
  uint64_t batch_size = 128;
  bool verify = false;
  unsigned trials = 1;
  bool collect_counters = false;
  int device = 0;          // extension: which GPU (the first one when gpus > 1)
  unsigned gpus = 1;       // extension: row-shard A over GPUs device .. device+gpus-1 through the
                           // library's multi-GPU driver (spmx_mg_*): the reference's fork-join over
                           // RowRanges (executor.cpp:66-99) with GPUs for workers, ranges from
                           // split_nnz(A, gpus) (partition.cpp:35-51); X replicated by one NCCL
                           // broadcast, Y row-sharded. The Strategy divides every shard again.
  unsigned shards = 0;     // extension: row blocks (0 = one per GPU; more puts several on a GPU)
  bool shard_by_merge = false;  // extension: split_merge(A, gpus) instead of split_nnz
  bool jit_width = true;   // extension: compile the kernel for exactly X.cols at run time (NVRTC,
                           // cached per d; d = 32/64/128 are precompiled), the counterpart of the
                           // reference's per-d code generation behind Backend::Native. Ignored
                           // when libnvrtc cannot be loaded (the runtime-d kernels run instead).
};

struct RunReport {
  std::vector<double> times_s;  // device time of each trial (CUDA events)
  double mean_s = 0.0;
  double codegen_s = 0.0;  // plan construction
  double gflops = 0.0;     // 2*nnz*d / mean_s / 1e9
  SimdTier tier = SimdTier::Scalar;
  unsigned threads = 0;
  std::optional<double> max_rel_err;  // when verify is set
  uint64_t n_chunks = 0;              // extension: size of the device work list
  unsigned gpus = 1;                  // extension: GPUs that shared the rows
  double x_broadcast_s = 0.0;         // extension: the one NCCL broadcast of X (gpus > 1)
  std::vector<RowRange> shard_rows;   // extension: the row block of every shard (gpus > 1)
};

inline constexpr double kVerifyTolerance = 1e-5;

// executor.cpp:27-34
inline double max_relative_error(const DenseMatrix& y, const DenseMatrix& ref) {
  if (y.data.size() != ref.data.size())
    throw std::invalid_argument("max_relative_error: shape mismatch");
  detail::Ctx& c = detail::thread_ctx();
  const size_t bytes = y.data.size() * sizeof(float);
  detail::DevBuf dy(c, bytes), dr(c, bytes);
  detail::check(spmx_h2d(c.h, dy.p, y.data.data(), bytes));
  detail::check(spmx_h2d(c.h, dr.p, ref.data.data(), bytes));
  double out = 0.0;
  detail::check(spmx_max_relative_error(c.h, (const float*)dy.p, (const float*)dr.p,
                                        y.data.size(), &out));
  return out;
}

// dense.cpp:17-28: FNV-1a-64 over the little-endian f32 bytes (sequential by definition)
inline uint64_t checksum(const DenseMatrix& y) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (float f : y.data) {
    uint32_t bits;
    std::memcpy(&bits, &f, 4);
    for (int s = 0; s < 32; s += 8) {
      h ^= (bits >> s) & 0xffu;
      h *= 0x100000001b3ull;
    }
  }
  return h;
}

// reference.hpp:11 — Alg. 1 (unfused), evaluated on the device
inline DenseMatrix spmm_reference(const CsrMatrix& a, const DenseMatrix& x) {
  if (a.n != x.rows) throw std::invalid_argument("spmm_reference: A.n != X.rows");
  detail::Ctx& c = detail::thread_ctx();
  detail::DevCsr da(c, a);
  DenseMatrix y(a.m, x.cols);
  detail::DevBuf dx(c, x.data.size() * 4), dy(c, y.data.size() * 4);
  detail::check(spmx_h2d(c.h, dx.p, x.data.data(), x.data.size() * 4));
  detail::check(spmx_spmm_reference(c.h, da.h, (const float*)dx.p, x.rows, x.cols, (float*)dy.p));
  detail::check(spmx_d2h(c.h, y.data.data(), dy.p, y.data.size() * 4));
  detail::check(spmx_ctx_synchronize(c.h));
  return y;
}

namespace detail {

struct Mg {
  spmx_mg* h = nullptr;
  ~Mg() { if (h) spmx_mg_destroy(h); }
};

// run_spmm over several GPUs (RunConfig.gpus > 1 or shards > 1): same contract, the rows of A
// divided among the GPUs first. Times are the max over GPUs of each GPU's own device time.
inline std::pair<DenseMatrix, RunReport> run_spmm_multi(const CsrMatrix& a, const DenseMatrix& x,
                                                        const RunConfig& cfg, bool dynamic,
                                                        unsigned flags) {
  if (a.row_ptr.size() != size_t(a.m) + 1)
    throw std::invalid_argument("invalid CSR: row_ptr length != m+1");
  if (a.col_indices.size() != size_t(a.nnz) || a.vals.size() != size_t(a.nnz))
    throw std::invalid_argument("invalid CSR: col_indices/vals length != nnz");
  const unsigned gpus = std::max(cfg.gpus, 1u);
  std::vector<int> devices(gpus);
  for (unsigned g = 0; g < gpus; ++g) devices[g] = cfg.device + int(g);
  Mg mg;
  check(spmx_mg_create(int(gpus), devices.data(), int(cfg.shards), &mg.h));
  int n_shards = 0;
  check(spmx_mg_info(mg.h, nullptr, nullptr, &n_shards, nullptr, nullptr));
  std::vector<uint64_t> flat(2 * size_t(n_shards));
  check(spmx_mg_shard_host(mg.h, a.m, a.n, a.nnz, a.row_ptr.data(), a.col_indices.data(), a.vals.data(),
                           cfg.shard_by_merge ? SPMX_SHARD_BY_MERGE : SPMX_SHARD_BY_NNZ, flat.data()));
  const int64_t d = x.cols;
  float h2d_ms = 0.f, bcast_ms = 0.f;
  check(spmx_mg_broadcast_x_host(mg.h, x.data.data(), 0, x.rows, d, &h2d_ms, &bcast_ms));

  RunReport report;
  report.gpus = gpus;
  report.x_broadcast_s = double(bcast_ms) * 1e-3;
  report.shard_rows = to_ranges(flat);
  {
    const double t0 = now_s();
    check(spmx_mg_plan(mg.h, to_c(cfg.strategy), cfg.threads, dynamic ? 1 : 0, cfg.batch_size, flags));
    check(spmx_mg_synchronize(mg.h));
    report.codegen_s = now_s() - t0;
  }
  report.threads = cfg.threads;
  if (flags & SPMX_JIT_WIDTH) {  // run-time code generation happens on the first launch for this d
    double before = 0.0, after = 0.0;
    check(spmx_jit_stats(nullptr, &before));
    check(spmx_mg_spmm(mg.h, 1, nullptr, nullptr));
    check(spmx_jit_stats(nullptr, &after));
    report.codegen_s += after - before;
  }
  for (unsigned trial = 0; trial < cfg.trials; ++trial) {
    float ms = 0.0f;
    check(spmx_mg_spmm(mg.h, 1, &ms, nullptr));
    report.times_s.push_back(double(ms) * 1e-3);
  }
  double sum = 0.0;
  for (double t : report.times_s) sum += t;
  report.mean_s = sum / double(report.times_s.size());
  report.gflops = report.mean_s > 0.0 ? 2.0 * double(a.nnz) * double(d) / report.mean_s / 1e9 : 0.0;
  DenseMatrix y(a.m, d);
  check(spmx_mg_download_y(mg.h, y.data.data()));
  if (cfg.verify) report.max_rel_err = max_relative_error(y, spmm_reference(a, x));
  return {std::move(y), std::move(report)};
}

}  // namespace detail

// executor.hpp:44-45
inline std::pair<DenseMatrix, RunReport> run_spmm(const CsrMatrix& a, const DenseMatrix& x,
                                                  const RunConfig& cfg) {
  // executor.cpp:38-46, same order and messages
  if (a.n != x.rows) throw std::invalid_argument("run_spmm: A.n != X.rows");
  if (cfg.trials < 1) throw std::invalid_argument("run_spmm: trials must be >= 1");
  if (cfg.batch_size < 1) throw std::invalid_argument("run_spmm: batch_size must be >= 1");
  if (cfg.dynamic_dispatch && cfg.strategy != Strategy::RowSplit)
    throw std::invalid_argument("dynamic dispatch pairs with row-split only");
  const bool dynamic = cfg.dynamic_dispatch && cfg.strategy == Strategy::RowSplit;
  const bool jit = cfg.jit_width && spmx_jit_available() != 0;
  const unsigned flags = (cfg.backend == Backend::Interp ? SPMX_EXACT_ORDER : 0u) |
                         (jit ? SPMX_JIT_WIDTH : 0u);

  if (cfg.gpus > 1 || cfg.shards > 1) return detail::run_spmm_multi(a, x, cfg, dynamic, flags);

  detail::Ctx& c = detail::thread_ctx(cfg.device);
  detail::DevCsr da(c, a);
  const int64_t d = x.cols;
  DenseMatrix y(a.m, d);
  detail::DevBuf dx(c, x.data.size() * 4), dy(c, y.data.size() * 4);
  detail::check(spmx_h2d(c.h, dx.p, x.data.data(), x.data.size() * 4));

  RunReport report;
  detail::Plan plan;
  {
    // plan once per run, before the timed trials (executor.cpp:54-62)
    detail::check(spmx_ctx_synchronize(c.h));
    const double t0 = detail::now_s();
    detail::check(spmx_plan_create(c.h, da.h, detail::to_c(cfg.strategy), cfg.threads,
                                   dynamic ? 1 : 0, cfg.batch_size, flags, &plan.h));
    detail::check(spmx_ctx_synchronize(c.h));
    report.codegen_s = detail::now_s() - t0;
  }
  unsigned parts = 0;
  uint64_t chunks = 0;
  detail::check(spmx_plan_info(plan.h, &parts, &chunks, nullptr));
  report.threads = parts;
  report.n_chunks = chunks;
  if (jit) {  // code generation happens on the first launch for this d: keep it out of
    double before = 0.0, after = 0.0;  // the timed trials, like the reference's emit()
    detail::check(spmx_jit_stats(nullptr, &before));
    detail::check(spmx_spmm(c.h, plan.h, da.h, (const float*)dx.p, x.rows, d, (float*)dy.p, nullptr));
    detail::check(spmx_ctx_synchronize(c.h));
    detail::check(spmx_jit_stats(nullptr, &after));
    report.codegen_s += after - before;
  }
  for (unsigned trial = 0; trial < cfg.trials; ++trial) {
    float ms = 0.0f;
    detail::check(spmx_spmm(c.h, plan.h, da.h, (const float*)dx.p, x.rows, d, (float*)dy.p, &ms));
    report.times_s.push_back(double(ms) * 1e-3);
  }
  double sum = 0.0;
  for (double t : report.times_s) sum += t;
  report.mean_s = sum / double(report.times_s.size());
  report.gflops = report.mean_s > 0.0 ? 2.0 * double(a.nnz) * double(d) / report.mean_s / 1e9 : 0.0;
  if (cfg.verify) {
    detail::DevBuf dref(c, y.data.size() * 4);
    detail::check(spmx_spmm_reference(c.h, da.h, (const float*)dx.p, x.rows, d, (float*)dref.p));
    double e = 0.0;
    detail::check(spmx_max_relative_error(c.h, (const float*)dy.p, (const float*)dref.p,
                                          y.data.size(), &e));
    report.max_rel_err = e;
  }
  detail::check(spmx_d2h(c.h, y.data.data(), dy.p, y.data.size() * 4));
  detail::check(spmx_ctx_synchronize(c.h));
  return {std::move(y), std::move(report)};
}

}  // namespace spmx

#include <chrono>
inline double spmx::detail::now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
