/*
 * spmx_b200.h — C ABI of the B200-native CSR SpMM path (libspmx_b200.so).
 *
 * Drop-in boundary for ONE path of the reference (arXiv 2312.05639, "spmx"):
 *   Y = A * X, A in CSR (fp32), X/Y dense row-major fp32, under the three
 *   workload-division schemes (row-split, nnz-split, merge-split).
 *
 * The reference has no C ABI of its own; its FFI-shaped seam is the flat record
 * `KernelArgs` passed by address to the JIT'd code (include/spmx/jit.hpp:16-30)
 * and, one level up, the C++ entry points of include/spmx/partition.hpp:44-68
 * and include/spmx/executor.hpp:44-45. Each function below names the reference
 * interface it replaces (paths relative to /root/reference/proj). The C++ mirror
 * of those entry points (same names and exception behaviour) lives in
 * paper_2312_05639_b200/host/spmx_b200.hpp and is a thin wrapper over this ABI;
 * INTEGRATION.md shows the binding a reference maintainer would add.
 *
 * Conventions: plain pointers and sizes only; every function returns an int
 * status (0 = ok); the message of the last failure on the calling thread is
 * spmx_last_error(). Index types are the reference's: row_ptr uint64,
 * col_indices uint32, values float (include/spmx/csr.hpp:10-20). There is no
 * CPU fallback anywhere behind this ABI: without a CUDA device every compute
 * entry point fails with SPMX_ERUNTIME.
 *
 * Threading (executor.cpp: run_spmm holds no global state): a context and the
 * handles created from it belong to one host thread at a time; concurrent callers use one
 * context each (the thread_local context of INTEGRATION.md). A CSR handle may be shared by the
 * plans of its own context only; a plan owns scratch (the carry rows) that its launches write,
 * so two launches of the same plan must be ordered on the context's stream, which they are.
 */
#ifndef SPMX_B200_H
#define SPMX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the C++ mirror maps them to the reference's exception types */
#define SPMX_OK 0
#define SPMX_EINVAL 1   /* std::invalid_argument: shapes, zero parts, bad diagonal ... */
#define SPMX_ERUNTIME 2 /* std::runtime_error: CUDA failure, no device, out of memory */
#define SPMX_ELOGIC 3   /* std::logic_error: use after destroy, handle/context mismatch */

/* division-method selector == spmx::Strategy (include/spmx/partition.hpp:14) */
#define SPMX_ROW_SPLIT 0
#define SPMX_NNZ_SPLIT 1
#define SPMX_MERGE_SPLIT 2

/* plan flags */
#define SPMX_EXACT_ORDER 1u /* row-granular work items, every Y element one fmaf chain in CSR
                               order: bitwise equal to the reference's run_spmm for all three
                               strategies. Without it (default), ranges heavier
                               than the chunk budget and the merge strategy split rows at nonzero
                               granularity; split rows are summed from per-chunk partials in an
                               order fixed by the plan (CSR order of the pieces; rows cut into more
                               than 16 pieces: 16 runs of consecutive pieces, then the runs) —
                               deterministic, within the north_star tolerance; all other rows stay
                               bitwise equal. */
#define SPMX_JIT_WIDTH 4u   /* instantiate the kernel for exactly this d at run time (NVRTC, cached
                               per d and device) instead of using the runtime-d kernels: the GPU
                               counterpart of the reference's per-d code generation
                               (plan.cpp:80-93, jit.cpp:136-154). d = 32/64/128 are precompiled. */

#define SPMX_CLAIM_KERNEL 8u /* dynamic plans only: run the literal form of the reference's dynamic
                               dispatch (persistent warps claim `batch` rows at a time from a device
                               counter, rows never cut). Without it a dynamic plan is served by the
                               row-split work list, whose chunks the hardware hands to the SMs as
                               they free up (long rows shared between chunks in the default mode,
                               given to the long-row kernel in exact-order mode). Same result. */

typedef struct spmx_ctx spmx_ctx;   /* one per (device, stream) */
typedef struct spmx_csr spmx_csr;   /* A resident on the device */
typedef struct spmx_plan spmx_plan; /* partition of A for one (strategy, parts, flags) */

const char* spmx_last_error(void);
int spmx_abi_version(void);
/* "key=value;" pairs describing the loaded build: SPMX_SASS_SCHED=<n> (kernels whose gather
 * pipeline was re-scheduled after linking, 0 = as compiled), cuda=<CUDART_VERSION>, arch. */
const char* spmx_build_info(void);
/* number of kernels this library has launched on the calling process (all contexts) */
uint64_t spmx_kernel_launch_count(void);

/* ---- context ------------------------------------------------------------------------ */
/* `stream` is a cudaStream_t to run on (borrowed), or NULL to create a private one
 * (cudaStreamNonBlocking: not ordered with the legacy default stream, whose handle is also
 * NULL — a caller whose other work runs on the default stream passes an explicit stream or
 * synchronises before handing device buffers over). */
int spmx_ctx_create(int device, void* stream, spmx_ctx** out);
int spmx_ctx_destroy(spmx_ctx* ctx);
int spmx_ctx_synchronize(spmx_ctx* ctx);
int spmx_ctx_sm_count(spmx_ctx* ctx, int* out);

/* raw device buffers on the context's device (X, Y and staging).
 * Host pointers of every entry point of this header may be pageable (std::vector, malloc — what
 * the reference's CsrMatrix / DenseMatrix hold) or pinned. Pinned (or registered) memory goes to
 * the copy engines directly and the copies are asynchronous on the context's stream. Pageable
 * arrays of 1 MB and more are staged by the library's own host threads (several times the rate of
 * the driver's staging): spmx_h2d then returns when the source has been read, spmx_d2h when the
 * data has arrived — the contract cudaMemcpyAsync has for pageable memory. */
int spmx_dev_alloc(spmx_ctx* ctx, size_t bytes, void** out);
int spmx_dev_free(spmx_ctx* ctx, void* ptr);
int spmx_h2d(spmx_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes);  /* on the ctx stream */
int spmx_d2h(spmx_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes);  /* on the ctx stream */
int spmx_host_alloc_pinned(size_t bytes, void** out);
int spmx_host_free_pinned(void* ptr);

/* ---- CSR: replaces spmx::CsrMatrix as the kernel's input (csr.hpp:10-20, KernelArgs
 *      row_ptr/col_indices/vals, jit.hpp:17-19). Invariants of validate_csr (csr.cpp:18-42)
 *      are checked on the device; a violation is SPMX_EINVAL. ------------------------------ */
int spmx_csr_upload(spmx_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const uint64_t* row_ptr,
                    const uint32_t* col_indices, const float* vals, spmx_csr** out);
/* borrow arrays that already live on the device (no copy, caller keeps ownership) */
int spmx_csr_wrap_device(spmx_ctx* ctx, int64_t m, int64_t n, int64_t nnz,
                         const uint64_t* d_row_ptr, const uint32_t* d_col_indices,
                         const float* d_vals, int validate, spmx_csr** out);
/* structure only: row_ptr without columns or values. Enough for the partitioner and for
 * spmx_plan_create (neither reads col_indices / vals: partition.cpp:35-84 only touches row_ptr);
 * spmx_spmm on such a handle is SPMX_ELOGIC. */
int spmx_rowptr_upload(spmx_ctx* ctx, int64_t m, int64_t nnz, const uint64_t* row_ptr,
                       spmx_csr** out);
int spmx_csr_destroy(spmx_csr* a);
int spmx_csr_dims(const spmx_csr* a, int64_t* m, int64_t* n, int64_t* nnz);

/* ---- partitioner, computed on the device, bit-exact with src/partition.cpp.
 *      Ranges are written to HOST memory as out[2t] = begin, out[2t+1] = end (RowRange,
 *      partition.hpp:18-24). ---------------------------------------------------------------- */
/* split_rows_static(m, T), partition.cpp:17-27 */
int spmx_split_rows_static(spmx_ctx* ctx, uint64_t m, unsigned parts, uint64_t* out_ranges);
/* split_nnz(A, T), partition.cpp:35-51 */
int spmx_split_nnz(spmx_ctx* ctx, const spmx_csr* a, unsigned parts, uint64_t* out_ranges);
/* split_merge(A, T), partition.cpp:69-84 (row-snapped) */
int spmx_split_merge(spmx_ctx* ctx, const spmx_csr* a, unsigned parts, uint64_t* out_ranges);
/* merge_path_search(k, row_end, m, nnz), partition.cpp:53-67, for n_diag diagonals at once;
 * any k > m + nnz is SPMX_EINVAL (the reference throws invalid_argument). */
int spmx_merge_path_search(spmx_ctx* ctx, const spmx_csr* a, size_t n_diag, const uint64_t* k,
                           uint64_t* out_i, uint64_t* out_j);
/* next_batch(counter, batch, m), partition.cpp:29-33: claims `n_claims` batches from one device
 * counter with concurrent atomics (one claim per thread) and returns the claimed ranges (begin ==
 * end == UINT64_MAX where the reference returns nullopt), in arbitrary order. */
int spmx_next_batch_claims(spmx_ctx* ctx, uint64_t m, uint64_t batch, size_t n_claims,
                           uint64_t* out_ranges);

/* ---- plan: make_partition(A, strategy, T, dynamic, batch) (partition.cpp:86-104) plus the
 *      device work list derived from it. parts == 0 picks a default that fills the GPU.
 *      dynamic != 0 (row-split only, else SPMX_EINVAL; no RowRange list, as in the reference)
 *      asks for dynamic dispatch, the analogue of DispatchCounter (partition.hpp:38-40): see
 *      SPMX_CLAIM_KERNEL for how it runs. */
int spmx_plan_create(spmx_ctx* ctx, const spmx_csr* a, int strategy, unsigned parts, int dynamic,
                     uint64_t batch, unsigned flags, spmx_plan** out);
int spmx_plan_destroy(spmx_plan* p);
/* the plan's strategy-level ranges (bit-exact with the reference's make_partition; `parts`
 * entries, none under dynamic dispatch) and its device work-list size */
int spmx_plan_info(const spmx_plan* p, unsigned* parts, uint64_t* n_chunks, int* dynamic);
int spmx_plan_ranges(const spmx_plan* p, uint64_t* out_ranges);
/* work-list coordinates (row, nnz) of the n_chunks+1 chunk boundaries */
int spmx_plan_chunks(const spmx_plan* p, uint64_t* out_row, uint64_t* out_nnz);

/* ---- the kernel: replaces the JIT'd EntryFn called per worker (jit.hpp:30, executor.cpp:77-87).
 *      d_x: N x d, d_y: M x d, row-major fp32 on the device (DenseMatrix, dense.hpp:9-21).
 *      Every row of Y is overwritten, empty rows with zeros (interp.cpp:53).
 *      elapsed_ms, when non-NULL, receives the device time of the launch(es) measured with CUDA
 *      events on the context's stream (the call then synchronises). -------------------------- */
int spmx_spmm(spmx_ctx* ctx, const spmx_plan* plan, const spmx_csr* a, const float* d_x,
              int64_t x_rows, int64_t d, float* d_y, float* elapsed_ms);

/* ---- run_spmm(A, X, cfg) with HOST buffers (executor.hpp:44-45): upload A and X, partition,
 *      multiply, download Y, pipelined over row blocks (col/vals upload, compute and Y download
 *      overlap). times_ms[0..5] (optional) = {row_ptr upload + plan, same, X upload wait,
 *      first block ready -> last Y byte, total wall, number of blocks}.
 *      For repeated calls on the same matrix keep the handles and use spmx_spmm instead. ------ */
int spmx_spmm_host(spmx_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const uint64_t* row_ptr,
                   const uint32_t* col_indices, const float* vals, const float* x, int64_t x_rows,
                   int64_t d, float* y, int strategy, unsigned parts, int dynamic, uint64_t batch,
                   unsigned flags, double* times_ms);

/* ---- verification, on the device (RunConfig.verify, executor.cpp:110) ------------------------
 * spmm_reference (reference.cpp:10-25, Alg. 1): one thread per output element, multiply then
 * add with two roundings, CSR order — bitwise equal to the reference's serial loop. */
int spmx_spmm_reference(spmx_ctx* ctx, const spmx_csr* a, const float* d_x, int64_t x_rows,
                        int64_t d, float* d_y);
/* max_relative_error (executor.cpp:27-34): max_i |y_i - ref_i| / max(|ref_i|, 1e-6) */
int spmx_max_relative_error(spmx_ctx* ctx, const float* d_y, const float* d_ref, size_t count,
                            double* out);

/* run-time code generation counters (RunReport.codegen_s of the reference, executor.cpp:54-60):
 * kernels compiled so far in this process and the seconds spent compiling them */
int spmx_jit_stats(uint64_t* kernels_compiled, double* seconds);
/* 1 when the run-time compiler (libnvrtc) can be loaded, i.e. SPMX_JIT_WIDTH can be honoured */
int spmx_jit_available(void);

/* L2 residency control for the context's stream: kernels launched after this call treat
 * [base, base + bytes) as a persisting access-policy window (hit ratio hit_ratio, everything else
 * streaming); bytes == 0 removes the window and resets the persisting lines. The window is clipped
 * to the device's limits (out_window_bytes, may be NULL). For callers whose hottest X rows are
 * contiguous (e.g. a column ordering by degree): tools/exp_hot_window.py measures what it buys. */
int spmx_ctx_l2_window(spmx_ctx* ctx, const void* base, size_t bytes, float hit_ratio,
                       size_t* out_window_bytes);

/* Self-check builds only (-DSPMX_DEBUG_BOUNDS=1, tools/bounds_check.py): per-site counts of
 * out-of-bounds accesses the SpMM kernels would have made (all zero = clean). A regular build
 * answers SPMX_ELOGIC. compute-sanitizer is not available on the GPU pool this was developed on. */
int spmx_debug_bounds(uint64_t* out16);

/* Measurement aid (bench.py roofline.gather): the L2 -> SM ceiling of this GPU at its current
 * clocks — random 256-byte rows of an L2-resident 64 MB buffer read by 8-lane groups with
 * LDG.128 (the SpMM's own access shape at d = 64), at 24, 32, 40 and 48 warps per SM; the best of
 * `repeats` launches each, in TB/s over the whole chip, and that launch's duration. Not on the hot path. */
int spmx_probe_l2_to_sm(spmx_ctx* ctx, int repeats, double* out_tbs, double* out_ms);

/* ---- helpers for the reference's report fields ---------------------------------------------- */
/* checksum(Y), dense.cpp:17-28, of a device buffer (FNV-1a is sequential: the buffer is copied
 * to the host and hashed there; a reporting helper, not on the hot path) */
int spmx_checksum_device(spmx_ctx* ctx, const float* d_y, size_t count, uint64_t* out);

/* ---- multi-GPU driver (north_star item 3) ------------------------------------
 * The reference parallelises ONE way: contiguous row ranges of A, one per worker, joined by a
 * barrier (fork-join over RowRanges, executor.cpp:66-99; single writer per output row,
 * SPEC.md:439). The driver applies the same division one level up: A is cut into G row blocks
 * ("shards") by the reference's own split_nnz(A, G) (partition.cpp:35-51; split_merge(A, G),
 * partition.cpp:69-84, on request), computed by the device partitioner and therefore bit-exact
 * with it; shard g lives on one GPU with a rebased row_ptr; X is replicated by ONE NCCL
 * broadcast; every GPU multiplies its shards with its own plan (the chosen Strategy divides the
 * shard again among the SMs); Y stays row-sharded. No collective is on the data path. An
 * all-gather-v of Y (one ncclBroadcast per shard inside one NCCL group, no padding) is offered
 * and timed separately.
 *
 * Two ways to build the communicator:
 *   spmx_mg_create       one process drives n_devices GPUs (ncclCommInitAll), one context and
 *                        stream per GPU — the C++ mirror's RunConfig.gpus and the CLI's --gpus;
 *   spmx_mg_create_rank  one process per GPU (torchrun / mpirun): rank `rank` of `world`, the
 *                        128-byte id made by spmx_mg_unique_id on rank 0 and handed to the
 *                        other ranks by the launcher. id128 == NULL builds the driver without a
 *                        communicator (world must then be served by another transport: only
 *                        the shard / plan / spmm calls work; used to exercise the rank code
 *                        path with several processes on one GPU).
 * n_shards == 0 means one shard per rank; n_shards > world puts several shards on a rank
 * (shard g on rank g * world / n_shards, run back to back on that rank's stream), which lets one
 * GPU stand in for a node in the tests. NCCL is loaded with dlopen (SPMX_NCCL_LIB, then
 * libnccl.so.2): the library has no link-time dependency on it, and the single-GPU entry
 * points above never touch it. Every rank calls every spmx_mg_* function with the same
 * arguments (its own copy of A's arrays), like any SPMD collective API. */
typedef struct spmx_mg spmx_mg;

#define SPMX_SHARD_BY_NNZ 1   /* split_nnz(A, G): equal nonzeros per shard (north_star) */
#define SPMX_SHARD_BY_MERGE 2 /* split_merge(A, G): equal rows + nonzeros per shard */

int spmx_mg_create(int n_devices, const int* devices, int n_shards, spmx_mg** out);
int spmx_mg_unique_id(void* out128);
int spmx_mg_create_rank(int device, void* stream, int rank, int world, int n_shards,
                        const void* id128, spmx_mg** out);
int spmx_mg_destroy(spmx_mg* mg);
/* world size, ranks driven by this process, shards in total / on this process, NCCL version
 * (0 without a communicator); any pointer may be NULL */
int spmx_mg_info(const spmx_mg* mg, int* world, int* n_local_ranks, int* n_shards,
                 int* n_local_shards, int* nccl_version);
/* pure host function: the rank that owns shard g (g * world / n_shards) */
int spmx_mg_shard_owner(int n_shards, int world, int shard);

/* Cut A into the driver's shards and place every LOCAL shard on its GPU. *_host reads the
 * reference's host arrays (CsrMatrix fields, csr.hpp:10-20): row_ptr goes to the first local GPU
 * once (structure only), col/vals slices go straight to their owners. *_device takes arrays
 * that already live on local rank `src_local_rank`'s GPU (copied device to device / peer to
 * peer). out_ranges (2 * n_shards, may be NULL) receives ALL shards' row ranges, which are
 * bit-exact with split_nnz / split_merge of the reference. Replaces any earlier sharding. */
int spmx_mg_shard_host(spmx_mg* mg, int64_t m, int64_t n, int64_t nnz, const uint64_t* row_ptr,
                       const uint32_t* col_indices, const float* vals, int shard_by,
                       uint64_t* out_ranges);
int spmx_mg_shard_device(spmx_mg* mg, int src_local_rank, int64_t m, int64_t n, int64_t nnz,
                         const uint64_t* d_row_ptr, const uint32_t* d_col_indices,
                         const float* d_vals, int shard_by, uint64_t* out_ranges);
/* local shard i: its global index, the device it lives on, its rows [begin, end) of A and nnz */
int spmx_mg_shard_info(const spmx_mg* mg, int local_shard, int* global_shard, int* device,
                       uint64_t* row_begin, uint64_t* row_end, uint64_t* nnz);

/* make_partition per shard (spmx_plan_create on every local shard) */
int spmx_mg_plan(spmx_mg* mg, int strategy, unsigned parts, int dynamic, uint64_t batch,
                 unsigned flags);

/* X (x_rows x d) to every GPU with ONE ncclBroadcast from rank root_rank, timed with CUDA events
 * (max over this process's ranks). *_host: the process that drives root_rank passes its host
 * matrix (uploaded to the root GPU first, h2d_ms), the driver owns the device copies.
 * *_device: d_x_local[i] is local rank i's x_rows x d buffer (borrowed; the root's holds X). */
int spmx_mg_broadcast_x_host(spmx_mg* mg, const float* x_host, int root_rank, int64_t x_rows,
                             int64_t d, float* h2d_ms, float* bcast_ms);
int spmx_mg_broadcast_x_device(spmx_mg* mg, float* const* d_x_local, int root_rank,
                               int64_t x_rows, int64_t d, float* bcast_ms);
/* as *_host, with the root's X already on the root's GPU (copied device to device into the
 * driver's buffer first, copy_ms). With driver-owned replicas (*_host and this call) every rank
 * also keeps a compact copy of its shards' hottest X rows behind X (SPMX_MG_HOT_ROWS, default
 * 50 000 per rank, 0 = off), remaps those columns of its shards to the copy and, when X is at
 * least SPMX_MG_HOT_MIN_MB (default 1024) large, protects the copy with a persisting L2 window:
 * on matrices whose X is far larger than the L2 the hot rows then stay resident (c5: DRAM reads
 * 85.7 -> 75.2 GB per multiply). Values, summation order and results are unchanged. */
int spmx_mg_broadcast_x_from_device(spmx_mg* mg, const float* d_x_root, int root_rank,
                                    int64_t x_rows, int64_t d, float* copy_ms, float* bcast_ms);

/* Y_g = A_g * X on every local shard (run_spmm's parallel region, executor.cpp:70-97, with
 * GPUs for threads), `steps` times back to back (the reference's trials loop, executor.cpp:68).
 * step_ms = max over this process's ranks of the device time of that rank's launches (CUDA
 * events on the rank's stream) / steps; ms_per_local_shard (may be NULL) gets each shard's own
 * time in the last step. The ranks never wait for each other. The call returns when every
 * local rank has finished. */
int spmx_mg_spmm(spmx_mg* mg, int steps, float* step_ms, float* ms_per_local_shard);
/* device pointer of local shard i's Y block ((row_end - row_begin) x d, owned by the driver) */
int spmx_mg_y_shard(const spmx_mg* mg, int local_shard, float** d_y);
/* the local shards' rows of Y into a host M x d matrix (other rows are left untouched) */
int spmx_mg_download_y(spmx_mg* mg, float* y_host);
/* every local shard's Y block into its own host buffer (host_per_local_shard[i]: rows_i x d
 * floats): the per-process form of the call above (one process per GPU keeps only its rows) */
int spmx_mg_download_y_shards(spmx_mg* mg, float* const* host_per_local_shard);
/* optional: the full M x d Y on every GPU, one ncclBroadcast per shard in one group
 * (all-gather-v: shards have unequal row counts, nothing is padded) */
int spmx_mg_allgather_y(spmx_mg* mg, float* elapsed_ms);
int spmx_mg_y_full(const spmx_mg* mg, int local_rank, float** d_y_full);

/* Statistics across ranks (max of the step time, sum of nonzeros ...): values[0..count) are
 * reduced over all `world` ranks with one ncclAllReduce and written back; count <= 16. A process
 * that drives several ranks passes its per-process figures (a sum counts them once). */
#define SPMX_REDUCE_SUM 0
#define SPMX_REDUCE_MAX 1
int spmx_mg_allreduce(spmx_mg* mg, double* values, int count, int op);
/* waits for every local rank's stream */
int spmx_mg_synchronize(spmx_mg* mg);

#ifdef __cplusplus
}
#endif
#endif /* SPMX_B200_H */
