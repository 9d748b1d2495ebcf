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
#define SPMX_NO_COOP 2u     /* reserved (no effect) */
#define SPMX_JIT_WIDTH 4u   /* instantiate the kernel for exactly this d at run time (NVRTC, cached
                               per d and device) instead of using the runtime-d kernels: the GPU
                               counterpart of the reference's per-d code generation
                               (plan.cpp:80-93, jit.cpp:136-154). d = 32/64/128 are precompiled. */

typedef struct spmx_ctx spmx_ctx;   /* one per (device, stream) */
typedef struct spmx_csr spmx_csr;   /* A resident on the device */
typedef struct spmx_plan spmx_plan; /* partition of A for one (strategy, parts, flags) */

const char* spmx_last_error(void);
int spmx_abi_version(void);
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

/* raw device buffers on the context's device (X, Y and staging) */
int spmx_dev_alloc(spmx_ctx* ctx, size_t bytes, void** out);
int spmx_dev_free(spmx_ctx* ctx, void* ptr);
int spmx_h2d(spmx_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes);  /* async on ctx stream */
int spmx_d2h(spmx_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes);  /* async on ctx stream */
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
 *      dynamic != 0 (row-split only, else SPMX_EINVAL) makes persistent CTAs claim `batch` rows
 *      at a time from a device counter, the analogue of DispatchCounter (partition.hpp:38-40). */
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

/* ---- helpers for the reference's report fields ---------------------------------------------- */
/* checksum(Y), dense.cpp:17-28, of a device buffer (FNV-1a is sequential: the buffer is copied
 * to the host and hashed there; a reporting helper, not on the hot path) */
int spmx_checksum_device(spmx_ctx* ctx, const float* d_y, size_t count, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* SPMX_B200_H */
