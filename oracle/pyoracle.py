"""ctypes bindings for the test-only oracle libraries.

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs. The product package
(paper_2312_05639_b200) never imports this module.

  Oracle  -> oracle/liboracle.so        (our C restatement, spmx_oracle.c)
  RefLib  -> oracle/_ref/libspmx_ref.so (the unmodified reference + ref_shim.cpp;
                                         present only where it was built)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libspmx_ref.so")

STRATEGY = {"row": 0, "nnz": 1, "merge": 2}

_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> None:
    """Compile liboracle.so (always possible) and _ref (when /root/reference exists)."""
    if force or not os.path.exists(ORACLE_SO) or (
        os.path.getmtime(ORACLE_SO) < os.path.getmtime(os.path.join(_HERE, "spmx_oracle.c"))
    ):
        subprocess.check_call(["make", "-C", _HERE, "liboracle.so"], stdout=subprocess.DEVNULL)
    if os.path.isdir("/root/reference/proj/src") and (force or not os.path.exists(REF_SO)):
        subprocess.check_call(["make", "-C", _HERE, "ref"], stdout=subprocess.DEVNULL)


def _as(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class OracleInvalidArgument(ValueError):
    """Raised where the reference throws std::invalid_argument."""


class Oracle:
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        L = self.lib = C.CDLL(ORACLE_SO)
        i64, u64, f64 = C.c_int64, C.c_uint64, C.c_double
        L.oracle_spmm_unfused.argtypes = [i64, i64, _u64p, _u32p, _f32p, _f32p, i64, i64, _f32p]
        L.oracle_spmm_fused.argtypes = [i64, i64, _u64p, _u32p, _f32p, _f32p, i64, i64, _f32p,
                                        C.c_int, C.POINTER(C.c_int)]
        L.oracle_spmm_fused_range.argtypes = [i64, i64, _u64p, _u32p, _f32p, _f32p, i64, i64,
                                              _f32p, u64, u64]
        L.oracle_abs_bound.argtypes = [i64, _u64p, _u32p, _f32p, _f32p, i64, _f64p]
        L.oracle_max_relative_error.argtypes = [_f32p, _f32p, C.c_size_t]
        L.oracle_max_relative_error.restype = f64
        L.oracle_checksum.argtypes = [_f32p, C.c_size_t]
        L.oracle_checksum.restype = u64
        L.oracle_split_rows_static.argtypes = [u64, C.c_uint, _u64p]
        L.oracle_split_nnz.argtypes = [u64, u64, _u64p, C.c_uint, _u64p]
        L.oracle_split_merge.argtypes = [u64, u64, _u64p, C.c_uint, _u64p]
        L.oracle_merge_path_search.argtypes = [u64, _u64p, u64, u64, C.POINTER(u64), C.POINTER(u64)]
        L.oracle_merge_walk.argtypes = [u64, _u64p, u64, u64, C.POINTER(u64), C.POINTER(u64)]
        L.oracle_merge_walk.restype = None
        L.oracle_next_batch.argtypes = [C.POINTER(u64), u64, u64, C.POINTER(u64), C.POINTER(u64)]
        L.oracle_validate_csr.argtypes = [i64, i64, i64, _u64p, _u32p]
        L.oracle_num_threads.restype = C.c_int

    @staticmethod
    def _chk(rc):
        if rc != 0:
            raise OracleInvalidArgument("oracle: invalid argument")

    # -- SpMM --
    def spmm_unfused(self, m, n, row_ptr, col, vals, x):
        x = _as(x, np.float32)
        d = x.shape[1]
        y = np.zeros((m, d), np.float32)
        self._chk(self.lib.oracle_spmm_unfused(m, n, _as(row_ptr, np.uint64), _as(col, np.uint32),
                                               _as(vals, np.float32), x, x.shape[0], d, y))
        return y

    def spmm_fused(self, m, n, row_ptr, col, vals, x, threads=0):
        x = _as(x, np.float32)
        d = x.shape[1]
        y = np.zeros((m, d), np.float32)
        used = C.c_int(0)
        self._chk(self.lib.oracle_spmm_fused(m, n, _as(row_ptr, np.uint64), _as(col, np.uint32),
                                             _as(vals, np.float32), x, x.shape[0], d, y,
                                             threads, C.byref(used)))
        self.last_threads = used.value
        return y

    def spmm_fused_range(self, m, n, row_ptr, col, vals, x, y, row_begin, row_end):
        x = _as(x, np.float32)
        self._chk(self.lib.oracle_spmm_fused_range(m, n, _as(row_ptr, np.uint64),
                                                   _as(col, np.uint32), _as(vals, np.float32), x,
                                                   x.shape[0], x.shape[1], y, row_begin, row_end))
        return y

    def abs_bound(self, m, row_ptr, col, vals, x):
        x = _as(x, np.float32)
        s = np.zeros((m, x.shape[1]), np.float64)
        self.lib.oracle_abs_bound(m, _as(row_ptr, np.uint64), _as(col, np.uint32),
                                  _as(vals, np.float32), x, x.shape[1], s)
        return s

    # -- metrics --
    def max_relative_error(self, y, ref):
        y, ref = _as(y, np.float32).ravel(), _as(ref, np.float32).ravel()
        return float(self.lib.oracle_max_relative_error(y, ref, y.size))

    def checksum(self, y):
        y = _as(y, np.float32).ravel()
        return int(self.lib.oracle_checksum(y, y.size))

    # -- partitioner --
    def split_rows_static(self, m, parts):
        out = np.zeros(2 * max(parts, 1), np.uint64)
        self._chk(self.lib.oracle_split_rows_static(m, parts, out))
        return out.reshape(-1, 2)

    def split_nnz(self, row_ptr, parts):
        row_ptr = _as(row_ptr, np.uint64)
        m = row_ptr.size - 1
        out = np.zeros(2 * max(parts, 1), np.uint64)
        self._chk(self.lib.oracle_split_nnz(m, int(row_ptr[m]), row_ptr, parts, out))
        return out.reshape(-1, 2)

    def split_merge(self, row_ptr, parts):
        row_ptr = _as(row_ptr, np.uint64)
        m = row_ptr.size - 1
        out = np.zeros(2 * max(parts, 1), np.uint64)
        self._chk(self.lib.oracle_split_merge(m, int(row_ptr[m]), row_ptr, parts, out))
        return out.reshape(-1, 2)

    def merge_path_search(self, row_ptr, k):
        row_ptr = _as(row_ptr, np.uint64)
        m = row_ptr.size - 1
        i, j = C.c_uint64(), C.c_uint64()
        self._chk(self.lib.oracle_merge_path_search(k, row_ptr[1:].copy() if m else
                                                    np.zeros(1, np.uint64), m, int(row_ptr[m]),
                                                    C.byref(i), C.byref(j)))
        return i.value, j.value

    def merge_walk(self, row_ptr, k):
        row_ptr = _as(row_ptr, np.uint64)
        m = row_ptr.size - 1
        i, j = C.c_uint64(), C.c_uint64()
        self.lib.oracle_merge_walk(k, row_ptr[1:].copy() if m else np.zeros(1, np.uint64), m,
                                   int(row_ptr[m]), C.byref(i), C.byref(j))
        return i.value, j.value

    def next_batch(self, counter, batch, m):
        """counter: one-element list holding the shared counter value."""
        c = C.c_uint64(counter[0])
        b, e = C.c_uint64(), C.c_uint64()
        ok = self.lib.oracle_next_batch(C.byref(c), batch, m, C.byref(b), C.byref(e))
        counter[0] = c.value
        return (b.value, e.value) if ok else None

    def validate_csr(self, m, n, nnz, row_ptr, col):
        return int(self.lib.oracle_validate_csr(m, n, nnz, _as(row_ptr, np.uint64),
                                                _as(col, np.uint32)))

    def num_threads(self):
        return int(self.lib.oracle_num_threads())


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code  # 1 invalid_argument, 2 runtime_error, 3 logic_error


class RefCsr:
    """A CsrMatrix living inside the reference library."""

    def __init__(self, ref: "RefLib", handle):
        self.ref, self.h = ref, handle
        m, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        ref.lib.ref_csr_dims(handle, C.byref(m), C.byref(n), C.byref(nnz))
        self.m, self.n, self.nnz = m.value, n.value, nnz.value

    def arrays(self):
        rp = np.zeros(self.m + 1, np.uint64)
        col = np.zeros(max(self.nnz, 1), np.uint32)
        vals = np.zeros(max(self.nnz, 1), np.float32)
        self.ref.lib.ref_csr_copy(self.h, rp, col, vals)
        return rp, col[: self.nnz].copy(), vals[: self.nnz].copy()

    def __del__(self):
        try:
            self.ref.lib.ref_csr_destroy(self.h)
        except Exception:
            pass


class RefLib:
    """The unmodified reference library behind ref_shim.cpp."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference; run oracle/Makefile)")
        L = self.lib = C.CDLL(REF_SO)
        i64, u64, vp = C.c_int64, C.c_uint64, C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_csr_create.argtypes = [i64, i64, i64, _u64p, _u32p, _f32p]
        L.ref_csr_create.restype = vp
        L.ref_csr_destroy.argtypes = [vp]
        L.ref_csr_destroy.restype = None
        L.ref_run_spmm.argtypes = [vp, _f32p, i64, i64, _f32p, C.c_int, C.c_int, C.c_uint, C.c_int,
                                   u64, C.c_uint, _f64p, C.POINTER(C.c_double),
                                   C.POINTER(C.c_uint), C.POINTER(C.c_double)]
        L.ref_spmm_reference.argtypes = [vp, _f32p, i64, i64, _f32p]
        L.ref_validate_csr_count.argtypes = [vp]
        L.ref_split_rows_static.argtypes = [u64, C.c_uint, _u64p]
        L.ref_split_nnz.argtypes = [vp, C.c_uint, _u64p]
        L.ref_split_merge.argtypes = [vp, C.c_uint, _u64p]
        L.ref_merge_path_search.argtypes = [vp, u64, C.POINTER(u64), C.POINTER(u64)]
        L.ref_merge_walk.argtypes = [vp, u64, C.POINTER(u64), C.POINTER(u64)]
        L.ref_make_partition.argtypes = [vp, C.c_int, C.c_uint, C.c_int, u64, _u64p,
                                         C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_checksum.argtypes = [_f32p, i64, i64]
        L.ref_checksum.restype = u64
        L.ref_max_relative_error.argtypes = [_f32p, _f32p, i64]
        L.ref_max_relative_error.restype = C.c_double
        L.ref_rng_create.argtypes = [u64]
        L.ref_rng_create.restype = vp
        L.ref_rng_destroy.argtypes = [vp]
        L.ref_rng_destroy.restype = None
        L.ref_rng_next.argtypes = [vp]
        L.ref_rng_next.restype = u64
        L.ref_random_csr_rect.argtypes = [vp, i64, i64, C.c_double]
        L.ref_random_csr_rect.restype = vp
        L.ref_random_csr.argtypes = [i64, C.c_double, C.c_double, u64]
        L.ref_random_csr.restype = vp
        L.ref_csr_dims.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
        L.ref_csr_dims.restype = None
        L.ref_csr_copy.argtypes = [vp, _u64p, _u32p, _f32p]
        L.ref_csr_copy.restype = None
        L.ref_random_dense.argtypes = [i64, i64, u64, _f32p]
        L.ref_save_csr_cache.argtypes = [vp, C.c_char_p]
        L.ref_load_csr_cache.argtypes = [C.c_char_p]
        L.ref_load_csr_cache.restype = vp
        L.ref_load_matrix_market.argtypes = [C.c_char_p]
        L.ref_load_matrix_market.restype = vp
        L.ref_write_matrix_market.argtypes = [vp, C.c_char_p]

    def _chk(self, rc):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode())

    def csr(self, m, n, row_ptr, col, vals) -> RefCsr:
        row_ptr = _as(row_ptr, np.uint64)
        nnz = int(row_ptr[m])
        col = _as(col, np.uint32) if nnz else np.zeros(1, np.uint32)
        vals = _as(vals, np.float32) if nnz else np.zeros(1, np.float32)
        return RefCsr(self, self.lib.ref_csr_create(m, n, nnz, row_ptr, col, vals))

    def run_spmm(self, a: RefCsr, x, strategy="row", dynamic=False, threads=0, backend="native",
                 batch=128, trials=1, want_y=True):
        x = _as(x, np.float32)
        d = x.shape[1]
        y = np.zeros((a.m, d), np.float32)
        times = np.zeros(max(trials, 1), np.float64)
        cg, thr, gf = C.c_double(), C.c_uint(), C.c_double()
        self._chk(self.lib.ref_run_spmm(a.h, x, x.shape[0], d, y, STRATEGY[strategy], int(dynamic),
                                        threads, 0 if backend == "native" else 1, batch, trials,
                                        times, C.byref(cg), C.byref(thr), C.byref(gf)))
        return y, {"times_s": times[:trials].tolist(), "codegen_s": cg.value,
                   "threads": thr.value, "gflops": gf.value}

    def spmm_reference(self, a: RefCsr, x):
        x = _as(x, np.float32)
        y = np.zeros((a.m, x.shape[1]), np.float32)
        self._chk(self.lib.ref_spmm_reference(a.h, x, x.shape[0], x.shape[1], y))
        return y

    def split_rows_static(self, m, parts):
        out = np.zeros(2 * max(parts, 1), np.uint64)
        self._chk(self.lib.ref_split_rows_static(m, parts, out))
        return out.reshape(-1, 2)

    def split_nnz(self, a: RefCsr, parts):
        out = np.zeros(2 * max(parts, 1), np.uint64)
        self._chk(self.lib.ref_split_nnz(a.h, parts, out))
        return out.reshape(-1, 2)

    def split_merge(self, a: RefCsr, parts):
        out = np.zeros(2 * max(parts, 1), np.uint64)
        self._chk(self.lib.ref_split_merge(a.h, parts, out))
        return out.reshape(-1, 2)

    def merge_path_search(self, a: RefCsr, k):
        i, j = C.c_uint64(), C.c_uint64()
        self._chk(self.lib.ref_merge_path_search(a.h, k, C.byref(i), C.byref(j)))
        return i.value, j.value

    def merge_walk(self, a: RefCsr, k):
        i, j = C.c_uint64(), C.c_uint64()
        self._chk(self.lib.ref_merge_walk(a.h, k, C.byref(i), C.byref(j)))
        return i.value, j.value

    def make_partition(self, a: RefCsr, strategy, parts, dynamic, batch):
        out = np.zeros(2 * max(parts, 1), np.uint64)
        n, dyn = C.c_int(), C.c_int()
        self._chk(self.lib.ref_make_partition(a.h, STRATEGY[strategy], parts, int(dynamic), batch,
                                              out, C.byref(n), C.byref(dyn)))
        return out.reshape(-1, 2)[: n.value], bool(dyn.value)

    def checksum(self, y):
        y = _as(y, np.float32)
        return int(self.lib.ref_checksum(y.ravel(), y.size, 1))

    def max_relative_error(self, y, ref):
        y, ref = _as(y, np.float32).ravel(), _as(ref, np.float32).ravel()
        return float(self.lib.ref_max_relative_error(y, ref, y.size))

    # the reference's own generators
    def rng(self, seed):
        return _RefRng(self, seed)

    def random_csr_rect(self, rng, m, n, density) -> RefCsr:
        return RefCsr(self, self.lib.ref_random_csr_rect(rng.h, m, n, density))

    def random_csr(self, rows, avg, skew, seed) -> RefCsr:
        return RefCsr(self, self.lib.ref_random_csr(rows, avg, skew, seed))

    def save_csr_cache(self, a: RefCsr, path):
        self._chk(self.lib.ref_save_csr_cache(a.h, path.encode()))

    def load_csr_cache(self, path) -> RefCsr:
        h = self.lib.ref_load_csr_cache(path.encode())
        if not h:
            raise RefError(2, self.lib.ref_last_error().decode())
        return RefCsr(self, h)

    def load_matrix_market(self, path) -> RefCsr:
        h = self.lib.ref_load_matrix_market(path.encode())
        if not h:
            raise RefError(2, self.lib.ref_last_error().decode())
        return RefCsr(self, h)

    def write_matrix_market(self, a: RefCsr, path):
        self._chk(self.lib.ref_write_matrix_market(a.h, path.encode()))

    def random_dense(self, rows, cols, seed):
        out = np.zeros((rows, cols), np.float32)
        self._chk(self.lib.ref_random_dense(rows, cols, seed, out))
        return out


class _RefRng:
    def __init__(self, ref, seed):
        self.ref = ref
        self.h = ref.lib.ref_rng_create(seed)

    def __call__(self):
        return int(self.ref.lib.ref_rng_next(self.h))

    def __del__(self):
        try:
            self.ref.lib.ref_rng_destroy(self.h)
        except Exception:
            pass
