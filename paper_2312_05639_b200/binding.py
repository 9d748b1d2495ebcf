"""ctypes binding of libspmx_b200.so (include/spmx_b200.h) for tests/ and bench.py.

Python is plumbing here: device memory comes from torch tensors (or the library's own
allocator), every compute call goes through the C ABI into the hand-written sm_100a
kernels. There is no CPU fallback: if the shared library is missing this module raises
at load time, and without a CUDA device every compute call raises SpmxRuntimeError.
"""
from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess
import sys

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
# SPMX_B200_LIB selects another build of the same library (kernel-tuning experiments only)
LIB_PATH = os.environ.get("SPMX_B200_LIB") or os.path.join(_PKG, "libspmx_b200.so")
ASBUILT_PATH = os.path.splitext(LIB_PATH)[0] + "_asbuilt.so"
CSRC = os.path.join(_PKG, "csrc")
HEADER = os.path.join(_ROOT, "include", "spmx_b200.h")

ROW, NNZ, MERGE = 0, 1, 2
STRATEGY = {"row": ROW, "nnz": NNZ, "merge": MERGE}
EXACT_ORDER = 1
JIT_WIDTH = 4
CLAIM_KERNEL = 8

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


class SpmxInvalidArgument(ValueError):
    """SPMX_EINVAL — where the reference throws std::invalid_argument."""


class SpmxRuntimeError(RuntimeError):
    """SPMX_ERUNTIME — where the reference throws std::runtime_error."""


class SpmxLogicError(RuntimeError):
    """SPMX_ELOGIC — where the reference throws std::logic_error."""


KERNEL_SRC_INC = os.path.join(CSRC, "spmx_kernels_src.inc")


def generate_kernel_source_include() -> None:
    """The kernel header as a C++ raw string literal, compiled into the library so that
    spmx_spmm can instantiate the kernel for any d at run time with NVRTC (the GPU role of the
    reference's emit(), src/jit.cpp:136-154)."""
    src = open(os.path.join(CSRC, "spmx_kernels.cuh")).read()
    assert ')SPMXSRC"' not in src
    text = 'R"SPMXSRC(' + src + ')SPMXSRC"\n'
    if not os.path.exists(KERNEL_SRC_INC) or open(KERNEL_SRC_INC).read() != text:
        with open(KERNEL_SRC_INC, "w") as f:
            f.write(text)


# nvcc releases whose SASS the post-link scheduling edit has been validated on (encoding of the
# control words, the walk loop's shape; tests/test_sass_ab_gpu.py is the bitwise A/B check)
VALIDATED_NVCC = ("12.9",)


def _nvcc_validated(verbose: bool) -> bool:
    """The edit rewrites undocumented scheduling fields: it is applied only under a compiler
    release it was validated with (SPMX_SASS_SCHED_ANY_NVCC=1 overrides; the preconditions and the
    A/B test still guard it). Under any other release the kernels ship as compiled."""
    if os.environ.get("SPMX_SASS_SCHED_ANY_NVCC"):
        return True
    try:
        out = subprocess.run(["nvcc", "--version"], capture_output=True, text=True, check=True).stdout
    except Exception:
        return False
    import re
    m = re.search(r"release (\d+\.\d+)", out)
    ok = bool(m) and m.group(1) in VALIDATED_NVCC
    if not ok and verbose:
        print(f"sass_sched: nvcc release {m.group(1) if m else '?'} is not in {VALIDATED_NVCC}: kernels are "
              "shipped as compiled (SPMX_SASS_SCHED_ANY_NVCC=1 to apply the edit anyway)", file=sys.stderr)
    return ok


def build_library(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/*.cu into libspmx_b200.so for sm_100a (nvcc cross-compiles without a GPU)."""
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".cu")]
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".inc")] + [HEADER]
    if not force and os.path.exists(LIB_PATH):
        if os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(d) for d in deps):
            return LIB_PATH
    generate_kernel_source_include()
    cmd = ["nvcc", *NVCC_FLAGS, "-o", LIB_PATH, *srcs, "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    # the library exactly as nvcc linked it, kept beside the shipped one for the A/B parity test
    # of the post-link step (tests/test_sass_ab_gpu.py); nothing else loads it
    shutil.copyfile(LIB_PATH, ASBUILT_PATH)
    # second scoreboard for half of the walk loop's gathers (sass_sched.py):
    # applied only when its preconditions hold, SPMX_NO_SASS_SCHED=1 leaves the kernels as compiled
    if not os.environ.get("SPMX_NO_SASS_SCHED") and _nvcc_validated(verbose):
        from . import sass_sched
        say = (lambda m: print("sass_sched:", m, file=sys.stderr)) if verbose else (lambda m: None)
        # strict: a precompiled width whose preconditions fail stops the build (a silent
        # fall-back to the compiled schedule would ship a 5-13 % slower kernel unnoticed)
        n = sass_sched.patch_library(LIB_PATH, log=say, strict=True)
        say(f"{n} kernel(s) re-scheduled")
    return LIB_PATH


_u64p = C.POINTER(C.c_uint64)


def _np_u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


class Lib:
    """Loaded libspmx_b200.so with typed signatures."""

    _inst = None

    @classmethod
    def get(cls) -> "Lib":
        if cls._inst is None:
            cls._inst = cls()
        return cls._inst

    def __init__(self, path: str | None = None):
        path = path or LIB_PATH
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` — there is no CPU fallback for this path")
        self.path = path
        L = self.lib = C.CDLL(path)
        vp, i64, u64, sz = C.c_void_p, C.c_int64, C.c_uint64, C.c_size_t
        P = C.POINTER
        L.spmx_last_error.restype = C.c_char_p
        L.spmx_abi_version.restype = C.c_int
        L.spmx_build_info.restype = C.c_char_p
        L.spmx_kernel_launch_count.restype = u64
        L.spmx_ctx_create.argtypes = [C.c_int, vp, P(vp)]
        L.spmx_ctx_destroy.argtypes = [vp]
        L.spmx_ctx_synchronize.argtypes = [vp]
        L.spmx_ctx_sm_count.argtypes = [vp, P(C.c_int)]
        L.spmx_dev_alloc.argtypes = [vp, sz, P(vp)]
        L.spmx_dev_free.argtypes = [vp, vp]
        L.spmx_h2d.argtypes = [vp, vp, vp, sz]
        L.spmx_d2h.argtypes = [vp, vp, vp, sz]
        L.spmx_host_alloc_pinned.argtypes = [sz, P(vp)]
        L.spmx_host_free_pinned.argtypes = [vp]
        L.spmx_csr_upload.argtypes = [vp, i64, i64, i64, vp, vp, vp, P(vp)]
        L.spmx_csr_wrap_device.argtypes = [vp, i64, i64, i64, vp, vp, vp, C.c_int, P(vp)]
        L.spmx_rowptr_upload.argtypes = [vp, i64, i64, vp, P(vp)]
        L.spmx_csr_destroy.argtypes = [vp]
        L.spmx_csr_dims.argtypes = [vp, P(i64), P(i64), P(i64)]
        L.spmx_split_rows_static.argtypes = [vp, u64, C.c_uint, vp]
        L.spmx_split_nnz.argtypes = [vp, vp, C.c_uint, vp]
        L.spmx_split_merge.argtypes = [vp, vp, C.c_uint, vp]
        L.spmx_merge_path_search.argtypes = [vp, vp, sz, vp, vp, vp]
        L.spmx_next_batch_claims.argtypes = [vp, u64, u64, sz, vp]
        L.spmx_plan_create.argtypes = [vp, vp, C.c_int, C.c_uint, C.c_int, u64, C.c_uint, P(vp)]
        L.spmx_plan_destroy.argtypes = [vp]
        L.spmx_plan_info.argtypes = [vp, P(C.c_uint), P(u64), P(C.c_int)]
        L.spmx_plan_ranges.argtypes = [vp, vp]
        L.spmx_plan_chunks.argtypes = [vp, vp, vp]
        L.spmx_spmm.argtypes = [vp, vp, vp, vp, i64, i64, vp, P(C.c_float)]
        L.spmx_spmm_host.argtypes = [vp, i64, i64, i64, vp, vp, vp, vp, i64, i64, vp, C.c_int,
                                     C.c_uint, C.c_int, u64, C.c_uint, P(C.c_double)]
        L.spmx_checksum_device.argtypes = [vp, vp, sz, P(u64)]
        L.spmx_spmm_reference.argtypes = [vp, vp, vp, i64, i64, vp]
        L.spmx_max_relative_error.argtypes = [vp, vp, vp, sz, P(C.c_double)]
        L.spmx_jit_stats.argtypes = [P(u64), P(C.c_double)]
        # multi-GPU driver
        ip, fp = P(C.c_int), P(C.c_float)
        L.spmx_mg_create.argtypes = [C.c_int, ip, C.c_int, P(vp)]
        L.spmx_mg_unique_id.argtypes = [vp]
        L.spmx_mg_create_rank.argtypes = [C.c_int, vp, C.c_int, C.c_int, C.c_int, vp, P(vp)]
        L.spmx_mg_destroy.argtypes = [vp]
        L.spmx_mg_info.argtypes = [vp, ip, ip, ip, ip, ip]
        L.spmx_mg_shard_owner.argtypes = [C.c_int, C.c_int, C.c_int]
        L.spmx_mg_shard_host.argtypes = [vp, i64, i64, i64, vp, vp, vp, C.c_int, vp]
        L.spmx_mg_shard_device.argtypes = [vp, C.c_int, i64, i64, i64, vp, vp, vp, C.c_int, vp]
        L.spmx_mg_shard_info.argtypes = [vp, C.c_int, ip, ip, P(u64), P(u64), P(u64)]
        L.spmx_mg_plan.argtypes = [vp, C.c_int, C.c_uint, C.c_int, u64, C.c_uint]
        L.spmx_mg_broadcast_x_host.argtypes = [vp, vp, C.c_int, i64, i64, fp, fp]
        L.spmx_mg_broadcast_x_device.argtypes = [vp, P(vp), C.c_int, i64, i64, fp]
        L.spmx_mg_broadcast_x_from_device.argtypes = [vp, vp, C.c_int, i64, i64, fp, fp]
        L.spmx_mg_spmm.argtypes = [vp, C.c_int, fp, fp]
        L.spmx_mg_y_shard.argtypes = [vp, C.c_int, P(vp)]
        L.spmx_mg_download_y.argtypes = [vp, vp]
        L.spmx_mg_download_y_shards.argtypes = [vp, P(vp)]
        L.spmx_ctx_l2_window.argtypes = [vp, vp, sz, C.c_float, P(sz)]
        L.spmx_probe_l2_to_sm.argtypes = [vp, C.c_int, P(C.c_double), P(C.c_double)]
        L.spmx_mg_allgather_y.argtypes = [vp, fp]
        L.spmx_mg_y_full.argtypes = [vp, C.c_int, P(vp)]
        L.spmx_mg_allreduce.argtypes = [vp, P(C.c_double), C.c_int, C.c_int]
        L.spmx_mg_synchronize.argtypes = [vp]

    def check(self, rc: int):
        if rc == 0:
            return
        msg = self.lib.spmx_last_error().decode(errors="replace")
        raise {1: SpmxInvalidArgument, 2: SpmxRuntimeError, 3: SpmxLogicError}.get(
            rc, SpmxRuntimeError)(msg)

    def jit_stats(self):
        """(number of per-d kernels compiled at run time, total seconds spent compiling)."""
        n, t = C.c_uint64(), C.c_double()
        self.lib.spmx_jit_stats(C.byref(n), C.byref(t))
        return n.value, t.value

    def build_info(self) -> dict:
        """{'SPMX_SASS_SCHED': '6', 'cuda': '12090', ...} of the loaded library."""
        txt = self.lib.spmx_build_info().decode()
        return dict(kv.split("=", 1) for kv in txt.split(";") if "=" in kv)

    def launch_count(self) -> int:
        return int(self.lib.spmx_kernel_launch_count())


def _ptr(a) -> int:
    """Address of a numpy array / torch tensor / raw int."""
    if a is None:
        return 0
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


class Context:
    """spmx_ctx: one (device, stream). stream=None creates a private stream; pass a torch
    stream's .cuda_stream to run on it."""

    def __init__(self, device: int = 0, stream: int | None = None, lib: "Lib | None" = None):
        self.L = lib or Lib.get()
        h = C.c_void_p()
        self.L.check(self.L.lib.spmx_ctx_create(device, C.c_void_p(stream or 0), C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def on_torch_stream(cls, device: int = 0) -> "Context":
        """A context whose kernels run on torch's CURRENT stream, made explicit first: the
        legacy default stream has handle 0, which the C ABI reads as "create a private
        (non-blocking) stream" — torch work issued before a library call (fills, slices,
        generators) would then not be ordered with it."""
        import torch
        stream = torch.cuda.Stream(device=device)
        torch.cuda.set_stream(stream)
        c = cls(device, stream.cuda_stream)
        c._torch_stream = stream
        return c

    def close(self):
        if self.h:
            self.L.check(self.L.lib.spmx_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        self.L.check(self.L.lib.spmx_ctx_synchronize(self.h))

    def sm_count(self) -> int:
        v = C.c_int()
        self.L.check(self.L.lib.spmx_ctx_sm_count(self.h, C.byref(v)))
        return v.value

    # -- CSR ---------------------------------------------------------------------------
    def csr_upload(self, m, n, row_ptr, col, vals) -> "DeviceCsr":
        rp = _np_u64(row_ptr)
        nnz = int(rp[m]) if rp.size > m else -1
        col = np.ascontiguousarray(col, dtype=np.uint32)
        vals = np.ascontiguousarray(vals, dtype=np.float32)
        h = C.c_void_p()
        self.L.check(self.L.lib.spmx_csr_upload(self.h, m, n, nnz, _ptr(rp), _ptr(col) if col.size else 0,
                                                _ptr(vals) if vals.size else 0, C.byref(h)))
        return DeviceCsr(self, h, m, n, nnz)

    def csr_upload_raw(self, m, n, nnz, row_ptr, col, vals) -> "DeviceCsr":
        """No consistency pre-checks on the host: lets tests feed invalid CSRs."""
        rp = _np_u64(row_ptr)
        col = np.ascontiguousarray(col, dtype=np.uint32)
        vals = np.ascontiguousarray(vals, dtype=np.float32)
        h = C.c_void_p()
        self.L.check(self.L.lib.spmx_csr_upload(self.h, m, n, nnz, _ptr(rp), _ptr(col) if col.size else 0,
                                                _ptr(vals) if vals.size else 0, C.byref(h)))
        return DeviceCsr(self, h, m, n, nnz)

    def rowptr_upload(self, m, row_ptr, nnz=None) -> "DeviceCsr":
        """Structure-only handle (partitioner and plan input)."""
        rp = _np_u64(row_ptr)
        if nnz is None:
            nnz = int(rp[m]) if rp.size > m else -1
        h = C.c_void_p()
        self.L.check(self.L.lib.spmx_rowptr_upload(self.h, m, nnz, _ptr(rp), C.byref(h)))
        return DeviceCsr(self, h, m, 0, nnz)

    def csr_wrap(self, csr, validate=True) -> "DeviceCsr":
        """Borrow a workloads.Csr whose tensors already live on this device."""
        h = C.c_void_p()
        self.L.check(self.L.lib.spmx_csr_wrap_device(self.h, csr.m, csr.n, csr.nnz,
                                                     _ptr(csr.row_ptr), _ptr(csr.col),
                                                     _ptr(csr.vals), int(validate), C.byref(h)))
        d = DeviceCsr(self, h, csr.m, csr.n, csr.nnz)
        d._keep = csr
        return d

    # -- partitioner -------------------------------------------------------------------
    def split_rows_static(self, m, parts):
        out = np.zeros(2 * max(parts, 1), np.uint64)
        self.L.check(self.L.lib.spmx_split_rows_static(self.h, m, parts, _ptr(out)))
        return out.reshape(-1, 2)

    def split_nnz(self, a: "DeviceCsr", parts):
        out = np.zeros(2 * max(parts, 1), np.uint64)
        self.L.check(self.L.lib.spmx_split_nnz(self.h, a.h, parts, _ptr(out)))
        return out.reshape(-1, 2)

    def split_merge(self, a: "DeviceCsr", parts):
        out = np.zeros(2 * max(parts, 1), np.uint64)
        self.L.check(self.L.lib.spmx_split_merge(self.h, a.h, parts, _ptr(out)))
        return out.reshape(-1, 2)

    def merge_path_search(self, a: "DeviceCsr", ks):
        ks = _np_u64(np.atleast_1d(ks))
        oi, oj = np.zeros_like(ks), np.zeros_like(ks)
        self.L.check(self.L.lib.spmx_merge_path_search(self.h, a.h, ks.size, _ptr(ks), _ptr(oi),
                                                       _ptr(oj)))
        return oi, oj

    def next_batch_claims(self, m, batch, n_claims):
        out = np.zeros(2 * max(n_claims, 1), np.uint64)
        self.L.check(self.L.lib.spmx_next_batch_claims(self.h, m, batch, n_claims, _ptr(out)))
        return out.reshape(-1, 2)[:n_claims]

    # -- plan / spmm -------------------------------------------------------------------
    def plan(self, a: "DeviceCsr", strategy="row", parts=0, dynamic=False, batch=128,
             flags=0) -> "Plan":
        h = C.c_void_p()
        s = STRATEGY[strategy] if isinstance(strategy, str) else strategy
        self.L.check(self.L.lib.spmx_plan_create(self.h, a.h, s, parts, int(dynamic), batch, flags,
                                                 C.byref(h)))
        return Plan(self, a, h)

    def spmm(self, plan: "Plan", a: "DeviceCsr", x, y, timed=False):
        """x: N x d, y: M x d float32 tensors on this device. Returns device ms when timed."""
        ms = C.c_float(0.0)
        x_rows, d = x.shape
        self.L.check(self.L.lib.spmx_spmm(self.h, plan.h, a.h, _ptr(x), x_rows, d, _ptr(y),
                                          C.byref(ms) if timed else None))
        return ms.value if timed else None

    def spmm_raw(self, plan, a, x_ptr, x_rows, d, y_ptr):
        self.L.check(self.L.lib.spmx_spmm(self.h, plan.h, a.h, x_ptr, x_rows, d, y_ptr, None))

    def spmm_host(self, m, n, row_ptr, col, vals, x, y=None, strategy="row", parts=0,
                  dynamic=False, batch=128, flags=0, nnz=None):
        """run_spmm with host (numpy) buffers. Returns (y, times_ms dict)."""
        rp = _np_u64(row_ptr)
        if nnz is None:
            nnz = int(rp[m])
        col = np.ascontiguousarray(col, dtype=np.uint32)
        vals = np.ascontiguousarray(vals, dtype=np.float32)
        x = np.ascontiguousarray(x, dtype=np.float32)
        x_rows, d = x.shape
        if y is None:
            y = np.empty((m, d), np.float32)
        t = (C.c_double * 6)()
        s = STRATEGY[strategy] if isinstance(strategy, str) else strategy
        self.L.check(self.L.lib.spmx_spmm_host(self.h, m, n, nnz, _ptr(rp), _ptr(col) if col.size else 0,
                                               _ptr(vals) if vals.size else 0, _ptr(x), x_rows, d,
                                               _ptr(y), s, parts, int(dynamic), batch, flags, t))
        return y, dict(plan=t[0], x_wait=t[2], stream_blocks=t[3], total=t[4], blocks=t[5])

    def spmm_reference(self, a: "DeviceCsr", x, y):
        """spmm_reference (unfused Alg. 1) on the device, for verification."""
        self.L.check(self.L.lib.spmx_spmm_reference(self.h, a.h, _ptr(x), x.shape[0], x.shape[1],
                                                    _ptr(y)))

    def max_relative_error(self, y, ref) -> float:
        out = C.c_double()
        self.L.check(self.L.lib.spmx_max_relative_error(self.h, _ptr(y), _ptr(ref), y.numel(),
                                                        C.byref(out)))
        return out.value

    def l2_window(self, ptr=0, nbytes=0, hit_ratio=1.0) -> int:
        """Persisting access-policy window on the context's stream (nbytes=0 clears it).
        Returns the window size actually set."""
        out = C.c_size_t()
        self.L.check(self.L.lib.spmx_ctx_l2_window(self.h, C.c_void_p(ptr or None), nbytes, hit_ratio,
                                                   C.byref(out)))
        return out.value

    def probe_l2_to_sm(self, repeats=10):
        """(TB/s, ms): the L2 -> SM ceiling measured now, on this GPU (spmx_probe_l2_to_sm)."""
        tbs, ms = C.c_double(), C.c_double()
        self.L.check(self.L.lib.spmx_probe_l2_to_sm(self.h, repeats, C.byref(tbs), C.byref(ms)))
        return tbs.value, ms.value

    def checksum(self, y) -> int:
        out = C.c_uint64()
        self.L.check(self.L.lib.spmx_checksum_device(self.h, _ptr(y), y.numel(), C.byref(out)))
        return out.value


class DeviceCsr:
    def __init__(self, ctx: Context, h, m, n, nnz):
        self.ctx, self.h, self.m, self.n, self.nnz = ctx, h, m, n, nnz

    def close(self):
        if self.h:
            self.ctx.L.check(self.ctx.L.lib.spmx_csr_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            if self.ctx.h:
                self.close()
        except Exception:
            pass


class Plan:
    def __init__(self, ctx: Context, a: DeviceCsr, h):
        self.ctx, self.a, self.h = ctx, a, h
        p, c, dyn = C.c_uint(), C.c_uint64(), C.c_int()
        ctx.L.check(ctx.L.lib.spmx_plan_info(h, C.byref(p), C.byref(c), C.byref(dyn)))
        self.parts, self.n_chunks, self.dynamic = p.value, c.value, bool(dyn.value)

    def ranges(self):
        if self.dynamic:
            return np.zeros((0, 2), np.uint64)
        out = np.zeros(2 * self.parts, np.uint64)
        self.ctx.L.check(self.ctx.L.lib.spmx_plan_ranges(self.h, _ptr(out)))
        return out.reshape(-1, 2)

    def chunks(self):
        r = np.zeros(self.n_chunks + 1, np.uint64)
        j = np.zeros(self.n_chunks + 1, np.uint64)
        self.ctx.L.check(self.ctx.L.lib.spmx_plan_chunks(self.h, _ptr(r), _ptr(j)))
        return r, j

    def close(self):
        if self.h:
            self.ctx.L.check(self.ctx.L.lib.spmx_plan_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            if self.ctx.h:
                self.close()
        except Exception:
            pass


SHARD_BY = {"nnz": 1, "merge": 2}


class MultiGpu:
    """spmx_mg: the library's multi-GPU driver (row-block shards from split_nnz(A, G) /
    split_merge(A, G), one NCCL broadcast of X, Y row-sharded, optional all-gather-v).

    MultiGpu(devices=[0, 1, ...])              one process drives all GPUs (ncclCommInitAll)
    MultiGpu.for_rank(device, rank, world, id) one process per GPU (torchrun); id from unique_id()
    n_shards > world places several row blocks on a GPU (tests: one GPU stands in for a node)."""

    def __init__(self, devices=(0,), n_shards=0, lib: "Lib | None" = None, _handle=None):
        self.L = lib or Lib.get()
        if _handle is not None:
            self.h = _handle
        else:
            devs = (C.c_int * len(devices))(*devices)
            h = C.c_void_p()
            self.L.check(self.L.lib.spmx_mg_create(len(devices), devs, n_shards, C.byref(h)))
            self.h = h
        self._keep = []

    @staticmethod
    def unique_id(lib: "Lib | None" = None) -> bytes:
        L = lib or Lib.get()
        buf = C.create_string_buffer(128)
        L.check(L.lib.spmx_mg_unique_id(buf))
        return buf.raw

    @classmethod
    def for_rank(cls, device, rank, world, uid: "bytes | None", n_shards=0, stream=None,
                 lib: "Lib | None" = None) -> "MultiGpu":
        L = lib or Lib.get()
        h = C.c_void_p()
        idbuf = C.create_string_buffer(uid, 128) if uid is not None else None
        L.check(L.lib.spmx_mg_create_rank(device, C.c_void_p(stream or 0), rank, world, n_shards,
                                          idbuf, C.byref(h)))
        return cls(lib=L, _handle=h)

    def close(self):
        if self.h:
            self.L.check(self.L.lib.spmx_mg_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        v = [C.c_int() for _ in range(5)]
        self.L.check(self.L.lib.spmx_mg_info(self.h, *[C.byref(x) for x in v]))
        return dict(zip(("world", "local_ranks", "shards", "local_shards", "nccl_version"),
                        (x.value for x in v)))

    def shard_owner(self, shard) -> int:
        i = self.info()
        return self.L.lib.spmx_mg_shard_owner(i["shards"], i["world"], shard)

    def shard_host(self, m, n, row_ptr, col, vals, by="nnz"):
        rp = _np_u64(row_ptr)
        nnz = int(rp[m])
        col = np.ascontiguousarray(col, dtype=np.uint32)
        vals = np.ascontiguousarray(vals, dtype=np.float32)
        out = np.zeros(2 * self.info()["shards"], np.uint64)
        self.L.check(self.L.lib.spmx_mg_shard_host(self.h, m, n, nnz, _ptr(rp), _ptr(col) if col.size else 0,
                                                   _ptr(vals) if vals.size else 0, SHARD_BY[by], _ptr(out)))
        return out.reshape(-1, 2)

    def shard_device(self, csr, by="nnz", src_local_rank=0):
        """csr: workloads.Csr whose tensors live on local rank src_local_rank's GPU."""
        out = np.zeros(2 * self.info()["shards"], np.uint64)
        self.L.check(self.L.lib.spmx_mg_shard_device(self.h, src_local_rank, csr.m, csr.n, csr.nnz,
                                                     _ptr(csr.row_ptr), _ptr(csr.col), _ptr(csr.vals),
                                                     SHARD_BY[by], _ptr(out)))
        return out.reshape(-1, 2)

    def shard_info(self, local_shard) -> dict:
        g, dev = C.c_int(), C.c_int()
        b, e, z = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.L.check(self.L.lib.spmx_mg_shard_info(self.h, local_shard, C.byref(g), C.byref(dev),
                                                   C.byref(b), C.byref(e), C.byref(z)))
        return dict(shard=g.value, device=dev.value, row_begin=b.value, row_end=e.value, nnz=z.value)

    def local_shards(self):
        return [self.shard_info(i) for i in range(self.info()["local_shards"])]

    def plan(self, strategy="merge", parts=0, dynamic=False, batch=128, flags=0):
        s = STRATEGY[strategy] if isinstance(strategy, str) else strategy
        self.L.check(self.L.lib.spmx_mg_plan(self.h, s, parts, int(dynamic), batch, flags))

    def broadcast_x_host(self, x, root=0):
        """x: numpy N x d on the process that drives `root` (None elsewhere). Returns (h2d_ms, bcast_ms)."""
        h2d, bc = C.c_float(), C.c_float()
        if x is not None:
            x = np.ascontiguousarray(x, dtype=np.float32)
            self._shape = x.shape
        rows, d = self._shape
        self.L.check(self.L.lib.spmx_mg_broadcast_x_host(self.h, _ptr(x) if x is not None else 0, root,
                                                         rows, d, C.byref(h2d), C.byref(bc)))
        return h2d.value, bc.value

    def set_x_shape(self, rows, d):
        self._shape = (rows, d)

    def broadcast_x_device(self, xs, root=0):
        """xs: one N x d float32 tensor per local rank, on that rank's GPU (the root's holds X)."""
        rows, d = xs[0].shape
        arr = (C.c_void_p * len(xs))(*[_ptr(x) for x in xs])
        bc = C.c_float()
        self.L.check(self.L.lib.spmx_mg_broadcast_x_device(self.h, arr, root, rows, d, C.byref(bc)))
        self._keep = list(xs)
        self._shape = (rows, d)
        return bc.value

    def broadcast_x_from_device(self, x, root=0, shape=None):
        """x: the root's N x d tensor on the root's GPU (None on processes that do not drive the
        root; pass shape=(N, d) there). The driver owns the replicas. Returns (copy_ms, bcast_ms)."""
        cp, bc = C.c_float(), C.c_float()
        if x is not None:
            self._shape = tuple(x.shape)
            self._keep = [x]
        elif shape is not None:
            self._shape = tuple(shape)
        rows, d = self._shape
        self.L.check(self.L.lib.spmx_mg_broadcast_x_from_device(self.h, _ptr(x) if x is not None else 0, root,
                                                                rows, d, C.byref(cp), C.byref(bc)))
        return cp.value, bc.value

    def spmm(self, steps=1, per_shard=False):
        ms = C.c_float()
        n = self.info()["local_shards"]
        per = (C.c_float * max(n, 1))()
        self.L.check(self.L.lib.spmx_mg_spmm(self.h, steps, C.byref(ms), per if per_shard else None))
        return (ms.value, list(per)[:n]) if per_shard else ms.value

    def download_y(self, y=None, m=None):
        rows, d = self._shape
        if y is None:
            y = np.zeros((m, d), np.float32)
        self.L.check(self.L.lib.spmx_mg_download_y(self.h, _ptr(y)))
        return y

    def download_y_shards(self, blocks):
        """blocks: one host array / tensor (rows_i x d float32) per local shard."""
        arr = (C.c_void_p * max(len(blocks), 1))(*[_ptr(b) for b in blocks])
        self.L.check(self.L.lib.spmx_mg_download_y_shards(self.h, arr))

    def y_shard_ptr(self, local_shard) -> int:
        p = C.c_void_p()
        self.L.check(self.L.lib.spmx_mg_y_shard(self.h, local_shard, C.byref(p)))
        return p.value or 0

    def allgather_y(self) -> float:
        ms = C.c_float()
        self.L.check(self.L.lib.spmx_mg_allgather_y(self.h, C.byref(ms)))
        return ms.value

    def y_full_ptr(self, local_rank=0) -> int:
        p = C.c_void_p()
        self.L.check(self.L.lib.spmx_mg_y_full(self.h, local_rank, C.byref(p)))
        return p.value or 0

    def allreduce(self, values, op="sum"):
        vals = [float(v) for v in np.atleast_1d(values)]
        arr = (C.c_double * len(vals))(*vals)
        self.L.check(self.L.lib.spmx_mg_allreduce(self.h, arr, len(vals), {"sum": 0, "max": 1}[op]))
        return list(arr)

    def synchronize(self):
        self.L.check(self.L.lib.spmx_mg_synchronize(self.h))
