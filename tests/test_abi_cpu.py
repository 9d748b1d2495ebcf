"""CPU suite: the C-ABI library loads, exports every symbol include/spmx_b200.h declares,
and fails loudly (no CPU fallback) when there is no CUDA device. No compute calls here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "spmx_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spmx_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_expected_surface():
    syms = declared_symbols()
    for must in ("spmx_spmm", "spmx_spmm_host", "spmx_split_nnz", "spmx_split_merge",
                 "spmx_split_rows_static", "spmx_merge_path_search", "spmx_plan_create",
                 "spmx_csr_upload", "spmx_csr_wrap_device", "spmx_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2312_05639_b200 import binding
    binding.build_library()
    lib = ctypes.CDLL(binding.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.spmx_abi_version() == 2


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_2312_05639_b200.binding import Context, SpmxRuntimeError
    with pytest.raises(SpmxRuntimeError, match="no CPU fallback"):
        Context(0)


def test_product_never_imports_the_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline legs may touch oracle/:
    nothing in the product package imports, links, loads or opens it."""
    pkg = os.path.join(ROOT, "paper_2312_05639_b200")
    banned = ("import oracle", "from oracle", "liboracle", "oracle/", "pyoracle", "spmx_oracle", "libspmx_ref")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h", ".inc")):
                text = open(os.path.join(dirpath, f), errors="replace").read()
                hits = [b for b in banned if b in text]
                assert not hits, (f, hits)


def test_stream_copy_equals_memcpy(tmp_path):
    """csrc/spmx_stage.cuh: the non-temporal copy that stages pageable host arrays, every size and
    alignment against memcpy (host-only: compiled with g++, no device call)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "test_stream_copy")
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-Wall", "-I/usr/local/cuda/include", "-o", exe,
                           os.path.join(root, "tests", "host", "test_stream_copy.cpp"), "-lpthread"])
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "stream_copy ok" in out.stdout


def _build_c_example(tmp_path):
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_2312_05639_b200")
    exe = str(tmp_path / "spmx_minimal")
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-o", exe,
                           os.path.join(root, "examples", "spmx_minimal.c"), "-L" + pkg, "-lspmx_b200",
                           "-Wl,-rpath," + pkg])
    return exe


def test_header_is_plain_c_and_links_from_c(tmp_path):
    """include/spmx_b200.h is the C-ABI boundary: it must compile as pedantic C99 (no C++ types in
    any signature) and a C program must link against the library (no compute call here)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-fsyntax-only", "-x", "c",
                           os.path.join(root, "include", "spmx_b200.h")])
    out = subprocess.run([_build_c_example(tmp_path), "--link-only"], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.startswith("abi "), out.stdout + out.stderr
