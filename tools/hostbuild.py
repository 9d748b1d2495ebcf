"""Build plumbing for the C++ pieces around the library (kept outside the product package: the
test driver links the test-only oracle). Builds the C++ test driver of the host mirror (tests/host/test_host_mirror.cpp) against
libspmx_b200.so. The driver links the test-only oracle for expected values; the mirror header
itself (host/spmx_b200.hpp) depends on the C ABI only."""
import os
import subprocess
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_PKG = os.path.join(_ROOT, "paper_2312_05639_b200")
SRC = os.path.join(_ROOT, "tests", "host", "test_host_mirror.cpp")
BIN = os.path.join(_ROOT, "tests", "host", "test_host_mirror")


IO_TOOL_SRC = os.path.join(_ROOT, "tests", "host", "spmx_io_tool.cpp")
IO_TOOL = os.path.join(_ROOT, "tests", "host", "spmx_io_tool")
CLI_SRC = os.path.join(_ROOT, "tools", "spmx_bench_b200.cpp")
CLI = os.path.join(_PKG, "spmx_bench_b200")
_HOST_HDRS = [os.path.join(_PKG, "host", h) for h in ("spmx_b200.hpp", "spmx_io.hpp", "spmx_types.hpp",
                                                        "spmx_workloads.hpp")]


def _stale(target, deps):
    return not os.path.exists(target) or os.path.getmtime(target) < max(os.path.getmtime(d) for d in deps)


def build_io_tool(verbose: bool = False) -> str:
    """Host-only tool over host/spmx_io.hpp (no CUDA): used by the CPU test-suite."""
    if _stale(IO_TOOL, [IO_TOOL_SRC] + _HOST_HDRS):
        cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-fopenmp", "-o", IO_TOOL, IO_TOOL_SRC]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    return IO_TOOL


def build_cli(verbose: bool = False) -> str:
    """spmx_bench_b200: the reference's bench CLI for the B200 path (tools/spmx_bench_b200.cpp)."""
    if _stale(CLI, [CLI_SRC, os.path.join(_ROOT, "include", "spmx_b200.h")] + _HOST_HDRS):
        cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-fopenmp", "-o", CLI, CLI_SRC, "-L" + _PKG, "-lspmx_b200",
               "-Wl,-rpath,$ORIGIN", "-L/usr/local/cuda/lib64", "-lcudart"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    return CLI


def build_host_tests(verbose: bool = False) -> str:
    build_io_tool(verbose)
    build_cli(verbose)
    deps = [SRC, os.path.join(_ROOT, "include", "spmx_b200.h")] + _HOST_HDRS
    if os.path.exists(BIN) and os.path.getmtime(BIN) >= max(os.path.getmtime(d) for d in deps):
        return BIN
    subprocess.check_call(["make", "-C", os.path.join(_ROOT, "oracle"), "liboracle.so"],
                          stdout=subprocess.DEVNULL)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-o", BIN, SRC,
           "-L" + _PKG, "-lspmx_b200", "-L" + os.path.join(_ROOT, "oracle"), "-loracle",
           "-Wl,-rpath,$ORIGIN/../../paper_2312_05639_b200", "-Wl,-rpath,$ORIGIN/../../oracle",
           "-L/usr/local/cuda/lib64", "-lcudart"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    return BIN
