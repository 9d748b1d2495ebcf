"""Builds the C++ test driver of the host mirror (tests/host/test_host_mirror.cpp) against
libspmx_b200.so. The driver links the test-only oracle for expected values; the mirror header
itself (host/spmx_b200.hpp) depends on the C ABI only."""
import os
import subprocess
import sys

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
SRC = os.path.join(_ROOT, "tests", "host", "test_host_mirror.cpp")
BIN = os.path.join(_ROOT, "tests", "host", "test_host_mirror")


def build_host_tests(verbose: bool = False) -> str:
    deps = [SRC, os.path.join(_PKG, "host", "spmx_b200.hpp"), os.path.join(_ROOT, "include", "spmx_b200.h")]
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
