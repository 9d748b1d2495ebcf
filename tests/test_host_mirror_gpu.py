"""Runs the C++ host-mirror test driver (the reference's executor/partition cases written
against paper_2312_05639_b200/host/spmx_b200.hpp) on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_cpp_host_mirror_cases():
    from tools import hostbuild
    exe = hostbuild.BIN
    if not os.path.exists(exe):
        exe = hostbuild.build_host_tests()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "host mirror: ALL PASS" in r.stdout
