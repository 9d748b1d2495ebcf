"""CPU suite: the host C++ generators of BASELINE.json's configurations
(paper_2312_05639_b200/host/spmx_workloads.hpp, used by the CLI's --config) produce the SAME
arrays as the Python generators the tests and bench.py use (workloads.py): integer structure and
uniform values bit for bit; N(0,1) values (c3) from the same fp64 Box-Muller formula."""
import os
import struct
import subprocess

import numpy as np
import pytest

from paper_2312_05639_b200 import workloads as W


@pytest.fixture(scope="module")
def tool():
    from tools import hostbuild
    return hostbuild.build_io_tool()


def read_jspm(path):
    raw = open(path, "rb").read()
    assert raw[:4] == b"JSPM"
    ver, m, n, nnz = struct.unpack_from("<Iqqq", raw, 4)
    off = 4 + 4 + 24
    rp = np.frombuffer(raw, np.uint64, m + 1, off); off += (m + 1) * 8
    col = np.frombuffer(raw, np.uint32, nnz, off); off += nnz * 4
    vals = np.frombuffer(raw, np.float32, nnz, off)
    return m, n, nnz, rp, col, vals


CASES = [("c1", 0, 512), ("c2", 11, 0), ("c3", 0, 4096), ("c4", 12, 0), ("c5", 11, 0), ("c1", 0, 0)]


@pytest.mark.parametrize("name,scale,rows", CASES, ids=[f"{n}-s{s}-r{r}" for n, s, r in CASES])
def test_cpp_generator_equals_python_generator(tool, tmp_path, name, scale, rows):
    a_path, x_path = tmp_path / "a.jspm", tmp_path / "x.f32"
    r = subprocess.run([tool, "config", name, str(scale), str(rows), str(a_path), str(x_path)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    a, x, spec = W.make_config(name, scale_override=scale or None, m_override=rows or None)
    rp, col, vals = a.numpy()
    m, n, nnz, rp2, col2, vals2 = read_jspm(a_path)
    assert (m, n, nnz) == (a.m, a.n, a.nnz)
    assert np.array_equal(rp2, rp) and np.array_equal(col2, col)
    x2 = np.fromfile(x_path, np.float32).reshape(a.n, spec["d"])
    if name == "c3":  # Box-Muller in fp64: the two libm's may differ in the last place
        assert np.allclose(vals2, vals, rtol=0, atol=1e-6) and np.mean(vals2.view(np.uint32) == vals.view(np.uint32)) > 0.99
        assert np.allclose(x2, x.numpy(), rtol=0, atol=1e-6)
    else:
        assert np.array_equal(vals2.view(np.uint32), vals.view(np.uint32))
        assert np.array_equal(x2.view(np.uint32), x.numpy().view(np.uint32))
