"""CPU suite: the data formats and generators either side of the path,
host/spmx_io.hpp, compared byte for byte with files written by the unmodified reference
(tests/golden/io/, produced by make_golden_io.py)."""
import os
import struct
import subprocess

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "io")


@pytest.fixture(scope="module")
def tool():
    from tools import hostbuild
    return hostbuild.build_io_tool()


def read_jspm(path):
    raw = open(path, "rb").read()
    assert raw[:4] == b"JSPM" and struct.unpack_from("<I", raw, 4)[0] == 1
    m, n, nnz = struct.unpack_from("<QQQ", raw, 8)
    off = 32
    rp = np.frombuffer(raw, np.uint64, m + 1, off); off += 8 * (m + 1)
    col = np.frombuffer(raw, np.uint32, nnz, off); off += 4 * nnz
    vals = np.frombuffer(raw, np.float32, nnz, off); off += 4 * nnz
    assert off == len(raw)
    return m, n, nnz, rp, col, vals


def run(tool, *args):
    return subprocess.run([tool, *map(str, args)], capture_output=True, text=True, timeout=120)


def test_random_csr_and_cache_are_byte_identical_to_the_reference(tool, tmp_path):
    out = tmp_path / "r.jspm"
    assert run(tool, "random-csr", 300, 8, 0.5, 7, out).returncode == 0
    assert open(out, "rb").read() == open(os.path.join(GOLD, "rand300.jspm"), "rb").read()
    z = np.load(os.path.join(GOLD, "rand300.npz"))
    m, n, nnz, rp, col, vals = read_jspm(out)
    assert [m, n, nnz] == z["dims"].tolist()
    assert np.array_equal(rp, z["row_ptr"]) and np.array_equal(col, z["col"]) and np.array_equal(vals, z["vals"])
    # load -> save round trip (csr.cpp:65-104; test_matrix_core.cpp:130-141)
    out2 = tmp_path / "copy.jspm"
    assert run(tool, "copy-jspm", out, out2).returncode == 0
    assert open(out2, "rb").read() == open(out, "rb").read()


def test_random_dense_matches_the_reference(tool, tmp_path):
    out = tmp_path / "x.f32"
    assert run(tool, "random-dense", 300, 5, 11, out).returncode == 0
    z = np.load(os.path.join(GOLD, "rand300.npz"))
    assert np.array_equal(np.fromfile(out, np.float32).reshape(300, 5), z["dense"])
    assert run(tool, "random-dense", 0, 3, 1, out).returncode == 3  # invalid_argument (dense.cpp:10)


def test_matrix_market_writer_is_byte_identical(tool, tmp_path):
    out = tmp_path / "r.mtx"
    assert run(tool, "jspm-to-mtx", os.path.join(GOLD, "rand300.jspm"), out).returncode == 0
    assert open(out, "rb").read() == open(os.path.join(GOLD, "rand300.mtx"), "rb").read()
    # reading it back: values survive %.9g; random_csr keeps duplicate columns, which the
    # loader sums — exactly as the reference's loader does on the same file
    back = tmp_path / "back.jspm"
    assert run(tool, "mtx-to-jspm", out, back).returncode == 0
    z = np.load(os.path.join(GOLD, "rand300.mtx.npz"))
    m, n, nnz, rp, col, vals = read_jspm(back)
    assert [m, n, nnz] == z["dims"].tolist() and nnz < np.load(os.path.join(GOLD, "rand300.npz"))["dims"][2]
    assert np.array_equal(rp, z["row_ptr"]) and np.array_equal(col, z["col"])
    assert np.array_equal(vals.view(np.uint32), z["vals"].view(np.uint32))


@pytest.mark.parametrize("name", ["sym_pattern.mtx", "general_dups.mtx", "integer_sym.mtx"])
def test_matrix_market_reader_matches_the_reference(tool, tmp_path, name):
    """pattern / integer / real, general / symmetric, comments, blank lines, duplicates summed
    (mmio.cpp:20-95; test_matrix_core.cpp:61-128): expected arrays are what the reference's
    load_matrix_market returned for the same files."""
    out = tmp_path / "m.jspm"
    assert run(tool, "mtx-to-jspm", os.path.join(GOLD, name), out).returncode == 0
    z = np.load(os.path.join(GOLD, name + ".npz"))
    m, n, nnz, rp, col, vals = read_jspm(out)
    assert [m, n, nnz] == z["dims"].tolist()
    assert np.array_equal(rp, z["row_ptr"]) and np.array_equal(col, z["col"])
    assert np.array_equal(vals.view(np.uint32), z["vals"].view(np.uint32))


def test_matrix_market_errors_carry_path_and_line(tool, tmp_path):
    cases = {
        "banner.mtx": ("%%NotMM matrix coordinate real general\n1 1 0\n", ":1: missing MatrixMarket banner"),
        "array.mtx": ("%%MatrixMarket matrix array real general\n1 1\n", ":1: array (dense) format not supported"),
        "field.mtx": ("%%MatrixMarket matrix coordinate complex general\n1 1 0\n", ":1: unsupported field type: complex"),
        "sym.mtx": ("%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n", ":1: unsupported symmetry: hermitian"),
        "range.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", ":3: entry index out of range"),
        "short.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "unexpected end of file"),
        "entry.mtx": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n", ":3: bad entry"),
    }
    for fname, (text, want) in cases.items():
        p = tmp_path / fname
        p.write_text(text)
        r = run(tool, "validate", p)
        assert r.returncode == 2 and want in r.stderr and str(p) in r.stderr, (fname, r.stderr)
    r = run(tool, "validate", tmp_path / "absent.mtx")
    assert r.returncode == 2 and "cannot open" in r.stderr


def test_cache_errors(tool, tmp_path):
    bad = tmp_path / "bad.jspm"
    bad.write_bytes(b"NOPE" + b"\0" * 40)
    r = run(tool, "validate", bad)
    assert r.returncode == 2 and "not a JSPM cache file" in r.stderr
    raw = open(os.path.join(GOLD, "rand300.jspm"), "rb").read()
    trunc = tmp_path / "trunc.jspm"
    trunc.write_bytes(raw[:-10])
    r = run(tool, "validate", trunc)
    assert r.returncode == 2 and "truncated cache file" in r.stderr
    # a structurally invalid CSR is rejected on load (csr.cpp:98-101)
    m, n, nnz, rp, col, vals = read_jspm(os.path.join(GOLD, "rand300.jspm"))
    col2 = col.copy(); col2[5] = n + 3
    inv = tmp_path / "inv.jspm"
    inv.write_bytes(raw[:32] + rp.tobytes() + col2.tobytes() + vals.tobytes())
    r = run(tool, "validate", inv)
    assert r.returncode == 2 and "invalid CSR in cache" in r.stderr and "column index out of range at 5" in r.stderr
