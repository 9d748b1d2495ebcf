"""CPU suite: pins the oracle (oracle/spmx_oracle.c) against the reference's own golden
vectors (restated from /root/reference/proj/tests) and against fixtures produced by running
the unmodified reference (tests/golden/, see make_golden.py)."""
import os

import numpy as np
import pytest

from helpers import PARTS, exact_cover, from_row_lengths, rand_csr

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_worked_example_and_shape_error(oracle):
    # test_matrix_core.cpp:181-189
    from oracle.pyoracle import OracleInvalidArgument
    rp = np.array([0, 1, 3], np.uint64)
    col = np.array([0, 0, 1], np.uint32)
    vals = np.array([2, 1, 3], np.float32)
    x = np.array([[1, 2], [3, 4]], np.float32)
    assert oracle.spmm_unfused(2, 2, rp, col, vals, x).ravel().tolist() == [2, 4, 10, 14]
    assert oracle.spmm_fused(2, 2, rp, col, vals, x).ravel().tolist() == [2, 4, 10, 14]
    with pytest.raises(OracleInvalidArgument):
        oracle.spmm_unfused(2, 2, rp, col, vals, np.zeros((3, 2), np.float32))


def test_identity_and_empty_rows(oracle):
    # test_matrix_core.cpp:159-178
    x = np.random.default_rng(1).random((3, 5), np.float32)
    rp = np.arange(4, dtype=np.uint64)
    y = oracle.spmm_unfused(3, 3, rp, np.arange(3, dtype=np.uint32), np.ones(3, np.float32), x)
    assert np.array_equal(y, x)
    y2 = oracle.spmm_fused(2, 2, np.array([0, 0, 1], np.uint64), np.array([1], np.uint32),
                           np.array([4], np.float32), x[:2, :3].copy())
    assert np.all(y2[0] == 0)


def test_partition_goldens(oracle):
    # test_partition.cpp:36-42, 76-83, 85-96, 119-126
    from oracle.pyoracle import OracleInvalidArgument
    assert oracle.split_rows_static(10, 4).tolist() == [[0, 3], [3, 6], [6, 8], [8, 10]]
    assert oracle.split_rows_static(4, 4).tolist() == [[0, 1], [1, 2], [2, 3], [3, 4]]
    assert oracle.split_rows_static(2, 4).tolist() == [[0, 1], [1, 2], [2, 2], [2, 2]]
    with pytest.raises(OracleInvalidArgument):
        oracle.split_rows_static(5, 0)
    rp, _, _ = from_row_lengths([4, 1, 1, 2])
    assert oracle.split_nnz(rp, 2).tolist() == [[0, 1], [1, 4]]
    assert oracle.split_nnz(rp, 1).tolist() == [[0, 4]]
    assert oracle.split_nnz(from_row_lengths([0, 0, 0])[0], 2).tolist() == [[0, 0], [0, 3]]
    assert oracle.merge_path_search(rp, 0) == (0, 0)
    assert oracle.merge_path_search(rp, 12) == (4, 8)
    assert oracle.merge_path_search(rp, 6) == (1, 5)
    with pytest.raises(OracleInvalidArgument):
        oracle.merge_path_search(rp, 13)
    assert oracle.split_merge(rp, 2).tolist() == [[0, 1], [1, 4]]
    assert oracle.split_merge(rp, 1).tolist() == [[0, 4]]
    assert oracle.split_merge(from_row_lengths([3] * 6)[0], 3).tolist() == [[0, 2], [2, 4], [4, 6]]


def test_next_batch_sequential(oracle):
    # test_partition.cpp:44-52
    c = [0]
    assert oracle.next_batch(c, 128, 300) == (0, 128)
    assert oracle.next_batch(c, 128, 300) == (128, 256)
    assert oracle.next_batch(c, 128, 300) == (256, 300)
    assert oracle.next_batch(c, 128, 300) is None
    assert oracle.next_batch([0], 128, 0) is None


def test_checksum_and_error_metric(oracle):
    # dense.cpp:17-28 (FNV-1a-64 of the empty input is the offset basis); executor.cpp:27-34
    assert oracle.checksum(np.zeros(0, np.float32)) == 0xcbf29ce484222325
    h = 0xcbf29ce484222325
    for byte in np.array([1.5, -2.0], np.float32).tobytes():
        h = ((h ^ byte) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    assert oracle.checksum(np.array([1.5, -2.0], np.float32)) == h
    y = np.array([1.0, 2.0, 0.0], np.float32)
    ref = np.array([1.0, 2.00002, 1e-9], np.float32)
    want = max(abs(2.0 - float(np.float32(2.00002))) / float(np.float32(2.00002)),
               float(np.float32(1e-9)) / 1e-6)
    assert abs(oracle.max_relative_error(y, ref) - want) < 1e-12


def test_oracle_equals_reference_on_golden_instances(oracle, golden_instances):
    """Fixtures were produced by the unmodified reference library: Y of run_spmm (native JIT,
    bitwise equal to its interpreter), Y of spmm_reference, all partitions, every diagonal."""
    assert len(golden_instances) == 40
    for g in golden_instances:
        m, n, nnz, d = (int(v) for v in g["dims"])
        yf = oracle.spmm_fused(m, n, g["row_ptr"], g["col"], g["vals"], g["x"], threads=3)
        yu = oracle.spmm_unfused(m, n, g["row_ptr"], g["col"], g["vals"], g["x"])
        assert np.array_equal(yf.view(np.uint32), g["y_fused"].view(np.uint32))
        assert np.array_equal(yu.view(np.uint32), g["y_unfused"].view(np.uint32))
        assert oracle.max_relative_error(yf, yu) <= 1e-5  # acceptance criterion 2
        for t in PARTS:
            assert np.array_equal(oracle.split_nnz(g["row_ptr"], t), g[f"nnz{t}"])
            assert np.array_equal(oracle.split_merge(g["row_ptr"], t), g[f"merge{t}"])
            assert np.array_equal(oracle.split_rows_static(m, t), g[f"rows{t}"])
        for k in range(0, m + nnz + 1, max(1, (m + nnz) // 97)):
            assert oracle.merge_path_search(g["row_ptr"], k) == (int(g["mp_i"][k]), int(g["mp_j"][k]))
            assert oracle.merge_walk(g["row_ptr"], k) == (int(g["mp_i"][k]), int(g["mp_j"][k]))


def test_range_decomposition_invariance(oracle):
    # test_interp.cpp:157-169: any exact row cover gives the same bits
    rng = np.random.default_rng(4)
    m, n, d = 90, 70, 33
    rp, col, vals = rand_csr(rng, m, n, 0.1)
    x = rng.random((n, d), np.float32)
    whole = oracle.spmm_fused(m, n, rp, col, vals, x)
    for t in (2, 5, 11):
        y = np.full((m, d), np.nan, np.float32)
        for b, e in oracle.split_merge(rp, t):
            oracle.spmm_fused_range(m, n, rp, col, vals, x, y, int(b), int(e))
        assert np.array_equal(y.view(np.uint32), whole.view(np.uint32))


def test_executor_fixture_checksum(oracle):
    z = np.load(os.path.join(GOLD, "ref_executor.npz"))
    y = oracle.spmm_fused(200, 200, z["row_ptr"], z["col"], z["vals"], z["x"])
    assert oracle.checksum(y) == int(z["checksum"][0])


def test_config_siblings_against_reference_checksums(oracle):
    from paper_2312_05639_b200 import workloads as W
    z = np.load(os.path.join(GOLD, "ref_configs.npz"))
    small = {"c1": {}, "c2": {"scale_override": 12}, "c3": {"m_override": 1 << 12},
             "c4": {"scale_override": 12}, "c5": {"scale_override": 11}}
    for name, kw in small.items():
        a, x, spec = W.make_config(name, **kw)
        rp, col, vals = a.numpy()
        assert [a.m, a.n, a.nnz, spec["d"]] == z[name + "_dims"].tolist()
        assert oracle.validate_csr(a.m, a.n, a.nnz, rp, col) == 0
        yf = oracle.spmm_fused(a.m, a.n, rp, col, vals, x.numpy())
        assert oracle.checksum(yf) == int(z[name + "_checksum_fused"][0])
        assert np.array_equal(yf[:4], z[name + "_y_head"])
        yu = oracle.spmm_unfused(a.m, a.n, rp, col, vals, x.numpy())
        assert oracle.checksum(yu) == int(z[name + "_checksum_unfused"][0])
        bound = oracle.abs_bound(a.m, rp, col, vals, x.numpy())
        assert np.all(np.abs(yf.astype(np.float64) - yu) <= 1e-5 * bound + 1e-6)
        for t in (7, 64):
            assert np.array_equal(oracle.split_nnz(rp, t), z[name + f"_nnz{t}"])
            assert np.array_equal(oracle.split_merge(rp, t), z[name + f"_merge{t}"])


def test_partition_properties(oracle):
    # test_partition.cpp:128-157
    rng = np.random.default_rng(23)
    for _ in range(200):
        m = int(rng.integers(200))
        rp, col, vals = rand_csr(rng, m, 30, 0.25 * rng.integers(100) / 100.0)
        nnz = int(rp[-1])
        t = 1 + int(rng.integers(16))
        lens = np.diff(rp.astype(np.int64))
        max_row = int(lens.max()) if m else 0
        rows, nnzs, merges = oracle.split_rows_static(m, t), oracle.split_nnz(rp, t), oracle.split_merge(rp, t)
        assert exact_cover(rows, m) and exact_cover(nnzs, m) and exact_cover(merges, m)
        share = (m + nnz + t - 1) // t
        for i in range(t):
            assigned = int(rp[nnzs[i, 1]]) - int(rp[nnzs[i, 0]])
            assert abs(assigned - nnz / t) <= max_row + 1e-9
            work = int(merges[i, 1] - merges[i, 0]) + int(rp[merges[i, 1]]) - int(rp[merges[i, 0]])
            assert work <= share + 1 + max_row


def test_live_reference_agrees_when_built(oracle, reflib):
    """Where oracle/_ref exists (this container), cross-check on fresh random instances."""
    rng = np.random.default_rng(99)
    for _ in range(10):
        m, n, d = 1 + int(rng.integers(150)), 1 + int(rng.integers(150)), 1 + int(rng.integers(70))
        rp, col, vals = rand_csr(rng, m, n, 0.1)
        x = rng.random((n, d), np.float32)
        a = reflib.csr(m, n, rp, col, vals)
        y, rep = reflib.run_spmm(a, x, "nnz", False, 3, "native")
        assert np.array_equal(oracle.spmm_fused(m, n, rp, col, vals, x).view(np.uint32), y.view(np.uint32))
        assert np.array_equal(oracle.spmm_unfused(m, n, rp, col, vals, x), reflib.spmm_reference(a, x))
        assert oracle.checksum(y) == reflib.checksum(y)
        for t in (1, 3, 9):
            assert np.array_equal(oracle.split_nnz(rp, t), reflib.split_nnz(a, t))
            assert np.array_equal(oracle.split_merge(rp, t), reflib.split_merge(a, t))
