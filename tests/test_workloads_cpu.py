"""CPU suite: the seeded generators for BASELINE.json's configs."""
import numpy as np
import torch

from paper_2312_05639_b200 import workloads as W


def test_mix64_matches_reference_splitmix():
    # splitmix64 known answers for state 0: first outputs of the published generator
    out = W.mix64(torch.tensor([0], dtype=torch.int64))
    assert int(out.item()) & 0xFFFFFFFFFFFFFFFF == 0xE220A8397B1DCDAF


def test_c1_exact_degree_sorted_distinct():
    a, x, spec = W.make_config("c1")
    rp, col, vals = a.numpy()
    assert (a.m, a.n, a.nnz, spec["d"]) == (4096, 4096, 65536, 32)
    assert np.all(np.diff(rp.astype(np.int64)) == 16)
    c = col.reshape(4096, 16).astype(np.int64)
    assert np.all(np.diff(c, axis=1) > 0)
    assert vals.min() >= -1 and vals.max() < 1 and x.min() >= -1 and x.max() < 1
    a2, x2, _ = W.make_config("c1")
    assert torch.equal(a.col, a2.col) and torch.equal(x, x2)


def test_rmat_properties():
    a, x, spec = W.make_config("c2", scale_override=12)
    rp, col, vals = a.numpy()
    assert a.m == 4096 and 0 < a.nnz <= 16 * 4096
    lens = np.diff(rp.astype(np.int64))
    for r in np.nonzero(lens > 1)[0][:200]:
        c = col[rp[r]:rp[r + 1]].astype(np.int64)
        assert np.all(np.diff(c) > 0)  # sorted, duplicates merged
    assert vals.min() > 0 and vals.max() <= 1
    assert lens.max() > 20 * lens.mean()  # power-law rows
    a4, _, _ = W.make_config("c4", scale_override=12)
    assert a4.nnz < 32 * 4096 and np.diff(a4.numpy()[0].astype(np.int64)).max() > lens.max()


def test_banded_properties():
    a, x, spec = W.make_config("c3", m_override=1 << 13)
    rp, col, vals = a.numpy()
    lens = np.diff(rp.astype(np.int64))
    assert lens.min() >= 1 and lens.max() <= 64 and abs(lens.mean() - 32) < 0.5
    rows = np.repeat(np.arange(a.m), lens)
    hb = min(65536, a.m // 4)
    assert np.all(np.abs(col.astype(np.int64) - rows) <= hb)
    assert abs(float(vals.mean())) < 0.02 and abs(float(vals.std()) - 1) < 0.02
    assert abs(float(x.std()) - 1) < 0.02


def test_row_slice_rebases():
    a, _, _ = W.make_config("c2", scale_override=10)
    s = a.row_slice(100, 300)
    assert s.m == 200 and int(s.row_ptr[0]) == 0 and int(s.row_ptr[-1]) == s.nnz
    lo = int(a.row_ptr[100])
    assert torch.equal(s.col, a.col[lo:lo + s.nnz])


def test_algorithmic_bytes_formula():
    # c2 upper bound 675 MB
    assert W.algorithmic_bytes(1 << 20, 1 << 20, 16 * (1 << 20), 64) == 8 * 16 * (1 << 20) + 4 * ((1 << 20) + 1) + 2 * 4 * (1 << 20) * 64
