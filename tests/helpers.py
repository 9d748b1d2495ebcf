"""Shared helpers for the parity tests."""
import numpy as np

D_POOL = [1, 2, 3, 4, 5, 7, 8, 15, 16, 17, 31, 32, 45, 64, 100]  # acceptance.cpp:71
PARTS = [1, 2, 3, 4, 7, 8, 16, 61]


def from_row_lengths(lens):
    """test_partition.cpp:22-32: CSR skeleton with the given row lengths, n = 1."""
    rp = np.zeros(len(lens) + 1, np.uint64)
    rp[1:] = np.cumsum(np.asarray(lens, np.uint64))
    nnz = int(rp[-1])
    return rp, np.zeros(nnz, np.uint32), np.ones(nnz, np.float32)


def exact_cover(ranges, m):
    expect = 0
    for b, e in ranges:
        if b != expect or e < b:
            return False
        expect = e
    return expect == m


def rand_csr(rng, m, n, density, dup=False):
    """Random rectangular CSR, sorted duplicate-free columns per row (like
    tests/oracles.hpp:53-72 but numpy-seeded)."""
    rp = [0]
    cols, vals = [], []
    for _ in range(m):
        c = np.nonzero(rng.random(n) < density)[0].astype(np.uint32)
        if dup and c.size:
            c = np.sort(np.concatenate([c, c[: max(1, c.size // 3)]]))
        cols.append(c)
        vals.append(rng.random(c.size).astype(np.float32))
        rp.append(rp[-1] + c.size)
    col = np.concatenate(cols) if cols else np.zeros(0, np.uint32)
    val = np.concatenate(vals) if vals else np.zeros(0, np.float32)
    return np.asarray(rp, np.uint64), col.astype(np.uint32), val.astype(np.float32)


def north_star_ok(y, y_ref, bound):
    """|y - y_ref| <= 1e-5 * sum|a*x| + 1e-6 elementwise (BASELINE.json north_star)."""
    return np.all(np.abs(y.astype(np.float64) - y_ref.astype(np.float64)) <= 1e-5 * bound + 1e-6)


def split_row_mask(m, chunk_row, chunk_nnz, row_ptr):
    """Rows cut by a chunk boundary of a plan (their sums come from partials)."""
    mask = np.zeros(m, bool)
    for r, j in zip(chunk_row[1:-1], chunk_nnz[1:-1]):
        r = int(r)
        if r < m and int(j) > int(row_ptr[r]):
            mask[r] = True
    return mask


def chain_lengths(m, chunk_row, chunk_nnz, row_ptr):
    """Lengths of the carry chains of a plan: for every chunk boundary that lies inside a row
    which the next chunk ends, the number of chunks holding partial sums of that row before
    the boundary (what carry_fixup_kernel adds to the row's tail)."""
    cr = np.asarray(chunk_row, np.int64); cj = np.asarray(chunk_nnz, np.int64)
    rp = np.asarray(row_ptr, np.int64)
    out = []
    n = len(cr) - 1
    for t in range(n - 1):
        r = cr[t + 1]
        if r < m and cj[t + 1] > rp[r] and cr[t + 2] != r:
            first = int(np.searchsorted(cj, rp[r], side="right")) - 1
            out.append(t - first + 1)
    return np.asarray(out, np.int64)
