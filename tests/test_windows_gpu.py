"""Row structures that stress the kernel's staging windows (csrc/spmx_kernels.cuh,
process_piece): a window ends after 64 staged non-empty rows or 512 scanned rows, whichever
comes first, and a piece (chunk of the work list, or a whole strategy range in exact-order
mode) may span many windows. Cases: runs of one-nonzero rows (record capacity reached inside
a chunk), long stretches of empty rows (scan limit reached with no record staged), mixtures
around both limits, and exact-order plans with few parts (thousands of rows and hundreds of
windows per lane group). Exact-order results must equal the reference's fused CSR-order
result bit for bit (src/interp.cpp:36-51 via the oracle); default-mode results must obey the
north_star bound against the unfused reference (src/reference.cpp:10-25) and be identical
across the three division schemes on rows no chunk boundary cuts.
"""
import numpy as np
import pytest
import torch

from helpers import north_star_ok
from paper_2312_05639_b200.binding import EXACT_ORDER

pytestmark = pytest.mark.gpu


def _lens(kind, rng):
    if kind == "ones":            # every row one nonzero: 128 non-empty rows per 256-item chunk
        return np.ones(40_000, np.int64)
    if kind == "ones_twos":       # 1-2 nonzeros per row
        return rng.integers(1, 3, size=30_000)
    if kind == "empty_runs":      # a nonzero row every 600-700 rows: scan limit (512) with nothing staged
        lens = np.zeros(200_000, np.int64)
        pos = np.cumsum(rng.integers(600, 700, size=280))
        lens[pos[pos < lens.size]] = rng.integers(1, 40, size=int((pos < lens.size).sum()))
        return lens
    if kind == "edge_64":         # exactly 64 / 65 non-empty rows between long empty stretches
        block = np.concatenate([np.ones(64, np.int64), np.zeros(511, np.int64), np.ones(65, np.int64),
                                np.zeros(513, np.int64), np.full(3, 100, np.int64)])
        return np.tile(block, 40)
    if kind == "mixed":           # power-law lengths with half of the rows empty
        lens = (rng.pareto(1.2, size=60_000) * 3).astype(np.int64)
        lens[rng.random(lens.size) < 0.5] = 0
        return np.minimum(lens, 5_000)
    raise ValueError(kind)


def _build(kind, d, seed):
    rng = np.random.default_rng(seed)
    lens = _lens(kind, rng)
    m = int(lens.size)
    n = 5_000
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(lens.astype(np.uint64))
    nnz = int(rp[-1])
    col = rng.integers(0, n, size=nnz, dtype=np.int64).astype(np.uint32)
    vals = (rng.random(nnz, np.float32) * 2 - 1).astype(np.float32)
    x = (rng.random((n, d), np.float32) * 2 - 1).astype(np.float32)
    return m, n, rp, col, vals, x


@pytest.mark.parametrize("kind", ["ones", "ones_twos", "empty_runs", "edge_64", "mixed"])
@pytest.mark.parametrize("d", [32, 64, 128, 5, 20])
def test_window_limits(ctx, oracle, kind, d):
    m, n, rp, col, vals, x = _build(kind, d, seed=11)
    fused = oracle.spmm_fused(m, n, rp, col, vals, x)
    unf = oracle.spmm_unfused(m, n, rp, col, vals, x)
    bound = oracle.abs_bound(m, rp, col, vals, x)
    xd = torch.from_numpy(x).cuda()
    a = ctx.csr_upload(m, n, rp, col, vals)
    # exact-order mode: a handful of parts -> every lane group walks thousands of rows
    for strat, parts in (("row", 3), ("nnz", 7), ("merge", 64), ("merge", 0)):
        p = ctx.plan(a, strat, parts, flags=EXACT_ORDER)
        yd = torch.full((m, d), float("nan"), device="cuda")
        ctx.spmm(p, a, xd, yd)
        ctx.synchronize()
        y = yd.cpu().numpy()
        assert np.array_equal(y.view(np.uint32), fused.view(np.uint32)), (kind, d, strat, parts)
        p.close()
    # dynamic row dispatch (row-granular pieces of 128 rows, several windows for sparse rows)
    p = ctx.plan(a, "row", 0, dynamic=True, flags=EXACT_ORDER | 8)  # 8 = SPMX_CLAIM_KERNEL
    yd = torch.full((m, d), float("nan"), device="cuda")
    ctx.spmm(p, a, xd, yd)
    ctx.synchronize()
    assert np.array_equal(yd.cpu().numpy().view(np.uint32), fused.view(np.uint32)), (kind, d, "dynamic")
    p.close()
    # default mode: bounded chunks, cut rows summed from partials
    for strat in ("row", "nnz", "merge"):
        p = ctx.plan(a, strat, 0)
        yd = torch.full((m, d), float("nan"), device="cuda")
        ctx.spmm(p, a, xd, yd)
        ctx.synchronize()
        y = yd.cpu().numpy()
        assert north_star_ok(y, unf, bound), (kind, d, strat)
        p.close()
    a.close()
