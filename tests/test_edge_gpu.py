"""Adversarial row structures for the work list, the carry fix-up and the host pipeline:
single rows far longer than the whole GPU's worth of chunks (chains of thousands of
partials, summed by the long-chain path), huge rows separated by empty rows, a matrix of
empty rows only. Every element must obey the north_star bound against the unfused
reference (reference.cpp:10-25, via the oracle), the result must be deterministic, and the
host-buffer entry point (row-block pipeline) must return the same bits as the device path.
"""
import numpy as np
import pytest
import torch

from helpers import chain_lengths, north_star_ok

pytestmark = pytest.mark.gpu

CASES = [
    ([1_200_000], 40_000, 64),
    ([500_000, 0, 700_000], 30_000, 64),
    ([600_000, 1, 0, 0, 400_000], 30_000, 48),
    ([1] * 5 + [900_000] + [0] * 1000 + [7] * 2000, 50_000, 128),
    ([0] * 50_000, 10, 32),
]


@pytest.mark.parametrize("lens,n,d", CASES, ids=[f"case{i}" for i in range(len(CASES))])
def test_extreme_rows(ctx, oracle, lens, n, d):
    rng = np.random.default_rng(5)
    m = len(lens)
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(np.asarray(lens, np.uint64))
    nnz = int(rp[-1])
    col = rng.integers(0, n, size=nnz, dtype=np.int64).astype(np.uint32)
    vals = (rng.random(nnz, np.float32) * 2 - 1).astype(np.float32)
    x = (rng.random((n, d), np.float32) * 2 - 1).astype(np.float32)
    unf = oracle.spmm_unfused(m, n, rp, col, vals, x)
    bound = oracle.abs_bound(m, rp, col, vals, x)
    xd = torch.from_numpy(x).cuda()
    for strat in ("row", "nnz", "merge"):
        a = ctx.csr_upload(m, n, rp, col, vals)
        p = ctx.plan(a, strat, 0)
        yd = torch.full((m, d), float("nan"), device="cuda")
        ctx.spmm(p, a, xd, yd)
        ctx.synchronize()
        y = yd.cpu().numpy()
        assert north_star_ok(y, unf, bound), strat
        yd.fill_(float("nan"))
        ctx.spmm(p, a, xd, yd)
        ctx.synchronize()
        assert np.array_equal(y.view(np.uint32), yd.cpu().numpy().view(np.uint32)), "not deterministic"
        yh, _ = ctx.spmm_host(m, n, rp, col, vals, x, strategy=strat)
        assert np.array_equal(yh.view(np.uint32), y.view(np.uint32)), "host pipeline differs"
        if nnz > 100_000:
            cr, cj = p.chunks()
            assert chain_lengths(m, cr, cj, rp).max() > 1000  # the long-chain path did the work
