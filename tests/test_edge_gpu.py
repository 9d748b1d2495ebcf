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


def _poison_carry_pool(ctx, rng):
    """Fills the stream-ordered pool with non-zero garbage where a later plan's carry rows
    will live: run a merge plan whose rows are all cut (large partial sums), then free it."""
    m, n, d = 3, 2000, 64
    lens = np.array([300_000, 200_000, 250_000], np.uint64)
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(lens)
    nnz = int(rp[-1])
    col = rng.integers(0, n, size=nnz, dtype=np.int64).astype(np.uint32)
    vals = np.full(nnz, 1000.0, np.float32)
    x = np.full((n, d), 7.0, np.float32)
    a = ctx.csr_upload(m, n, rp, col, vals)
    p = ctx.plan(a, "merge", 0)
    yd = torch.empty(m, d, device="cuda")
    ctx.spmm(p, a, torch.from_numpy(x).cuda(), yd)
    ctx.synchronize()
    p.close()
    a.close()


@pytest.mark.parametrize("m,row_nnz,parts", [(1, 1, 4), (1, 1, 64), (2, 3, 50), (5, 2, 301), (3, 40, 1000)])
def test_more_parts_than_merge_items(ctx, oracle, m, row_nnz, parts):
    """merge-split with parts >> m + nnz: duplicate diagonals give empty chunks that sit inside
    a row's carry chain. Their partial is zero by definition; the carry buffer comes from the
    stream-ordered pool unzeroed, so the empty chunk itself must write that zero. Run after
    the pool has been filled with large values, twice, on several widths."""
    rng = np.random.default_rng(11)
    n = 37
    rp = np.arange(m + 1, dtype=np.uint64) * np.uint64(row_nnz)
    nnz = int(rp[-1])
    col = rng.integers(0, n, size=nnz, dtype=np.int64).astype(np.uint32)
    vals = (rng.random(nnz, np.float32) + 0.5).astype(np.float32)
    for d in (64, 32, 5, 128):
        x = (rng.random((n, d), np.float32) + 0.5).astype(np.float32)
        unf = oracle.spmm_unfused(m, n, rp, col, vals, x)
        bound = oracle.abs_bound(m, rp, col, vals, x)
        for rep in range(2):
            _poison_carry_pool(ctx, rng)
            a = ctx.csr_upload(m, n, rp, col, vals)
            p = ctx.plan(a, "merge", parts)
            yd = torch.full((m, d), float("nan"), device="cuda")
            ctx.spmm(p, a, torch.from_numpy(x).cuda(), yd)
            ctx.synchronize()
            assert north_star_ok(yd.cpu().numpy(), unf, bound), (d, rep, yd.cpu().numpy()[:, :4], unf[:, :4])
            p.close()
            a.close()


def test_invalid_column_under_dynamic_dispatch_is_einval(ctx):
    """spmx_spmm_host validates column indices on the device while the kernels are queued: an
    out-of-range column must come back as SPMX_EINVAL for dynamic row dispatch too (the
    reference's default mode), not as an illegal-address fault."""
    from paper_2312_05639_b200.binding import SpmxInvalidArgument
    rng = np.random.default_rng(3)
    m, n, d = 4000, 300, 64
    lens = rng.integers(0, 40, size=m)
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(lens.astype(np.uint64))
    nnz = int(rp[-1])
    col = rng.integers(0, n, size=nnz, dtype=np.int64).astype(np.uint32)
    col[nnz // 2] = np.uint32(0x7fffff00)  # far outside X
    vals = rng.random(nnz, np.float32)
    x = rng.random((n, d), np.float32)
    for dyn, flags in ((True, 8), (True, 0), (False, 0)):  # 8 = SPMX_CLAIM_KERNEL: spmm_dynamic_kernel
        with pytest.raises(SpmxInvalidArgument, match="column index out of range"):
            ctx.spmm_host(m, n, rp, col, vals, x, strategy="row", dynamic=dyn, flags=flags)
    # the context is still usable afterwards (no sticky CUDA error)
    col[nnz // 2] = 0
    y, _ = ctx.spmm_host(m, n, rp, col, vals, x, strategy="row", dynamic=True, flags=8)
    assert np.isfinite(y).all()


def test_structure_only_handle(ctx, oracle):
    """spmx_rowptr_upload: partitioner and plans work from row_ptr alone; SpMM refuses it."""
    from paper_2312_05639_b200.binding import SpmxLogicError
    rng = np.random.default_rng(1)
    m = 5000
    lens = rng.integers(0, 30, size=m)
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(lens.astype(np.uint64))
    s = ctx.rowptr_upload(m, rp)
    for parts in (1, 7, 64):
        assert np.array_equal(ctx.split_nnz(s, parts), oracle.split_nnz(rp, parts))
        assert np.array_equal(ctx.split_merge(s, parts), oracle.split_merge(rp, parts))
    p = ctx.plan(s, "merge", 16)
    assert np.array_equal(p.ranges(), oracle.split_merge(rp, 16))
    with pytest.raises(SpmxLogicError):
        ctx.spmm(p, s, torch.zeros(1, 4, device="cuda"), torch.zeros(m, 4, device="cuda"))
    p.close()
    s.close()


@pytest.mark.parametrize("d", [64, 32, 128, 100, 45, 7, 300])
def test_long_rows_in_exact_order_mode_are_bitwise(ctx, oracle, d):
    """Exact-order plans hand rows of 1024 nonzeros or more to spmm_long_row_kernel (one CTA per
    row: all threads gather, one warp runs the fmaf chain in CSR order). Bitwise equal to the
    oracle's fused result (interp.cpp:36-51) for every strategy, for widths that are not a
    multiple of 4 or 32, wider than one 128-column slab, and for X / Y that are only 4-byte
    aligned (scalar loads); rows just below and at the threshold included."""
    from paper_2312_05639_b200.binding import EXACT_ORDER
    rng = np.random.default_rng(21)
    lens = [5000, 0, 1023, 1024, 3, 70_000, 0, 0, 1500, 17] + [int(v) for v in rng.integers(0, 40, size=300)]
    m, n = len(lens), 3000
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(np.asarray(lens, np.uint64))
    nnz = int(rp[-1])
    col = rng.integers(0, n, size=nnz, dtype=np.int64).astype(np.uint32)
    vals = (rng.random(nnz, np.float32) * 2 - 1).astype(np.float32)
    x = (rng.random((n, d), np.float32) * 2 - 1).astype(np.float32)
    want = oracle.spmm_fused(m, n, rp, col, vals, x)
    a = ctx.csr_upload(m, n, rp, col, vals)
    for shift in (0, 1):  # 1: X and Y start 4 bytes off a 16-byte boundary
        xbuf = torch.zeros(n * d + 4, device="cuda")
        ybuf = torch.full((m * d + 4,), float("nan"), device="cuda")
        xd = xbuf[shift:shift + n * d].view(n, d)
        yd = ybuf[shift:shift + m * d].view(m, d)
        xd.copy_(torch.from_numpy(x))
        for strat in ("row", "nnz", "merge"):
            for parts in (0, 3):
                p = ctx.plan(a, strat, parts, flags=EXACT_ORDER)
                yd.fill_(float("nan"))
                ctx.spmm(p, a, xd, yd)
                ctx.synchronize()
                got = yd.cpu().numpy()
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (d, shift, strat, parts)
                p.close()
    # the host-buffer entry point takes the same route (one block when the plan has long rows)
    yh, _ = ctx.spmm_host(m, n, rp, col, vals, x, strategy="merge", flags=EXACT_ORDER)
    assert np.array_equal(yh.view(np.uint32), want.view(np.uint32))
    a.close()
