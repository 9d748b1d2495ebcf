"""More than 2^32 nonzeros: the CSR offsets of the reference are 64-bit (include/spmx/csr.hpp:14,
row_ptr is uint64) and so are the library's — this is the one test where nonzero offsets, the
merge-path diagonals (m + nnz) and the work-list coordinates really exceed 32 bits (c5, the
largest BASELINE config, stops at 2.6e8 nonzeros / 2^31 elements of X and Y).

A: 2^20 rows of 4094 .. 4100 nonzeros (nnz = 2^32 + 2^20 - 6: one row straddles offset 2^32),
random columns in [0, 2^16), values U[-1, 1); X: 2^16 x 8. About 35 GB of device memory; skipped
on a device with less than 60 GB free.

Checks, for row / nnz / merge:
  * partition ranges equal to the CPU oracle's (split_nnz / split_merge with 64-bit targets:
    t * nnz overflows 32 bits from t = 1 on);
  * SPMX_EXACT_ORDER: every element within the north_star bound of a float64 SpMM evaluated by
    plain torch ops, the sampled rows (first, last, the row across offset 2^32, its neighbours,
    random ones) BITWISE equal to the C oracle's fused chain, and one result for all strategies;
  * default mode: every element within |y - y64| <= 1e-5 * sum|a x| + 1e-6.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

EXACT = 1
M, N, D = 1 << 20, 1 << 16, 8
TOL_REL, TOL_ABS = 1e-5, 1e-6  # BASELINE.json north_star


def _build():
    from paper_2312_05639_b200 import workloads as W
    dev = torch.device("cuda")
    lens = 4097 + (torch.arange(M, device=dev, dtype=torch.int64) % 7) - 3
    rp = torch.zeros(M + 1, dtype=torch.int64, device=dev)
    rp[1:] = torch.cumsum(lens, 0)
    nnz = int(rp[-1])
    assert nnz > (1 << 32)
    g = torch.Generator(device=dev)
    g.manual_seed(2312)
    col = torch.randint(0, N, (nnz,), dtype=torch.int32, device=dev, generator=g)
    vals = torch.rand(nnz, dtype=torch.float32, device=dev, generator=g).mul_(2.0).sub_(1.0)
    x = torch.rand(N, D, dtype=torch.float32, device=dev, generator=g).mul_(2.0).sub_(1.0)
    return W.Csr(M, N, nnz, rp, col, vals), x


def _y64_and_bound(a, x, block_rows=1 << 14):
    """float64 SpMM and sum |a x| by plain torch ops over blocks of rows (independent of the
    library under test)."""
    d = x.shape[1]
    y = torch.empty(a.m, d, dtype=torch.float64, device=x.device)
    b = torch.empty(a.m, d, dtype=torch.float64, device=x.device)
    xd = x.double()
    lens = a.row_ptr[1:] - a.row_ptr[:-1]
    for r in range(0, a.m, block_rows):
        r1 = min(r + block_rows, a.m)
        lo, hi = int(a.row_ptr[r]), int(a.row_ptr[r1])
        prod = a.vals[lo:hi].double().unsqueeze(1) * xd[a.col[lo:hi].long()]
        rows_local = torch.repeat_interleave(torch.arange(r1 - r, device=x.device), lens[r:r1])
        y[r:r1] = torch.zeros(r1 - r, d, dtype=torch.float64, device=x.device).index_add_(0, rows_local, prod)
        b[r:r1] = torch.zeros(r1 - r, d, dtype=torch.float64, device=x.device).index_add_(0, rows_local, prod.abs_())
        del prod, rows_local
    return y, b


def test_more_than_2_pow_32_nonzeros(ctx, oracle):
    free, _ = torch.cuda.mem_get_info()
    if free < 60 * (1 << 30):
        pytest.skip(f"needs about 35 GB of device memory for A alone ({free >> 30} GiB free)")
    a, x = _build()
    da = ctx.csr_wrap(a)  # validates row_ptr and every column index on the device
    y64, bound = _y64_and_bound(a, x)
    tol = TOL_REL * bound + TOL_ABS
    rp_h = a.row_ptr.cpu().numpy().view(np.uint64)
    cross = int(np.searchsorted(rp_h, np.uint64(1 << 32), side="right")) - 1  # the row that holds offset 2^32
    assert rp_h[cross] < (1 << 32) < rp_h[cross + 1]
    rng = np.random.default_rng(11)
    rows = np.unique(np.concatenate([[0, 1, M - 2, M - 1, cross - 1, cross, cross + 1], rng.integers(0, M, 24)]))
    xh = x.cpu().numpy()
    fused = np.zeros((len(rows), D), np.float32)
    for i, r in enumerate(rows):
        lo, hi = int(rp_h[r]), int(rp_h[r + 1])
        fused[i] = oracle.spmm_fused(1, N, np.array([0, hi - lo], np.uint64),
                                     a.col[lo:hi].cpu().numpy().view(np.uint32), a.vals[lo:hi].cpu().numpy(),
                                     xh, threads=1)[0]
    rows_t = torch.from_numpy(rows).cuda()
    y = torch.empty(M, D, device="cuda")
    first_exact = None
    parts = 1000
    for strat in ("row", "nnz", "merge"):
        # the partitioner's 64-bit arithmetic against the oracle's
        p = ctx.plan(da, strat, parts, flags=EXACT)
        want = {"row": lambda: oracle.split_rows_static(M, parts), "nnz": lambda: oracle.split_nnz(rp_h, parts),
                "merge": lambda: oracle.split_merge(rp_h, parts)}[strat]()
        assert np.array_equal(p.ranges(), want), strat
        p.close()
        for flags, label in ((EXACT, "exact"), (0, "default")):
            p = ctx.plan(da, strat, 0, flags=flags)
            y.fill_(float("nan"))
            ctx.spmm(p, da, x, y)
            ctx.synchronize()
            p.close()
            err = (y.double() - y64).abs_()
            bad = int((~(err <= tol)).sum())
            assert bad == 0, f"{strat} {label}: {bad} elements outside the north_star bound"
            del err
            if flags == EXACT:
                got = y[rows_t].cpu().numpy()
                assert np.array_equal(got.view(np.uint32), fused.view(np.uint32)), f"{strat}: sampled rows not bitwise"
                if first_exact is None:
                    first_exact = y.clone()
                else:
                    assert torch.equal(first_exact.view(torch.int32), y.view(torch.int32)), \
                        f"{strat}: exact-order result differs from row-split's"
    da.close()
    del a, x, y, y64, bound, first_exact
    torch.cuda.empty_cache()
