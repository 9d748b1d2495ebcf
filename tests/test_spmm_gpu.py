"""CUDA SpMM (through the C ABI) vs the oracle / the reference's golden vectors.

Exact mode (SPMX_EXACT_ORDER): bitwise equal to the reference's run_spmm for every
strategy and part count (checksum equality, dense.cpp:17-28).
Default mode: rows not cut by a chunk boundary (interior cuts never fall inside rows
shorter than LONG_SEG) are still bitwise equal; every element obeys the north_star bound
|y - y_ref| <= 1e-5 * sum|a*x| + 1e-6 against the unfused reference (reference.cpp:10-25).
"""
import numpy as np
import pytest
import torch

from helpers import D_POOL, chain_lengths, north_star_ok, rand_csr, split_row_mask

pytestmark = pytest.mark.gpu

EXACT = 1
CLAIM = 8  # SPMX_CLAIM_KERNEL
LONG_SEG = 128  # interior chunk cuts never split rows shorter than this (snap_len in csrc/spmx_capi.cu)
STRATS = ("row", "nnz", "merge")


def run(ctx, m, n, rp, col, vals, x, strategy="row", parts=0, flags=0, dynamic=False, batch=128,
        poison=True):
    a = ctx.csr_upload(m, n, rp, col, vals)
    p = ctx.plan(a, strategy, parts, dynamic=dynamic, batch=batch, flags=flags)
    xd = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    yd = torch.full((m, x.shape[1]), float("nan") if poison else 0.0, device="cuda")
    ctx.spmm(p, a, xd, yd)
    ctx.synchronize()
    return yd.cpu().numpy(), p


def test_worked_example(ctx):
    # test_matrix_core.cpp:181-186: [[2,0],[1,3]] * [[1,2],[3,4]] = [[2,4],[10,14]]
    rp = np.array([0, 1, 3], np.uint64)
    col = np.array([0, 0, 1], np.uint32)
    vals = np.array([2, 1, 3], np.float32)
    x = np.array([[1, 2], [3, 4]], np.float32)
    for s in STRATS:
        for fl in (0, EXACT):
            y, _ = run(ctx, 2, 2, rp, col, vals, x, s, 2, fl)
            assert y.tolist() == [[2, 4], [10, 14]]


def test_shape_errors(ctx):
    # test_executor.cpp:163-175, executor.cpp:38: A.n != X.rows -> invalid_argument
    from paper_2312_05639_b200.binding import SpmxInvalidArgument
    rp = np.arange(5, dtype=np.uint64)
    a = ctx.csr_upload(4, 4, rp, np.arange(4, dtype=np.uint32), np.ones(4, np.float32))
    p = ctx.plan(a, "row")
    x = torch.zeros(5, 4, device="cuda")
    y = torch.zeros(4, 4, device="cuda")
    with pytest.raises(SpmxInvalidArgument):
        ctx.spmm(p, a, x, y)


def test_identity_returns_x_bitwise(ctx):
    # test_executor.cpp:53-65: identity(64), d=45, every strategy x dispatch x T
    n, d = 64, 45
    rp = np.arange(n + 1, dtype=np.uint64)
    col = np.arange(n, dtype=np.uint32)
    vals = np.ones(n, np.float32)
    x = np.random.default_rng(3).random((n, d), np.float32)
    for t in (1, 3, 8, 0):
        for s in STRATS:
            for fl in (0, EXACT):
                y, _ = run(ctx, n, n, rp, col, vals, x, s, t, fl)
                assert np.array_equal(y, x)
        for fl in (0, CLAIM):  # dynamic dispatch: served by the work list / by the claim kernel
            y, _ = run(ctx, n, n, rp, col, vals, x, "row", t, fl, dynamic=True, batch=16)
            assert np.array_equal(y, x)


def test_empty_rows_are_zeroed(ctx):
    # test_matrix_core.cpp:170-178, test_interp.cpp:81-93: stale Y is overwritten with zeros
    rp = np.array([0, 0, 1, 1, 1], np.uint64)
    col = np.array([1], np.uint32)
    vals = np.array([4], np.float32)
    x = np.random.default_rng(2).random((2, 3), np.float32)
    for s in STRATS:
        for fl in (0, EXACT):
            y, _ = run(ctx, 4, 2, rp, col, vals, x, s, 3, fl)
            assert np.all(y[[0, 2, 3]] == 0) and np.array_equal(y[1], np.float32(4) * x[1])
    # all-empty matrix, and m = 0
    y, _ = run(ctx, 3, 2, np.zeros(4, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32), x)
    assert np.all(y == 0)
    y, _ = run(ctx, 0, 2, np.zeros(1, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.float32), x)
    assert y.shape == (0, 3)


def test_reference_golden_instances_bitwise(ctx, golden_instances, oracle):
    """The reference's acceptance instances (acceptance.cpp:69-124); expected Y comes from
    the unmodified reference (run_spmm native == interpreter), stored in tests/golden."""
    for idx, g in enumerate(golden_instances):
        m, n, nnz, d = (int(v) for v in g["dims"])
        want = g["y_fused"]
        for s in STRATS:
            for t in (1, 2, 4, 8, 0):
                y, _ = run(ctx, m, n, g["row_ptr"], g["col"], g["vals"], g["x"], s, t, EXACT)
                assert np.array_equal(y.view(np.uint32), want.view(np.uint32)), (idx, s, t)
                assert oracle.checksum(y) == oracle.checksum(want)
        for fl in (EXACT, EXACT | CLAIM):
            y, _ = run(ctx, m, n, g["row_ptr"], g["col"], g["vals"], g["x"], "row", 0, fl,
                       dynamic=True, batch=32)
            assert np.array_equal(y.view(np.uint32), want.view(np.uint32))
        # acceptance criterion 2: within 1e-5 of spmm_reference (positive data, no cancellation)
        assert oracle.max_relative_error(y, g["y_unfused"]) <= 1e-5


def test_reference_golden_instances_default_mode(ctx, golden_instances, oracle):
    for idx, g in enumerate(golden_instances):
        m, n, nnz, d = (int(v) for v in g["dims"])
        bound = oracle.abs_bound(m, g["row_ptr"], g["col"], g["vals"], g["x"])
        lens = np.diff(g["row_ptr"].astype(np.int64))
        for s in STRATS:
            for t in (1, 3, 16, 0):
                y, p = run(ctx, m, n, g["row_ptr"], g["col"], g["vals"], g["x"], s, t, 0)
                assert north_star_ok(y, g["y_unfused"], bound), (idx, s, t)
                cr, cj = p.chunks()
                exact_rows = ~split_row_mask(m, cr, cj, g["row_ptr"]) & (lens < LONG_SEG)
                assert np.array_equal(y[exact_rows].view(np.uint32),
                                      g["y_fused"][exact_rows].view(np.uint32)), (idx, s, t)
        # dynamic row dispatch in the default mode: the row-split work list, and the literal
        # claim kernel (row-granular: every row one fmaf chain, bitwise equal to the reference)
        y, _ = run(ctx, m, n, g["row_ptr"], g["col"], g["vals"], g["x"], "row", 0, 0, dynamic=True, batch=32)
        assert north_star_ok(y, g["y_unfused"], bound), (idx, "dynamic")
        y, _ = run(ctx, m, n, g["row_ptr"], g["col"], g["vals"], g["x"], "row", 0, CLAIM, dynamic=True, batch=32)
        assert np.array_equal(y.view(np.uint32), g["y_fused"].view(np.uint32)), (idx, "claims")


def test_executor_checksum_invariant(ctx, oracle):
    # test_executor.cpp:67-87 instance; the expected checksum was produced by the reference
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_executor.npz"))
    want = int(z["checksum"][0])
    for s in STRATS:
        for t in (1, 2, 4, 7):
            y, _ = run(ctx, 200, 200, z["row_ptr"], z["col"], z["vals"], z["x"], s, t, EXACT)
            assert oracle.checksum(y) == want
    for t in (1, 2, 4, 7):
        for fl in (EXACT, EXACT | CLAIM):
            y, _ = run(ctx, 200, 200, z["row_ptr"], z["col"], z["vals"], z["x"], "row", t, fl,
                       dynamic=True, batch=16)
            assert oracle.checksum(y) == want
    # checksum helper of the library agrees with dense.cpp:17-28
    yd = torch.from_numpy(y).cuda()
    assert ctx.checksum(yd) == want


@pytest.mark.parametrize("d", sorted(set(D_POOL + [6, 12, 20, 33, 128, 130, 256, 300, 1024, 1030, 2052])))
def test_every_width_against_oracle(ctx, oracle, d):
    """Per-d instantiation: vector widths, ragged tails, multi-tile and multi-slab d."""
    rng = np.random.default_rng(1000 + d)
    m, n = 157, 93
    rp, col, vals = rand_csr(rng, m, n, 0.15, dup=(d % 2 == 0))
    lens = np.diff(rp.astype(np.int64))
    x = (rng.random((n, d), np.float32) * 2 - 1).astype(np.float32)
    want = oracle.spmm_fused(m, n, rp, col, vals, x)
    unf = oracle.spmm_unfused(m, n, rp, col, vals, x)
    bound = oracle.abs_bound(m, rp, col, vals, x)
    for s in STRATS:
        y, _ = run(ctx, m, n, rp, col, vals, x, s, 5, EXACT)
        assert np.array_equal(y.view(np.uint32), want.view(np.uint32)), (d, s)
        y, p = run(ctx, m, n, rp, col, vals, x, s, 0, 0)
        assert north_star_ok(y, unf, bound), (d, s)
    y, _ = run(ctx, m, n, rp, col, vals, x, "row", 0, EXACT | CLAIM, dynamic=True, batch=7)
    assert np.array_equal(y.view(np.uint32), want.view(np.uint32))


def test_unaligned_base_pointers(ctx, oracle):
    """X/Y not 16-byte aligned -> scalar path, same bits."""
    rng = np.random.default_rng(8)
    m, n, d = 64, 64, 32
    rp, col, vals = rand_csr(rng, m, n, 0.2)
    x = rng.random((n, d), np.float32)
    want = oracle.spmm_fused(m, n, rp, col, vals, x)
    a = ctx.csr_upload(m, n, rp, col, vals)
    p = ctx.plan(a, "nnz", 0, flags=EXACT)
    xb = torch.zeros(n * d + 1, device="cuda")
    yb = torch.zeros(m * d + 1, device="cuda")
    xb[1:] = torch.from_numpy(x).cuda().reshape(-1)
    ctx.spmm_raw(p, a, xb.data_ptr() + 4, n, d, yb.data_ptr() + 4)
    ctx.synchronize()
    assert np.array_equal(yb[1:].reshape(m, d).cpu().numpy().view(np.uint32), want.view(np.uint32))


def test_long_rows_and_skew(ctx, oracle):
    """Rows far longer than a chunk: split across chunks (carry + fix-up) and across the
    groups of a warp; exact mode stays bitwise."""
    rng = np.random.default_rng(11)
    m, n = 300, 5000
    lens = rng.integers(0, 12, size=m)
    lens[7] = 4000
    lens[8] = 0
    lens[150] = 2500
    lens[299] = 3300
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(lens)
    nnz = int(rp[-1])
    col = np.concatenate([np.sort(rng.choice(n, size=l, replace=False)) for l in lens]).astype(np.uint32)
    vals = (rng.random(nnz, np.float32) * 2 - 1).astype(np.float32)
    longest_chain = 0
    for d in (32, 64, 128, 45, 6):
        x = (rng.random((n, d), np.float32) * 2 - 1).astype(np.float32)
        want = oracle.spmm_fused(m, n, rp, col, vals, x)
        unf = oracle.spmm_unfused(m, n, rp, col, vals, x)
        bound = oracle.abs_bound(m, rp, col, vals, x)
        for s in STRATS:
            for t in (0, 1, 5, 64, 999):
                y, _ = run(ctx, m, n, rp, col, vals, x, s, t, EXACT)
                assert np.array_equal(y.view(np.uint32), want.view(np.uint32)), (d, s, t)
                y, p = run(ctx, m, n, rp, col, vals, x, s, t, 0)
                assert north_star_ok(y, unf, bound), (d, s, t)
                cr, cj = p.chunks()
                ch = chain_lengths(m, cr, cj, rp)
                longest_chain = max(longest_chain, int(ch.max()) if ch.size else 0)
                exact_rows = ~split_row_mask(m, cr, cj, rp) & (lens < LONG_SEG)
                assert np.array_equal(y[exact_rows].view(np.uint32), want[exact_rows].view(np.uint32))
                y2, _ = run(ctx, m, n, rp, col, vals, x, s, t, 0)
                assert np.array_equal(y.view(np.uint32), y2.view(np.uint32)), "not deterministic"
    # both fix-up paths ran: short chains (one lane group each) and long ones (one CTA each,
    # more than 16 partials; kLongChain in csrc/spmx_kernels.cuh)
    assert longest_chain > 16


def test_config_siblings_match_reference_checksums(ctx, oracle):
    """Scaled-down siblings of BASELINE configs c1..c5; expected checksums were produced by
    the unmodified reference (tests/golden/make_golden.py)."""
    import os
    from paper_2312_05639_b200 import workloads as W
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_configs.npz"))
    small = {"c1": {}, "c2": {"scale_override": 12}, "c3": {"m_override": 1 << 12},
             "c4": {"scale_override": 12}, "c5": {"scale_override": 11}}
    for name, kw in small.items():
        a, x, spec = W.make_config(name, **kw)
        rp, col, vals = a.numpy()
        assert [a.m, a.n, a.nnz, spec["d"]] == z[name + "_dims"].tolist(), "generator drifted"
        xn = x.numpy()
        unf = oracle.spmm_unfused(a.m, a.n, rp, col, vals, xn)
        assert oracle.checksum(unf) == int(z[name + "_checksum_unfused"][0])
        bound = oracle.abs_bound(a.m, rp, col, vals, xn)
        for s in STRATS:
            y, _ = run(ctx, a.m, a.n, rp, col, vals, xn, s, 0, EXACT)
            assert oracle.checksum(y) == int(z[name + "_checksum_fused"][0]), (name, s)
            y, _ = run(ctx, a.m, a.n, rp, col, vals, xn, s, 0, 0)
            assert north_star_ok(y, unf, bound), (name, s)
        da = ctx.csr_upload(a.m, a.n, rp, col, vals)
        for t in (7, 64):
            assert np.array_equal(ctx.split_nnz(da, t), z[name + f"_nnz{t}"])
            assert np.array_equal(ctx.split_merge(da, t), z[name + f"_merge{t}"])


def test_work_list_is_monotone_and_covers(ctx):
    """Chunk coordinates of every plan are nondecreasing in both components, start at (0, 0),
    end at (m, nnz), and strategy-level ranges are kept as chunk boundaries."""
    from paper_2312_05639_b200 import workloads as W
    for name, kw in (("c2", {"scale_override": 12}), ("c4", {"scale_override": 12}),
                     ("c3", {"m_override": 1 << 12}), ("c1", {})):
        a, _, _ = W.make_config(name, **kw)
        rp, col, vals = a.numpy()
        da = ctx.csr_upload(a.m, a.n, rp, col, vals)
        for s in STRATS:
            for parts in (0, 1, 7, 300):
                for fl in (0, EXACT):
                    p = ctx.plan(da, s, parts, flags=fl)
                    cr, cj = (v.astype(np.int64) for v in p.chunks())
                    assert cr[0] == 0 and cj[0] == 0 and cr[-1] == a.m and cj[-1] == a.nnz
                    assert np.all(np.diff(cr) >= 0) and np.all(np.diff(cj) >= 0), (name, s, parts, fl)
                    # a coordinate (i, j) lies on the merge path: row_ptr[i] <= j <= row_ptr[i+1]
                    inner = cr < a.m
                    assert np.all(cj[inner] >= rp[cr[inner]].astype(np.int64))
                    assert np.all(cj[inner] <= rp[cr[inner] + 1].astype(np.int64))


def test_host_entry_point(ctx, oracle):
    """spmx_spmm_host: the run_spmm-shaped call with host buffers."""
    rng = np.random.default_rng(21)
    m, n, d = 500, 400, 64
    rp, col, vals = rand_csr(rng, m, n, 0.05)
    x = rng.random((n, d), np.float32)
    want = oracle.spmm_fused(m, n, rp, col, vals, x)
    for s in STRATS:
        y, times = ctx.spmm_host(m, n, rp, col, vals, x, strategy=s, flags=EXACT)
        assert np.array_equal(y.view(np.uint32), want.view(np.uint32))
        assert times["total"] > 0
    from paper_2312_05639_b200.binding import SpmxInvalidArgument
    with pytest.raises(SpmxInvalidArgument):
        ctx.spmm_host(m, n, rp, col, vals, rng.random((n + 1, d), np.float32))
    with pytest.raises(SpmxInvalidArgument):
        ctx.spmm_host(m, n, rp, col, vals, x, strategy="nnz", dynamic=True)


def test_device_reference_and_error_metric(ctx, oracle):
    """spmx_spmm_reference (Alg. 1 on the device, used by RunConfig.verify) is bitwise the
    reference's unfused loop; spmx_max_relative_error equals executor.cpp:27-34."""
    rng = np.random.default_rng(31)
    m, n, d = 300, 200, 45
    rp, col, vals = rand_csr(rng, m, n, 0.08)
    x = (rng.random((n, d), np.float32) * 2 - 1).astype(np.float32)
    a = ctx.csr_upload(m, n, rp, col, vals)
    xd = torch.from_numpy(x).cuda()
    yr = torch.empty(m, d, device="cuda")
    ctx.spmm_reference(a, xd, yr)
    ctx.synchronize()
    want = oracle.spmm_unfused(m, n, rp, col, vals, x)
    assert np.array_equal(yr.cpu().numpy().view(np.uint32), want.view(np.uint32))
    p = ctx.plan(a, "merge")
    y = torch.empty(m, d, device="cuda")
    ctx.spmm(p, a, xd, y)
    ctx.synchronize()
    got = ctx.max_relative_error(y, yr)
    assert got == oracle.max_relative_error(y.cpu().numpy(), want)


@pytest.mark.parametrize("d", [1, 20, 45, 48, 96, 100, 256, 1000])
def test_runtime_instantiation_per_width(ctx, oracle, d):
    """SPMX_JIT_WIDTH: the kernel is compiled for exactly this d at run time (NVRTC) — the GPU
    counterpart of the reference's emit(). Same bits as the precompiled path."""
    from paper_2312_05639_b200.binding import JIT_WIDTH, Lib
    rng = np.random.default_rng(500 + d)
    m, n = 211, 137
    rp, col, vals = rand_csr(rng, m, n, 0.12)
    x = (rng.random((n, d), np.float32) * 2 - 1).astype(np.float32)
    want = oracle.spmm_fused(m, n, rp, col, vals, x)
    unf = oracle.spmm_unfused(m, n, rp, col, vals, x)
    bound = oracle.abs_bound(m, rp, col, vals, x)
    before = Lib.get().jit_stats()
    for s in STRATS:
        y, _ = run(ctx, m, n, rp, col, vals, x, s, 5, EXACT | JIT_WIDTH)
        assert np.array_equal(y.view(np.uint32), want.view(np.uint32)), (d, s)
        y, _ = run(ctx, m, n, rp, col, vals, x, s, 0, JIT_WIDTH)
        assert north_star_ok(y, unf, bound), (d, s)
    after = Lib.get().jit_stats()
    assert after[0] >= before[0] and after[0] >= 1   # compiled once per (device, d), then cached
    assert after[0] - before[0] <= 1


def test_no_fixup_without_cut_rows_and_tail_taper(ctx):
    """A plan in which no row is cut (regular matrix, rows shorter than LONG_SEG, row-granular
    strategy boundaries) runs as ONE kernel launch per SpMM: no carry buffer, no fix-up. The
    chunks at the end of the work list are smaller than those in its body (tail taper: the SMs
    run dry together), and the list still covers the merge path exactly."""
    from paper_2312_05639_b200 import workloads as W
    from paper_2312_05639_b200.binding import Lib
    a, x, spec = W.make_config("c3", device="cuda", m_override=1 << 17)
    rp = a.numpy()[0]
    da = ctx.csr_wrap(a)
    y = torch.empty(a.m, spec["d"], device="cuda")
    for s, max_launches in (("row", 1), ("nnz", 1), ("merge", 2)):
        p = ctx.plan(da, s, 0)
        ctx.spmm(p, da, x, y)
        ctx.synchronize()
        before = Lib.get().launch_count()
        ctx.spmm(p, da, x, y)
        ctx.synchronize()
        assert 1 <= Lib.get().launch_count() - before <= max_launches, s
        cr, cj = (v.astype(np.int64) for v in p.chunks())
        assert cr[0] == 0 and cj[0] == 0 and cr[-1] == a.m and cj[-1] == a.nnz
        items = np.diff(cr) + np.diff(cj)
        assert items.min() >= 1 and items.max() <= 256 + LONG_SEG
        body, tail = items[: len(items) // 2], items[-len(items) // 50:]
        assert np.median(tail) <= 0.3 * np.median(body), (s, np.median(tail), np.median(body))
        if s != "merge":
            assert not split_row_mask(a.m, cr, cj, rp).any()
        p.close()
    da.close()


def test_row_shards_on_one_device_concatenate_to_the_whole(ctx, oracle):
    """The multi-GPU layout run on one device: A cut into the G ranges of
    split_nnz(A, G) with rebased row_ptr, X shared, each shard multiplied on its own; the
    concatenated Y equals the unsharded result bit for bit in exact mode (rows are never cut
    there) and within the north_star bound in default mode."""
    from paper_2312_05639_b200 import workloads as W
    a, x, spec = W.make_config("c5", device="cuda", scale_override=13)
    rp, col, vals = a.numpy()
    xn = x.cpu().numpy()
    want = oracle.spmm_fused(a.m, a.n, rp, col, vals, xn)
    unf = oracle.spmm_unfused(a.m, a.n, rp, col, vals, xn)
    bound = oracle.abs_bound(a.m, rp, col, vals, xn)
    da = ctx.csr_wrap(a)
    for G in (2, 4, 8):
        ranges = ctx.split_nnz(da, G)
        assert np.array_equal(ranges, oracle.split_nnz(rp, G))
        assert int(ranges[0, 0]) == 0 and int(ranges[-1, 1]) == a.m
        for flags in (EXACT, 0):
            parts = []
            for b, e in ranges:
                sh = a.row_slice(int(b), int(e))
                ds = ctx.csr_wrap(sh)
                y = torch.full((sh.m, spec["d"]), float("nan"), device="cuda")
                p = ctx.plan(ds, "nnz", 0, flags=flags)
                ctx.spmm(p, ds, x, y)
                ctx.synchronize()
                parts.append(y.cpu().numpy())
                p.close(); ds.close()
            got = np.concatenate(parts, axis=0)
            if flags == EXACT:
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), G
            else:
                assert north_star_ok(got, unf, bound), G
    da.close()


def test_golden_instances_through_the_long_row_kernel(ctx, golden_instances, monkeypatch):
    """SPMX_LONG_ROW=8: nearly every row of the reference's acceptance instances is 'long', so the
    exact-order plans send them through spmm_long_row_kernel (every width of the reference's d
    pool, scalar and float4 pieces, ragged tiles). Bitwise equal to the reference's run_spmm."""
    monkeypatch.setenv("SPMX_LONG_ROW", "8")
    for idx, g in enumerate(golden_instances):
        m, n, nnz, d = (int(v) for v in g["dims"])
        for s in STRATS:
            for t in (0, 3):
                y, p = run(ctx, m, n, g["row_ptr"], g["col"], g["vals"], g["x"], s, t, EXACT)
                assert np.array_equal(y.view(np.uint32), g["y_fused"].view(np.uint32)), (idx, s, t, d)
        y, _ = run(ctx, m, n, g["row_ptr"], g["col"], g["vals"], g["x"], "row", 0, EXACT, dynamic=True)
        assert np.array_equal(y.view(np.uint32), g["y_fused"].view(np.uint32)), (idx, "dynamic")
