"""The library's multi-GPU driver (spmx_mg_*, include/spmx_b200.h) on ONE device.

This run has one GPU, so the driver is exercised the two ways one GPU allows:
  * world = 1 through the real NCCL path (ncclCommInitAll / ncclCommInitRank on one device:
    the broadcast of X, the all-gather-v of Y and the statistics all-reduce are NCCL calls);
  * G = 2, 4, 8 row blocks placed on that one GPU (n_shards > world): the same sharding,
    planning, launching and gathering code a G-GPU node runs, every shard on its own CSR with
    a rebased row_ptr — the layout SURVEY section 8e asks to be tested this way.
Parity: shard ranges bit-exact with split_nnz / split_merge of the oracle
(partition.cpp:35-51, 69-84); concatenated Y bitwise equal to the oracle's fused result in
exact-order mode, within the north_star bound in default mode.
"""
import numpy as np
import pytest
import torch

from helpers import north_star_ok

pytestmark = pytest.mark.gpu

EXACT = 1


@pytest.fixture(scope="module")
def small_c5():
    from paper_2312_05639_b200 import workloads as W
    a, x, spec = W.make_config("c5", device="cuda", scale_override=13)
    torch.cuda.synchronize()
    return a, x, spec


@pytest.fixture(scope="module")
def truth(small_c5, oracle):
    a, x, spec = small_c5
    rp, col, vals = a.numpy()
    xn = x.cpu().numpy()
    return dict(rp=rp, col=col, vals=vals, xn=xn,
                fused=oracle.spmm_fused(a.m, a.n, rp, col, vals, xn),
                unf=oracle.spmm_unfused(a.m, a.n, rp, col, vals, xn),
                bound=oracle.abs_bound(a.m, rp, col, vals, xn))


def _y_full(ctx, mg, m, d):
    """The driver's all-gathered Y (device buffer) copied out through the C ABI."""
    out = np.empty((m, d), np.float32)
    mg.synchronize()
    ctx.L.check(ctx.L.lib.spmx_d2h(ctx.h, out.ctypes.data, mg.y_full_ptr(0), out.nbytes))
    ctx.synchronize()
    return out


@pytest.mark.parametrize("by", ["nnz", "merge"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_shards_on_one_gpu_concatenate_to_the_whole(ctx, small_c5, truth, oracle, G, by):
    from paper_2312_05639_b200.binding import MultiGpu
    a, x, spec = small_c5
    d = spec["d"]
    mg = MultiGpu([0], n_shards=G)
    info = mg.info()
    assert info["world"] == 1 and info["shards"] == G and info["nccl_version"] >= 20000
    ranges = mg.shard_device(a, by=by)
    want_ranges = (oracle.split_nnz if by == "nnz" else oracle.split_merge)(truth["rp"], G)
    assert np.array_equal(ranges, want_ranges)
    shards = mg.local_shards()
    assert [s["shard"] for s in shards] == list(range(G))
    assert sum(s["nnz"] for s in shards) == a.nnz
    for s, (b, e) in zip(shards, want_ranges):
        assert (s["row_begin"], s["row_end"]) == (int(b), int(e))
        assert s["nnz"] == int(truth["rp"][int(e)]) - int(truth["rp"][int(b)])
    bc = mg.broadcast_x_device([x], root=0)
    assert bc >= 0.0
    for strat in ("row", "nnz", "merge"):
        for flags in (EXACT, 0):
            mg.plan(strat, 0, flags=flags)
            ms, per = mg.spmm(steps=2, per_shard=True)
            assert ms > 0 and len(per) == G and all(t > 0 for t in per)
            got = mg.download_y(m=a.m)
            if flags == EXACT:
                assert np.array_equal(got.view(np.uint32), truth["fused"].view(np.uint32)), (G, strat)
            else:
                assert north_star_ok(got, truth["unf"], truth["bound"]), (G, strat)
    # all-gather-v of the row-sharded Y (one ncclBroadcast per shard, unequal row counts)
    ag = mg.allgather_y()
    assert ag >= 0.0
    full = _y_full(ctx, mg, a.m, d)
    assert np.array_equal(full.view(np.uint32), got.view(np.uint32))
    # statistics all-reduce over the communicator
    assert mg.allreduce([3.5, 7.0], "max") == [3.5, 7.0]
    assert mg.allreduce([a.nnz], "sum") == [float(a.nnz)]
    mg.close()


def test_shard_host_and_broadcast_from_host(small_c5, truth, oracle):
    """The host-array entry points (CsrMatrix fields straight from the reference's structs)."""
    from paper_2312_05639_b200.binding import MultiGpu
    a, x, spec = small_c5
    mg = MultiGpu([0], n_shards=3)
    ranges = mg.shard_host(a.m, a.n, truth["rp"], truth["col"], truth["vals"], by="nnz")
    assert np.array_equal(ranges, oracle.split_nnz(truth["rp"], 3))
    h2d, bc = mg.broadcast_x_host(truth["xn"], root=0)
    assert h2d > 0
    mg.plan("merge", 0, flags=EXACT)
    mg.spmm()
    got = mg.download_y(m=a.m)
    assert np.array_equal(got.view(np.uint32), truth["fused"].view(np.uint32))
    # re-sharding replaces the previous shards; X stays
    ranges = mg.shard_host(a.m, a.n, truth["rp"], truth["col"], truth["vals"], by="merge")
    assert np.array_equal(ranges, oracle.split_merge(truth["rp"], 3))
    mg.plan("nnz", 0, flags=EXACT)
    mg.spmm()
    assert np.array_equal(mg.download_y(m=a.m).view(np.uint32), truth["fused"].view(np.uint32))
    mg.close()


def test_rank_mode_with_unique_id(small_c5, truth):
    """One process per GPU (the torchrun form): world = 1 communicator from a unique id."""
    from paper_2312_05639_b200.binding import MultiGpu
    a, x, spec = small_c5
    uid = MultiGpu.unique_id()
    assert len(uid) == 128
    stream = torch.cuda.current_stream().cuda_stream
    mg = MultiGpu.for_rank(0, 0, 1, uid, n_shards=2, stream=stream)
    assert mg.info()["nccl_version"] >= 20000
    mg.shard_device(a, by="nnz")
    mg.broadcast_x_device([x], 0)
    mg.plan("merge", 0, flags=EXACT)
    mg.spmm(steps=3)
    assert np.array_equal(mg.download_y(m=a.m).view(np.uint32), truth["fused"].view(np.uint32))
    mg.close()


def test_rank_code_path_without_communicator(small_c5, truth):
    """Rank r of a 2-rank world, built without a communicator: only the shard / plan / spmm
    calls work. Both ranks' row blocks, computed one after the other on this GPU, tile Y."""
    from paper_2312_05639_b200.binding import MultiGpu, SpmxRuntimeError
    a, x, spec = small_c5
    y = np.full((a.m, spec["d"]), np.nan, np.float32)
    rows = []
    for rank in range(2):
        mg = MultiGpu.for_rank(0, rank, 2, None, n_shards=4)
        assert mg.info()["nccl_version"] == 0
        mg.shard_device(a, by="nnz")
        loc = mg.local_shards()
        assert [s["shard"] for s in loc] == [2 * rank, 2 * rank + 1]
        with pytest.raises(SpmxRuntimeError, match="communicator"):
            mg.broadcast_x_device([x], 0)
        mg.close()
        rows.append((loc[0]["row_begin"], loc[-1]["row_end"]))
    assert rows[0][0] == 0 and rows[0][1] == rows[1][0] and rows[1][1] == a.m


def test_errors(small_c5):
    from paper_2312_05639_b200.binding import (MultiGpu, SpmxInvalidArgument, SpmxLogicError)
    a, x, spec = small_c5
    with pytest.raises(SpmxInvalidArgument):
        MultiGpu([0, 0])          # the same device twice
    with pytest.raises(SpmxInvalidArgument):
        MultiGpu([99])            # no such device
    with pytest.raises(SpmxInvalidArgument):
        MultiGpu.for_rank(0, 2, 2, None)
    mg = MultiGpu([0], n_shards=2)
    with pytest.raises(SpmxLogicError):
        mg.plan("merge")          # nothing sharded yet
    mg.shard_device(a)
    mg.set_x_shape(a.n, spec["d"])
    with pytest.raises(SpmxLogicError):
        mg.spmm()                 # no X yet
    mg.broadcast_x_device([x], 0)
    with pytest.raises(SpmxLogicError):
        mg.spmm()                 # no plan yet
    with pytest.raises(SpmxInvalidArgument, match="dynamic dispatch pairs with row-split only"):
        mg.plan("merge", dynamic=True)
    with pytest.raises(SpmxInvalidArgument, match="A.n != X.rows"):
        mg.broadcast_x_device([x[:-1]], 0)
    # an invalid matrix is rejected per shard (validate_csr on the device)
    bad = a.col.clone()
    bad[a.nnz // 2] = a.n + 5
    torch.cuda.synchronize()
    import types
    a_bad = types.SimpleNamespace(m=a.m, n=a.n, nnz=a.nnz, row_ptr=a.row_ptr, col=bad, vals=a.vals)
    with pytest.raises(SpmxInvalidArgument, match="column index out of range"):
        mg.shard_device(a_bad)
    mg.close()


@pytest.mark.parametrize("G", [1, 3])
def test_hot_row_copy_keeps_results_bitwise(small_c5, truth, oracle, monkeypatch, G):
    """With driver-owned X replicas every rank keeps a compact copy of its hottest X rows behind
    X, remaps those columns of its shards to the copy and puts an L2 window over it
    (SPMX_MG_HOT_ROWS; forced on here for a small matrix). Values and order are untouched, so
    exact-order results stay bitwise equal to the oracle — through the host and the device
    entry, after switching to borrowed X buffers (remap undone) and back, and across a re-shard."""
    from paper_2312_05639_b200.binding import MultiGpu
    monkeypatch.setenv("SPMX_MG_HOT_ROWS", "300")
    monkeypatch.setenv("SPMX_MG_HOT_MIN_MB", "0")
    a, x, spec = small_c5
    want = truth["fused"].view(np.uint32)
    mg = MultiGpu([0], n_shards=G)
    mg.shard_device(a, by="nnz")

    def check(tag):
        for strat, flags in (("merge", EXACT), ("row", EXACT), ("nnz", 0)):
            mg.plan(strat, 0, flags=flags)
            mg.spmm(steps=2)
            got = mg.download_y(m=a.m)
            if flags:
                assert np.array_equal(got.view(np.uint32), want), (tag, strat)
            else:
                assert north_star_ok(got, truth["unf"], truth["bound"]), (tag, strat)

    mg.broadcast_x_host(truth["xn"], root=0)          # owned: hot copy + remap + window
    check("host")
    mg.broadcast_x_device([x], root=0)                # borrowed: remap undone
    check("borrowed")
    cp, bc = mg.broadcast_x_from_device(x, root=0)    # owned again, X from the device
    assert cp > 0
    check("from_device")
    mg.shard_host(a.m, a.n, truth["rp"], truth["col"], truth["vals"], by="merge")  # re-shard, X stays
    check("reshard")
    mg.allgather_y()
    mg.close()
