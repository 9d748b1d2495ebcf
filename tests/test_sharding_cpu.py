"""CPU suite: the multi-GPU host logic with world_size 2 over gloo. Each rank owns an
nnz-balanced row block (split_nnz at rank granularity), receives X by broadcast, computes
its block (here with the oracle standing in for the device kernel — this test is about the
sharding/collective plumbing, not the arithmetic) and the gathered Y must equal the
single-rank result bitwise."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.pyoracle import Oracle
    from paper_2312_05639_b200 import sharding, workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    a, x, spec = W.make_config("c2", scale_override=11)
    rp, col, vals = a.numpy()
    ranges = orc.split_nnz(rp, world)           # the reference's split_nnz(A, G)
    shard, (b, e) = sharding.local_shard(a, ranges, rank)
    if rank != 0:
        x = torch.zeros_like(x)                 # only rank 0 holds X before the broadcast
    sharding.broadcast_x(x, 0)
    srp, scol, svals = shard.numpy()
    y_local = torch.from_numpy(orc.spmm_fused(shard.m, shard.n, srp, scol, svals, x.numpy(), threads=1))
    y_full = sharding.allgather_rows(y_local, ranges)
    t = sharding.max_over_ranks(float(rank + 1), "cpu")
    nnz_total = sharding.sum_over_ranks(float(shard.nnz), "cpu")
    np.save(os.path.join(out_dir, f"y{rank}.npy"), y_full.numpy())
    np.save(os.path.join(out_dir, f"meta{rank}.npy"), np.array([t, nnz_total, b, e, shard.nnz]))
    dist.destroy_process_group()


def test_two_rank_row_shards_gloo(tmp_path, oracle):
    from paper_2312_05639_b200 import workloads as W
    world, port = 2, _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    a, x, spec = W.make_config("c2", scale_override=11)
    rp, col, vals = a.numpy()
    want = oracle.spmm_fused(a.m, a.n, rp, col, vals, x.numpy())
    metas = [np.load(tmp_path / f"meta{r}.npy") for r in range(world)]
    for r in range(world):
        got = np.load(tmp_path / f"y{r}.npy")
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
        assert metas[r][0] == world and metas[r][1] == a.nnz
    # shards are contiguous, cover all rows, and are nnz-balanced to within the longest row
    assert metas[0][2] == 0 and metas[0][3] == metas[1][2] and metas[1][3] == a.m
    max_row = int(np.diff(rp.astype(np.int64)).max())
    assert abs(metas[0][4] - a.nnz / 2) <= max_row


def test_allgather_rows_unequal_shards_single_process():
    """Degenerate world of 1 still pads/unpads correctly."""
    import os
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    from paper_2312_05639_b200 import sharding
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        y = torch.arange(12, dtype=torch.float32).reshape(3, 4)
        assert torch.equal(sharding.allgather_rows(y, np.array([[0, 3]], np.uint64)), y)
    finally:
        dist.destroy_process_group()
