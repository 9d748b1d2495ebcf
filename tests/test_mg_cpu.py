"""CPU suite: the host logic of the N > 1 path with world_size 2 over gloo (no GPU here).

What can be checked without a device is exactly what bench.py's torchrun form does on the
host side before any GPU work: rank 0 makes the 128-byte communicator id and hands it to the
other ranks through a gloo broadcast; every rank evaluates the same split of A's rows, asks the
library which shards it owns (spmx_mg_shard_owner, a pure host function of the C ABI) and
computes only those row blocks; the blocks tile Y. The oracle stands in for the device kernel
(this test is about ownership and tiling, not arithmetic), and the driver itself must refuse to
come up without a CUDA device — there is no CPU fallback."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, n_shards):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.pyoracle import Oracle
    from paper_2312_05639_b200 import workloads as W
    from paper_2312_05639_b200.binding import Lib
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = Lib.get().lib
    # the id hand-over of bench.py (here a stand-in token: ncclGetUniqueId needs the device)
    box = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    assert box[0] == bytes(range(128))
    orc = Oracle()
    a, x, spec = W.make_config("c2", scale_override=11)
    rp, col, vals = a.numpy()
    ranges = orc.split_nnz(rp, n_shards)        # the reference's split_nnz(A, G)
    mine = [g for g in range(n_shards) if lib.spmx_mg_shard_owner(n_shards, world, g) == rank]
    rows = []
    for g in mine:
        b, e = int(ranges[g, 0]), int(ranges[g, 1])
        sh = a.row_slice(b, e)                  # rebased row_ptr, like the driver's shards
        srp, scol, svals = sh.numpy()
        y = orc.spmm_fused(sh.m, sh.n, srp, scol, svals, x.numpy(), threads=1)
        rows.append((b, e, y))
    gathered = [None] * world
    dist.all_gather_object(gathered, [(b, e, y) for b, e, y in rows])
    y_full = np.full((a.m, spec["d"]), np.nan, np.float32)
    for part in gathered:
        for b, e, y in part:
            y_full[b:e] = y
    np.save(os.path.join(out_dir, f"y{rank}.npy"), y_full)
    np.save(os.path.join(out_dir, f"mine{rank}.npy"), np.asarray(mine, np.int64))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_shards", [2, 5])
def test_two_ranks_own_and_tile_the_row_blocks(tmp_path, oracle, n_shards):
    from paper_2312_05639_b200 import workloads as W
    world, port = 2, _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path), n_shards), nprocs=world, join=True)
    a, x, spec = W.make_config("c2", scale_override=11)
    rp, col, vals = a.numpy()
    want = oracle.spmm_fused(a.m, a.n, rp, col, vals, x.numpy())
    owned = [np.load(tmp_path / f"mine{r}.npy").tolist() for r in range(world)]
    assert sorted(owned[0] + owned[1]) == list(range(n_shards))      # every shard has one owner
    assert owned[0] == sorted(owned[0]) and max(owned[0]) < min(owned[1])  # contiguous per rank
    for r in range(world):
        got = np.load(tmp_path / f"y{r}.npy")
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_shard_owner_is_balanced_and_monotone():
    from paper_2312_05639_b200.binding import Lib
    lib = Lib.get().lib
    for world in (1, 2, 3, 8):
        for n_shards in (world, world + 1, 3 * world, 64):
            owners = [lib.spmx_mg_shard_owner(n_shards, world, g) for g in range(n_shards)]
            assert owners == sorted(owners) and owners[0] == 0 and owners[-1] == world - 1
            counts = np.bincount(owners, minlength=world)
            assert counts.max() - counts.min() <= 1
    assert lib.spmx_mg_shard_owner(4, 2, 4) == -1 and lib.spmx_mg_shard_owner(0, 1, 0) == -1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the behaviour without a device")
def test_driver_refuses_to_start_without_a_device():
    from paper_2312_05639_b200.binding import MultiGpu, SpmxRuntimeError
    with pytest.raises(SpmxRuntimeError, match="no CPU fallback|NCCL"):
        MultiGpu([0])
    with pytest.raises(SpmxRuntimeError, match="no CPU fallback"):
        MultiGpu.for_rank(0, 0, 2, None)
