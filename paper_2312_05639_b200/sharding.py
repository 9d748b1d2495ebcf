"""Multi-GPU driver pieces: one process per GPU, A sharded into nnz-balanced row blocks
(the reference's split_nnz(A, G), src/partition.cpp:35-51, applied at rank granularity),
X replicated by one NCCL broadcast, Y kept row-sharded, optional all-gather of Y.

Row blocks are independent (single writer per output row, reference SPEC.md:439), so
the data path has no collective: the only exchanges are the one-off broadcast of X and
the optional gather of Y, both timed separately from the SpMM. Works with any
torch.distributed backend (nccl on GPUs; gloo on CPU tensors for the host-logic tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_ranges_to_list(ranges) -> list[tuple[int, int]]:
    return [(int(b), int(e)) for b, e in ranges]


def local_shard(csr, ranges, rank: int):
    """Rows [b, e) of `csr` for this rank, with a rebased row_ptr (workloads.Csr.row_slice)."""
    b, e = shard_ranges_to_list(ranges)[rank]
    return csr.row_slice(b, e), (b, e)


def broadcast_x(x: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """One broadcast of the dense right-hand side (in place)."""
    dist.broadcast(x, src=src, group=group)
    return x


def allgather_rows(y_local: torch.Tensor, ranges, group=None) -> torch.Tensor:
    """All-gather of row-sharded Y with unequal row counts: pad to the largest shard,
    all_gather, then drop the padding. Returns the full M x d matrix on every rank."""
    rl = shard_ranges_to_list(ranges)
    world = dist.get_world_size(group)
    assert len(rl) == world
    d = y_local.shape[1]
    max_rows = max(e - b for b, e in rl)
    pad = torch.zeros(max_rows, d, dtype=y_local.dtype, device=y_local.device)
    pad[: y_local.shape[0]] = y_local
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return torch.cat([o[: e - b] for o, (b, e) in zip(out, rl)], dim=0)


def max_over_ranks(value: float, device, group=None) -> float:
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value: float, device, group=None) -> float:
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())
