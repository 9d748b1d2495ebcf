"""Experiment: what do contiguous hot X rows + an L2 persisting window buy?

The matrix is relabelled by column degree (column with the most nonzeros -> index 0, ...) and X
is permuted the same way, so Y is unchanged and the hottest X rows are one contiguous block.
Timed: original labelling; relabelled; relabelled + cudaAccessPolicyWindow over the first H rows
(hit ratio swept). An upper bound for any scheme that keeps hot rows resident in L2.

    python tools/exp_hot_window.py c5 [--scale N] [--iters K]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_05639_b200 import workloads as W  # noqa: E402
from paper_2312_05639_b200.binding import Context  # noqa: E402


def timed(ctx, p, da, x, y, iters):
    for _ in range(3):
        ctx.spmm(p, da, x, y)
    ts = [ctx.spmm(p, da, x, y, timed=True) for _ in range(iters)]
    return float(np.median(ts)), float(min(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c5")
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--strategy", default="merge")
    ap.add_argument("--profile", action="store_true",
                    help="ncu mode: two launches each of original / relabelled / relabelled + 50k-row window")
    args = ap.parse_args()
    ctx = Context.on_torch_stream(0)
    a, x, spec = W.make_config(args.config, device="cuda", scale_override=args.scale)
    d = spec["d"]
    y = torch.empty(a.m, d, device="cuda")
    byts = W.algorithmic_bytes(a.m, a.n, a.nnz, d)
    print(f"{args.config}: m={a.m} nnz={a.nnz} d={d} X={a.n*d*4/1e9:.2f} GB algorithmic={byts/1e9:.2f} GB", flush=True)
    da = ctx.csr_wrap(a)
    p = ctx.plan(da, args.strategy, 0)
    if args.profile:
        ctx.spmm(p, da, x, y); ctx.spmm(p, da, x, y); ctx.synchronize()
    ms, mn = (0.0, 0.0) if args.profile else timed(ctx, p, da, x, y, args.iters)
    print(f"  original labelling            {ms*1e3:9.1f} us (min {mn*1e3:.1f})", flush=True)
    y0 = y.clone()
    p.close(); da.close()
    # relabel by degree
    col64 = a.col.long() & 0xFFFFFFFF
    deg = torch.bincount(col64, minlength=a.n)
    order = torch.argsort(deg, descending=True, stable=True)       # new index -> old column
    rank = torch.empty_like(order)
    rank[order] = torch.arange(a.n, device="cuda")                   # old column -> new index
    cum = torch.cumsum(deg[order].double(), 0) / a.nnz
    for h in (50_000, 100_000, 150_000, 200_000, 250_000):
        if h < a.n:
            print(f"    hottest {h} X rows ({h*d*4/1e6:.0f} MB) hold {float(cum[h-1])*100:.1f} % of the nonzeros")
    a2 = W.Csr(a.m, a.n, a.nnz, a.row_ptr, rank[col64].to(torch.int32), a.vals)
    x2 = x[order].contiguous()
    del col64, deg, rank, cum
    torch.cuda.synchronize()
    da = ctx.csr_wrap(a2)
    p = ctx.plan(da, args.strategy, 0)
    if args.profile:
        ctx.spmm(p, da, x2, y); ctx.spmm(p, da, x2, y); ctx.synchronize()
        win = ctx.l2_window(x2.data_ptr(), 50_000 * d * 4, 1.0)
        ctx.spmm(p, da, x2, y); ctx.spmm(p, da, x2, y); ctx.synchronize()
        ctx.l2_window(0, 0)
        print(f"  profile mode: launches 1-2 original, 3-4 relabelled, 5-6 relabelled + {win/1e6:.1f} MB window")
        return
    ms, mn = timed(ctx, p, da, x2, y, args.iters)
    print(f"  relabelled by degree          {ms*1e3:9.1f} us (min {mn*1e3:.1f})  max|dY|={float((y-y0).abs().max()):.2e}", flush=True)
    for rows in (50_000, 100_000, 150_000, 250_000):
        for hit in (1.0, 0.6):
            nbytes = min(rows, a.n) * d * 4
            win = ctx.l2_window(x2.data_ptr(), nbytes, hit)
            ms, mn = timed(ctx, p, da, x2, y, args.iters)
            print(f"  + window {rows:7d} rows ({win/1e6:6.1f} MB set) hit {hit:.1f}: {ms*1e3:9.1f} us (min {mn*1e3:.1f})", flush=True)
    ctx.l2_window(0, 0)
    ms, mn = timed(ctx, p, da, x2, y, args.iters)
    print(f"  window removed                {ms*1e3:9.1f} us (min {mn*1e3:.1f})", flush=True)


if __name__ == "__main__":
    main()
