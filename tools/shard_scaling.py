"""Per-shard kernel times of the multi-GPU layout, measured one shard at a time on ONE GPU.

The multi-GPU path has no data-path collective: rank g owns the g-th
range of split_nnz(A, G) with a rebased row_ptr, X is replicated, Y stays row-sharded. The
step time at G GPUs is therefore max over ranks of (that rank's SpMM kernel time on its
shard), and each of those is a single-GPU quantity: this tool builds every shard of
G = 1, 2, 4, 8 on one device, times its SpMM alone, and reports max over shards, the
aggregate GFLOP/s that implies, and the nnz balance. It is a projection from real per-shard
measurements, not a multi-GPU run (the X broadcast and the optional Y all-gather are not in
it; bench.py --gpus N times those separately when N GPUs exist).

    python tools/shard_scaling.py [c5] [--scale N] [--iters K] [--json out.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_05639_b200 import workloads as W  # noqa: E402
from paper_2312_05639_b200.binding import Context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c5")
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--iters", type=int, default=7)
    ap.add_argument("--strategy", default="nnz")
    ap.add_argument("--shard-by", default="nnz", choices=("nnz", "merge"),
                    help="rank-level split: split_nnz(A, G) (north_star) or split_merge(A, G) (rows + nonzeros)")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    peak = 6551.0
    try:
        peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    ctx = Context.on_torch_stream(0)
    a, x, spec = W.make_config(args.config, device="cuda", scale_override=args.scale)
    d = spec["d"]
    da = ctx.csr_wrap(a)
    rows = []
    base = None
    for G in (1, 2, 4, 8):
        ranges = (ctx.split_nnz if args.shard_by == "nnz" else ctx.split_merge)(da, G)
        times, nnzs = [], []
        for b, e in ranges:
            b, e = int(b), int(e)
            sh = a.row_slice(b, e)
            ds = ctx.csr_wrap(sh)
            y = torch.empty(sh.m, d, device="cuda")
            p = ctx.plan(ds, args.strategy, 0)
            for _ in range(2):
                ctx.spmm(p, ds, x, y)
            ts = [ctx.spmm(p, ds, x, y, timed=True) for _ in range(args.iters)]
            times.append(float(np.median(ts)))
            nnzs.append(sh.nnz)
            p.close(); ds.close()
            del y, sh
        step = max(times)
        gf = 2.0 * a.nnz * d / step / 1e6
        byts = W.algorithmic_bytes(a.m, a.n, a.nnz, d)
        byts_repl = byts + (G - 1) * 4 * a.n * d
        if base is None:
            base = step
        row = {"gpus": G, "step_ms": step, "shard_ms": times, "gflops": gf,
               "speedup_vs_1": base / step, "efficiency": base / step / G,
               "nnz_imbalance": max(nnzs) / (sum(nnzs) / G),
               "frac_of_G_x_peak": byts / step / 1e6 / (peak * G),
               "frac_replicated_x": byts_repl / step / 1e6 / (peak * G)}
        rows.append(row)
        print(f"G={G}: step {step:8.3f} ms (shards {' '.join(f'{t:.3f}' for t in times)})  "
              f"{gf:9.0f} GFLOP/s  speed-up {row['speedup_vs_1']:.2f}  efficiency {row['efficiency']:.2f}  "
              f"nnz imbalance {row['nnz_imbalance']:.3f}  frac {row['frac_of_G_x_peak']:.3f} "
              f"(X per rank: {row['frac_replicated_x']:.3f})", flush=True)
    if args.json:
        json.dump({"config": args.config, "shard_by": args.shard_by, "m": a.m, "nnz": a.nnz, "d": d, "strategy": args.strategy,
                   "how": "per-shard SpMM kernel time measured one shard at a time on one B200; step = max over shards",
                   "rows": rows}, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
