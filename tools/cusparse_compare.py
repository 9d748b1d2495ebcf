"""Context for the roofline fraction: the same SpMM through NVIDIA's library on the same GPU and
the same arrays (torch.sparse.mm on a CSR tensor = cuSPARSE SpMM, row-major dense operands)
beside this repo's kernel. A comparison aid only: nothing in the product calls cuSPARSE.

    python tools/cusparse_compare.py c2 c4 [c3 c5] [--iters 10]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_05639_b200 import workloads as W  # noqa: E402
from paper_2312_05639_b200.binding import Context  # noqa: E402


def timed(fn, iters):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(min(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2"])
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    ctx = Context.on_torch_stream(0)
    for name in args.configs:
        a, x, spec = W.make_config(name, device="cuda")
        d = spec["d"]
        byts = W.algorithmic_bytes(a.m, a.n, a.nnz, d)
        y = torch.empty(a.m, d, device="cuda")
        da = ctx.csr_wrap(a)
        p = ctx.plan(da, "merge", 0)
        ours, ours_min = timed(lambda: ctx.spmm(p, da, x, y), args.iters)
        # cuSPARSE takes signed indices of one type: int32 row pointers and columns (every config fits)
        assert a.nnz < 2**31 and a.n < 2**31
        crow = a.row_ptr.to(torch.int32)
        ccol = a.col.to(torch.int32)
        A = torch.sparse_csr_tensor(crow, ccol, a.vals, size=(a.m, a.n))
        yl = torch.sparse.mm(A, x)
        lib_ms, lib_min = timed(lambda: torch.sparse.mm(A, x), args.iters)
        err = ((yl - y).abs().max() / yl.abs().max().clamp_min(1e-30)).item()
        print(f"{name}: m={a.m} nnz={a.nnz} d={d}  this repo {ours*1e3:9.1f} us (min {ours_min*1e3:.1f})   "
              f"cuSPARSE via torch.sparse.mm {lib_ms*1e3:9.1f} us (min {lib_min*1e3:.1f}, includes the output "
              f"allocation)   ratio {lib_ms/ours:.2f}x   max |diff| / max |y| = {err:.2e}   "
              f"algorithmic GB/s: {byts/ours/1e6:.0f} vs {byts/lib_ms/1e6:.0f}", flush=True)
        p.close(); da.close()
        del A, yl, y, a, x


if __name__ == "__main__":
    main()
