"""Developer timing loop (not the contract bench): per-config, per-strategy device times.

    python tools/dev_bench.py c2 [c3 ...] [--scale N] [--iters K] [--check]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_05639_b200 import workloads as W  # noqa: E402
from paper_2312_05639_b200.binding import Context, EXACT_ORDER, JIT_WIDTH  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2"])
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--parts", type=int, default=0)
    ap.add_argument("--d", type=int, default=None, help="override the dense width")
    ap.add_argument("--modes", default="fast,exact")
    ap.add_argument("--strategies", default="row,nnz,merge,row-dyn")
    args = ap.parse_args()
    peak = 6551.0
    try:
        peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    ctx = Context.on_torch_stream(0)
    for name in args.configs:
        t0 = time.time()
        a, x, spec = W.make_config(name, device="cuda", scale_override=args.scale, m_override=args.m)
        torch.cuda.synchronize()
        if args.d:
            spec["d"] = args.d
            x = W.dense(a.n, args.d, spec["seed"], spec["x_dist"], "cuda")
            torch.cuda.synchronize()
        d = spec["d"]
        byts = W.algorithmic_bytes(a.m, a.n, a.nnz, d)
        print(f"== {name}: m={a.m} nnz={a.nnz} d={d} bytes={byts/1e6:.1f}MB gen={time.time()-t0:.1f}s "
              f"roofline_t={byts/peak/1e3:.1f}us", flush=True)
        da = ctx.csr_wrap(a)
        y = torch.empty(a.m, d, device="cuda")
        ref = None
        for strat in args.strategies.split(","):
            for mode in args.modes.split(","):
                flags = {"fast": 0, "exact": EXACT_ORDER, "jit": JIT_WIDTH}[mode]
                dyn = strat in ("row-dyn", "row-claim")  # row-claim: the literal claim kernel
                if strat == "row-claim":
                    flags |= 8  # SPMX_CLAIM_KERNEL
                tp = time.time()
                p = ctx.plan(da, strat.split("-")[0], args.parts, dynamic=dyn, flags=flags)
                ctx.synchronize()
                tp = time.time() - tp
                for _ in range(3):
                    ctx.spmm(p, da, x, y)
                ts = [ctx.spmm(p, da, x, y, timed=True) for _ in range(args.iters)]
                ms = float(np.median(ts))
                line = (f"  {strat:8s} {mode:6s} chunks={p.n_chunks:8d} plan={tp*1e3:7.1f}ms "
                        f"t={ms*1e3:9.1f}us min={min(ts)*1e3:9.1f}us GF={2*a.nnz*d/ms/1e6:9.1f} "
                        f"GB/s={byts/ms/1e6:8.1f} frac={byts/ms/1e6/peak:.3f}")
                if args.check:
                    if ref is None:
                        ref = y.clone()
                    else:
                        diff = (y - ref).abs().max().item()
                        line += f" maxdiff_vs_first={diff:.3e} bitwise={bool(torch.equal(y, ref))}"
                print(line, flush=True)
                p.close()
        da.close()
        del a, x, y


if __name__ == "__main__":
    main()
