"""One config, one strategy, a few launches: the command ncu wraps.
    python tools/prof_one.py c2 merge fast [iters] [--scale N]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_05639_b200 import workloads as W
from paper_2312_05639_b200.binding import Context, EXACT_ORDER
name, strat, mode = sys.argv[1], sys.argv[2], sys.argv[3]
iters = int(sys.argv[4]) if len(sys.argv) > 4 and not sys.argv[4].startswith("--") else 5
scale = int(sys.argv[sys.argv.index("--scale") + 1]) if "--scale" in sys.argv else None
ctx = Context.on_torch_stream(0)
a, x, spec = W.make_config(name, device="cuda", scale_override=scale)
da = ctx.csr_wrap(a)
y = torch.empty(a.m, spec["d"], device="cuda")
p = ctx.plan(da, strat.split("-")[0], 0, dynamic=strat.endswith("dyn"),
             flags={"fast": 0, "exact": EXACT_ORDER}[mode])
for _ in range(iters):
    ms = ctx.spmm(p, da, x, y, timed=True)
print(name, strat, mode, "nnz", a.nnz, "last ms", ms)
