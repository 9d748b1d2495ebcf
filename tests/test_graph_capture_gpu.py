"""spmx_spmm inside a CUDA graph: the call launches kernels only (no allocation, no host
synchronisation; the fix-up rides on programmatic stream serialisation, the long rows of
exact-order plans on forked auxiliary streams joined by events), so a caller that captures its
step into a graph can include it. The replayed graph must write the same bits as the eager call,
in both modes, and a second replay after X has changed must follow the new X."""
import pytest
import torch

pytestmark = pytest.mark.gpu

EXACT = 1


@pytest.mark.parametrize("flags", [0, EXACT], ids=["default", "exact"])
def test_spmm_is_graph_capturable(ctx, flags):
    from paper_2312_05639_b200 import workloads as W
    a, x, spec = W.make_config("c2", device="cuda", scale_override=14)
    d = spec["d"]
    da = ctx.csr_wrap(a)
    p = ctx.plan(da, "merge", 0, flags=flags)
    y_eager = torch.empty(a.m, d, device="cuda")
    y_graph = torch.full((a.m, d), float("nan"), device="cuda")
    ctx.spmm(p, da, x, y_eager)
    ctx.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=ctx._torch_stream):
        ctx.spmm(p, da, x, y_graph)
    # capture must not have executed anything
    assert bool(torch.isnan(y_graph).all())
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y_eager.view(torch.int32), y_graph.view(torch.int32))
    # the graph reads X through the captured pointer: new contents, new result
    x.mul_(-2.0)
    ctx.spmm(p, da, x, y_eager)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y_eager.view(torch.int32), y_graph.view(torch.int32))
    p.close()
    da.close()
