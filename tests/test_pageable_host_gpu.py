"""Host-buffer entry points with PAGEABLE host memory — what a caller of the reference's run_spmm
holds (std::vector-backed CsrMatrix / DenseMatrix, include/spmx/csr.hpp:10-20, dense.hpp:9-21).
Arrays of 1 MB and more are staged through pinned slots by several host threads
(csrc/spmx_stage.cuh) instead of the driver's single one. The result must be the same bits as
with pinned arrays and as the device-resident path, for any mix of pageable and pinned
arguments, for unaligned pageable pointers, with the staging switched off, and an invalid
matrix must still come back as SPMX_EINVAL with nothing left running."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pinned_like(a):
    v = a.view(np.int64) if a.dtype == np.uint64 else a.view(np.int32) if a.dtype == np.uint32 else a
    return torch.from_numpy(v).pin_memory().numpy().view(a.dtype)


@pytest.fixture(scope="module")
def case():
    from paper_2312_05639_b200 import workloads as W
    a, x, spec = W.make_config("c2", device="cuda", scale_override=17)  # 131 072 rows, ~2 M nonzeros, X and Y 32 MB
    rp, col, vals = a.numpy()
    return a, x, spec["d"], rp, col, vals, x.cpu().numpy()


def test_pageable_equals_pinned_and_device_path(case):
    from paper_2312_05639_b200.binding import Context
    a, x, d, rp, col, vals, xn = case
    ctx = Context(0)
    # device-resident path
    da = ctx.csr_upload(a.m, a.n, rp, col, vals)     # pageable arrays: the staged upload
    p = ctx.plan(da, "merge", 0)
    y_dev = torch.empty(a.m, d, device="cuda")
    ctx.spmm(p, da, x, y_dev)
    ctx.synchronize()
    want = y_dev.cpu().numpy()
    p.close(); da.close()
    pins = dict(rp=_pinned_like(rp), col=_pinned_like(col), vals=_pinned_like(vals), x=_pinned_like(xn))
    page = dict(rp=rp, col=col, vals=vals, x=xn)
    for pinned_args in ([], ["rp", "col", "vals", "x"], ["x"], ["col", "vals"], ["rp"]):
        src = {k: (pins if k in pinned_args else page)[k] for k in page}
        for y_pinned in (False, True):
            y = torch.empty(a.m, d).pin_memory().numpy() if y_pinned else np.empty((a.m, d), np.float32)
            y.fill(np.nan)
            ctx.spmm_host(a.m, a.n, src["rp"], src["col"], src["vals"], src["x"], y=y, strategy="merge", nnz=a.nnz)
            assert np.array_equal(y.view(np.uint32), want.view(np.uint32)), (pinned_args, y_pinned)
    ctx.close()


def test_unaligned_pageable_pointers(case):
    """Pageable arrays at odd byte offsets of their allocations (the streaming copy aligns its
    stores itself; the 4-byte element alignment the types need is kept)."""
    from paper_2312_05639_b200.binding import Context
    a, x, d, rp, col, vals, xn = case
    ctx = Context(0)

    def shifted(arr, elems):
        buf = np.empty(arr.size + elems + 8, arr.dtype)
        out = buf[elems:elems + arr.size].reshape(arr.shape)
        out[...] = arr
        return out

    y0, _ = ctx.spmm_host(a.m, a.n, rp, col, vals, xn, strategy="nnz", nnz=a.nnz)
    ybuf = np.empty(a.m * d + 16, np.float32)
    y1 = ybuf[3:3 + a.m * d].reshape(a.m, d)
    ctx.spmm_host(a.m, a.n, shifted(rp, 1), shifted(col, 3), shifted(vals, 1), shifted(xn.ravel(), 5).reshape(xn.shape),
                  y=y1, strategy="nnz", nnz=a.nnz)
    assert np.array_equal(y0.view(np.uint32), y1.view(np.uint32))
    ctx.close()


def test_staging_switched_off_gives_the_same_bits(case, monkeypatch):
    from paper_2312_05639_b200.binding import Context
    a, x, d, rp, col, vals, xn = case
    ctx = Context(0)
    y0, _ = ctx.spmm_host(a.m, a.n, rp, col, vals, xn, strategy="row", nnz=a.nnz)
    monkeypatch.setenv("SPMX_HOST_STAGE_THREADS", "0")
    y1, _ = ctx.spmm_host(a.m, a.n, rp, col, vals, xn, strategy="row", nnz=a.nnz)
    assert np.array_equal(y0.view(np.uint32), y1.view(np.uint32))
    ctx.close()


def test_invalid_matrix_from_pageable_arrays_is_einval(case):
    from paper_2312_05639_b200.binding import Context, SpmxInvalidArgument
    a, x, d, rp, col, vals, xn = case
    ctx = Context(0)
    bad = col.copy()
    bad[bad.size // 2] = a.n + 7            # a column index past X, in the middle of the staged upload
    with pytest.raises(SpmxInvalidArgument):
        ctx.spmm_host(a.m, a.n, rp, bad, vals, xn, strategy="merge", nnz=a.nnz)
    bad_rp = rp.copy()
    bad_rp[100] = bad_rp[99] - 1 if bad_rp[99] > 0 else bad_rp[101] + 5   # not monotone
    with pytest.raises(SpmxInvalidArgument):
        ctx.spmm_host(a.m, a.n, bad_rp, col, vals, xn, strategy="merge", nnz=a.nnz)
    # the context is still usable and correct afterwards
    y0, _ = ctx.spmm_host(a.m, a.n, rp, col, vals, xn, strategy="merge", nnz=a.nnz)
    y1, _ = ctx.spmm_host(a.m, a.n, rp, col, vals, xn, strategy="merge", nnz=a.nnz)
    assert np.array_equal(y0.view(np.uint32), y1.view(np.uint32)) and np.isfinite(y0).all()
    ctx.close()


@pytest.mark.parametrize("nbytes", [(1 << 20) - 4, 1 << 20, (4 << 20) - 4, 4 << 20, (4 << 20) + 4, (8 << 20) + 12,
                                    (33 << 20) + 20, (64 << 20) - 8])
def test_staged_copies_round_trip(nbytes):
    """spmx_h2d / spmx_d2h with pageable arrays whose sizes sit on and around the stager's 1 MB
    threshold and 4 MB piece boundaries, at a misaligned host address: up, down, same bytes, and
    nothing written outside the destination."""
    import ctypes as C
    from paper_2312_05639_b200.binding import Context
    ctx = Context(0)
    rng = np.random.default_rng(nbytes)
    src_buf = rng.integers(0, 256, nbytes + 64, dtype=np.uint8)
    dst_buf = np.full(nbytes + 128, 0xA5, np.uint8)
    src = src_buf[4:4 + nbytes]              # 4-byte offsets into the allocations
    dst = dst_buf[36:36 + nbytes]
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    L = ctx.L
    L.check(L.lib.spmx_h2d(ctx.h, C.c_void_p(dev.data_ptr()), C.c_void_p(src.ctypes.data), C.c_size_t(nbytes)))
    ctx.synchronize()
    assert np.array_equal(dev.cpu().numpy(), src)
    L.check(L.lib.spmx_d2h(ctx.h, C.c_void_p(dst.ctypes.data), C.c_void_p(dev.data_ptr()), C.c_size_t(nbytes)))
    ctx.synchronize()
    assert np.array_equal(dst, src)
    assert (dst_buf[:36] == 0xA5).all() and (dst_buf[36 + nbytes:] == 0xA5).all()
    ctx.close()
