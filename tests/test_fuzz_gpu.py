"""Randomised parity sweep: seeded matrices with adversarial row structures (runs of empty rows,
a few giant rows, rows exactly at the window / long-row / chunk thresholds, duplicate columns,
rectangular shapes) x widths x strategies x partition counts x both modes, each compared with
the CPU oracle: bitwise against the fused CSR-order chain in exact-order mode (interp.cpp:36-51),
within the north_star bound against the unfused reference (reference.cpp:10-25) otherwise.
The long-row threshold is lowered for half of the cases so that spmm_long_row_kernel sees
ordinary rows too."""
import numpy as np
import pytest
import torch

from helpers import north_star_ok

pytestmark = pytest.mark.gpu
EXACT, CLAIM = 1, 8


def _row_lengths(rng, m, kind):
    if kind == "powerlaw":
        lens = np.minimum((rng.pareto(1.1, m) * 3).astype(np.int64), 6000)
    elif kind == "mostly_empty":
        lens = np.where(rng.random(m) < 0.9, 0, rng.integers(1, 200, m))
    elif kind == "giants":
        lens = rng.integers(0, 12, m)
        for r in rng.choice(m, size=min(4, m), replace=False):
            lens[r] = int(rng.integers(1000, 9000))
    elif kind == "thresholds":
        pool = np.array([0, 1, 63, 64, 65, 127, 128, 129, 255, 256, 257, 511, 512, 1023, 1024, 1025])
        lens = rng.choice(pool, m)
    else:  # regular
        lens = rng.integers(20, 44, m)
    return lens.astype(np.int64)


CASES = [(seed, kind) for seed, kind in enumerate(
    ["powerlaw", "mostly_empty", "giants", "thresholds", "regular"] * 4)]


@pytest.mark.parametrize("seed,kind", CASES, ids=[f"{k}-{s}" for s, k in CASES])
def test_random_structures_against_the_oracle(ctx, oracle, monkeypatch, seed, kind):
    rng = np.random.default_rng(9000 + seed)
    m = int(rng.integers(1, 700))
    n = int(rng.integers(1, 900))
    d = int(rng.choice([1, 3, 4, 8, 12, 16, 20, 32, 45, 64, 100, 128, 160]))
    if seed % 2:
        monkeypatch.setenv("SPMX_LONG_ROW", str(int(rng.choice([4, 16, 100]))))
    lens = _row_lengths(rng, m, kind)
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum(lens.astype(np.uint64))
    nnz = int(rp[-1])
    col = rng.integers(0, n, size=nnz, dtype=np.int64).astype(np.uint32)  # duplicates allowed
    vals = (rng.random(nnz, np.float32) * 2 - 1).astype(np.float32)
    x = (rng.random((n, d), np.float32) * 2 - 1).astype(np.float32)
    fused = oracle.spmm_fused(m, n, rp, col, vals, x)
    unf = oracle.spmm_unfused(m, n, rp, col, vals, x)
    bound = oracle.abs_bound(m, rp, col, vals, x)
    a = ctx.csr_upload(m, n, rp, col, vals)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty(m, d, device="cuda")
    configs = [(s, p, f, False) for s in ("row", "nnz", "merge") for p in (0, 1, 5, 1000) for f in (0, EXACT)]
    configs += [("row", 0, f, True) for f in (0, EXACT, CLAIM, EXACT | CLAIM)]
    for strat, parts, flags, dyn in configs:
        plan = ctx.plan(a, strat, parts, dynamic=dyn, batch=int(rng.integers(1, 200)), flags=flags)
        yd.fill_(float("nan"))
        ctx.spmm(plan, a, xd, yd)
        ctx.synchronize()
        got = yd.cpu().numpy()
        tag = (seed, kind, m, n, d, strat, parts, flags, dyn)
        if flags & EXACT or (dyn and flags & CLAIM):
            assert np.array_equal(got.view(np.uint32), fused.view(np.uint32)), tag
        else:
            assert north_star_ok(got, unf, bound), tag
        plan.close()
    # the host-buffer entry point, both modes
    for flags in (0, EXACT):
        yh, _ = ctx.spmm_host(m, n, rp, col, vals, x, strategy="merge", flags=flags)
        if flags:
            assert np.array_equal(yh.view(np.uint32), fused.view(np.uint32)), (seed, kind, "host exact")
        else:
            assert north_star_ok(yh, unf, bound), (seed, kind, "host")
    a.close()
