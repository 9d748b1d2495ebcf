"""Seeded synthetic inputs with the shapes of BASELINE.json's five configs.

The reference ships no generator for these distributions (its random_csr,
src/csr.cpp:106-133, makes power-law row lengths with duplicate columns and
U[0,1) values), and the paper's SuiteSparse matrices are not available, so
these stand in for them.

Everything is a counter-based hash (splitmix64 finaliser) of (seed, stream,
index) evaluated with wrapping int64 tensor arithmetic, so the same call gives
bit-identical arrays on a CPU tensor and on a CUDA tensor: generate once on
whichever device is at hand and give the same arrays to the CUDA path and to
the CPU oracle. The only floating-point step is Box-Muller for N(0,1), done in
float64 and rounded to float32.

This module is input plumbing for tests/ and bench.py; it is not on the
hot path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

_M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    """Python int -> the signed 64-bit value with the same bit pattern."""
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


_GOLD = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _lsr(x: torch.Tensor, s: int) -> torch.Tensor:
    """Logical shift right on int64 (torch's >> is arithmetic)."""
    return (x >> s) & ((1 << (64 - s)) - 1)


def mix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 output function on int64 tensors (wrapping arithmetic)."""
    x = x + _GOLD
    x = (x ^ _lsr(x, 30)) * _C1
    x = (x ^ _lsr(x, 27)) * _C2
    return x ^ _lsr(x, 31)


def _key(seed: int, stream: int) -> int:
    # scalar splitmix of (seed, stream), computed in Python ints
    z = (seed * 0x9E3779B97F4A7C15 + stream * 0xD1B54A32D192ED03 + 0x2545F4914F6CDD1D) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return _s64(z ^ (z >> 31))


def hash_index(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """64 hashed bits per int64 index."""
    return mix64(mix64(idx) ^ _key(seed, stream))


def u24(h: torch.Tensor) -> torch.Tensor:
    """Top 24 bits as an integer in [0, 2^24)."""
    return _lsr(h, 40)


def uniform_pm1(h: torch.Tensor) -> torch.Tensor:
    """U[-1,1) on the 2^-23 grid (exact in fp32)."""
    return (u24(h).to(torch.float32) * (2.0 ** -23)) - 1.0


def uniform_01_open_left(h: torch.Tensor) -> torch.Tensor:
    """U(0,1] on the 2^-24 grid (exact in fp32)."""
    return (u24(h) + 1).to(torch.float32) * (2.0 ** -24)


def normal01(h: torch.Tensor) -> torch.Tensor:
    """N(0,1) by Box-Muller from two 26-bit uniforms of one hash, in float64."""
    u1 = (_lsr(h, 38).to(torch.float64) + 1.0) * (2.0 ** -26)          # (0,1]
    u2 = ((h & ((1 << 26) - 1)).to(torch.float64)) * (2.0 ** -26)      # [0,1)
    z = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos((2.0 * math.pi) * u2)
    return z.to(torch.float32)


@dataclass
class Csr:
    """Host- or device-resident CSR with the reference's field types
    (include/spmx/csr.hpp:10-20): row_ptr u64 (stored int64), col u32 (stored
    int32 bit pattern), vals f32."""
    m: int
    n: int
    nnz: int
    row_ptr: torch.Tensor   # int64 [m+1]
    col: torch.Tensor       # int32 [nnz] (bit pattern of uint32)
    vals: torch.Tensor      # float32 [nnz]

    def numpy(self):
        return (self.row_ptr.cpu().numpy().view(np.uint64),
                self.col.cpu().numpy().view(np.uint32),
                self.vals.cpu().numpy())

    def to(self, device):
        return Csr(self.m, self.n, self.nnz, self.row_ptr.to(device), self.col.to(device),
                   self.vals.to(device))

    def row_slice(self, r0: int, r1: int) -> "Csr":
        """Rows [r0,r1) as a standalone CSR with a rebased row_ptr (the shard a
        rank owns under nnz-balanced row sharding)."""
        lo, hi = int(self.row_ptr[r0]), int(self.row_ptr[r1])
        return Csr(r1 - r0, self.n, hi - lo, (self.row_ptr[r0:r1 + 1] - lo).contiguous(),
                   self.col[lo:hi].contiguous(), self.vals[lo:hi].contiguous())


def dense(rows: int, d: int, seed: int, dist: str = "uniform_pm1", device="cpu",
          stream: int = 7) -> torch.Tensor:
    # element i is a function of (seed, stream, i) alone: generated in blocks of 2^26 elements so
    # that the int64 intermediates stay small (c5's X is 2^31 elements: 17 GB per int64 copy)
    fn = {"uniform_pm1": uniform_pm1, "normal": normal01}[dist]
    total = rows * d
    out = torch.empty(total, dtype=torch.float32, device=device)
    step = 1 << 26
    for lo in range(0, total, step):
        hi = min(lo + step, total)
        idx = torch.arange(lo, hi, dtype=torch.int64, device=device)
        out[lo:hi] = fn(hash_index(seed, stream, idx))
    return out.reshape(rows, d)


def _csr_from_sorted_keys(keys: torch.Tensor, m: int, n: int, shift: int, seed: int,
                          val_dist: str) -> Csr:
    rows = _lsr(keys, shift) if shift else None
    rows = keys >> shift
    cols = keys & ((1 << shift) - 1)
    nnz = keys.numel()
    counts = torch.bincount(rows, minlength=m)
    row_ptr = torch.zeros(m + 1, dtype=torch.int64, device=keys.device)
    torch.cumsum(counts, 0, out=row_ptr[1:])
    idx = torch.arange(nnz, dtype=torch.int64, device=keys.device)
    # value keyed by position in the final CSR order
    h = hash_index(seed, 3, idx)
    vals = {"uniform_pm1": uniform_pm1, "uniform_01": uniform_01_open_left,
            "normal": normal01}[val_dist](h)
    return Csr(m, n, nnz, row_ptr, cols.to(torch.int32), vals)


def uniform_fixed_degree(m: int, n: int, deg: int, seed: int, device="cpu") -> Csr:
    """Exactly `deg` distinct uniformly random columns per row, sorted (config c1).
    O(m*n) hashes: intended for small n only."""
    r = torch.arange(m, dtype=torch.int64, device=device).unsqueeze(1)
    c = torch.arange(n, dtype=torch.int64, device=device).unsqueeze(0)
    score = _lsr(hash_index(seed, 1, r * n + c), 1)           # non-negative
    cols = torch.topk(score, deg, dim=1, largest=False).indices
    cols, _ = torch.sort(cols, dim=1)
    keys = (r * (1 << 32) + cols).reshape(-1)
    return _csr_from_sorted_keys(keys, m, n, 32, seed, "uniform_pm1")


def rmat(scale: int, edge_factor: int, abcd, seed: int, device="cpu",
         chunk: int = 1 << 26) -> Csr:
    """R-MAT: edge_factor * 2^scale (row, col) draws, one quadrant per bit level
    with probabilities (a,b,c,d) = (top-left, top-right, bottom-left,
    bottom-right); duplicate edges merged; columns sorted per row; one U(0,1]
    value per surviving edge (configs c2, c4, c5)."""
    a, b, c, _ = abcd
    ta = int(round(a * (1 << 24)))
    tab = int(round((a + b) * (1 << 24)))
    tabc = int(round((a + b + c) * (1 << 24)))
    n = 1 << scale
    e_total = edge_factor * n
    parts = []
    for e0 in range(0, e_total, chunk):
        e = torch.arange(e0, min(e0 + chunk, e_total), dtype=torch.int64, device=device)
        row = torch.zeros_like(e)
        col = torch.zeros_like(e)
        for lvl in range(scale):
            u = u24(hash_index(seed, 100 + lvl, e))
            right = ((u >= ta) & (u < tab)) | (u >= tabc)      # quadrants b, d
            down = u >= tab                                   # quadrants c, d
            row = (row << 1) | down.to(torch.int64)
            col = (col << 1) | right.to(torch.int64)
        parts.append(torch.unique((row << 32) | col))
        del row, col, e
    keys = torch.unique(torch.cat(parts)) if len(parts) > 1 else parts[0]
    return _csr_from_sorted_keys(keys, n, n, 32, seed, "uniform_01")


def _poisson_clipped_table(lam: float, lo: int, hi: int) -> list[int]:
    """Integer CDF thresholds (scaled by 2^53) of Poisson(lam) clipped to [lo,hi]."""
    pmf = [math.exp(-lam + k * math.log(lam) - math.lgamma(k + 1)) for k in range(0, 4 * hi)]
    prob = [0.0] * (hi + 1)
    for k, p in enumerate(pmf):
        prob[min(max(k, lo), hi)] += p
    total = sum(prob)
    cdf, acc = [], 0.0
    for k in range(lo, hi + 1):
        acc += prob[k] / total
        cdf.append(min(int(acc * (1 << 53)), (1 << 53)))
    cdf[-1] = 1 << 53
    return cdf


def banded_poisson(m: int, lam: float, lo: int, hi: int, half_band: int, seed: int,
                   device="cpu") -> Csr:
    """Near-regular matrix (config c3): nnz/row ~ Poisson(lam) clipped to
    [lo,hi]; each column drawn uniformly from [i-half_band, i+half_band] and
    clamped to [0,m); columns sorted per row; duplicate columns are KEPT (CSR
    allows them and each contributes, reference SPEC.md:87); values N(0,1)."""
    r = torch.arange(m, dtype=torch.int64, device=device)
    u53 = _lsr(hash_index(seed, 1, r), 11)
    table = torch.tensor(_poisson_clipped_table(lam, lo, hi), dtype=torch.int64, device=device)
    lens = torch.searchsorted(table, u53, right=True) + lo
    lens = lens.clamp_(lo, hi)
    row_ptr = torch.zeros(m + 1, dtype=torch.int64, device=device)
    torch.cumsum(lens, 0, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    rows = torch.repeat_interleave(r, lens)
    idx = torch.arange(nnz, dtype=torch.int64, device=device)
    off = (_lsr(hash_index(seed, 2, idx), 1) % (2 * half_band + 1)) - half_band
    cols = (rows + off).clamp_(0, m - 1)
    keys, _ = torch.sort((rows << 32) | cols)
    return _csr_from_sorted_keys(keys, m, m, 32, seed, "normal")


# ---- the five BASELINE.json configs (and scaled-down siblings for tests) ------

CONFIGS = {
    "c1": dict(kind="uniform16", m=4096, d=32, seed=1, x_dist="uniform_pm1",
               strategies=("row",)),
    "c2": dict(kind="rmat", scale=20, ef=16, abcd=(0.57, 0.19, 0.19, 0.05), d=64, seed=2,
               x_dist="uniform_pm1", strategies=("row", "nnz", "merge")),
    "c3": dict(kind="banded", m=1 << 22, lam=32.0, lo=1, hi=64, half_band=65536, d=128, seed=3,
               x_dist="normal", strategies=("nnz",)),
    "c4": dict(kind="rmat", scale=22, ef=32, abcd=(0.65, 0.15, 0.15, 0.05), d=32, seed=4,
               x_dist="uniform_pm1", strategies=("merge", "row")),
    "c5": dict(kind="rmat", scale=24, ef=16, abcd=(0.57, 0.19, 0.19, 0.05), d=128, seed=5,
               x_dist="uniform_pm1", strategies=("nnz",)),
}


def make_config(name: str, device="cpu", scale_override: int | None = None,
                m_override: int | None = None):
    """Returns (Csr, X, spec). scale_override / m_override shrink the config to
    a sibling with the same distribution for CPU-sized parity tests."""
    spec = dict(CONFIGS[name])
    if spec["kind"] == "uniform16":
        m = m_override or spec["m"]
        a = uniform_fixed_degree(m, m, 16, spec["seed"], device)
    elif spec["kind"] == "rmat":
        sc = scale_override or spec["scale"]
        spec["scale"] = sc
        a = rmat(sc, spec["ef"], spec["abcd"], spec["seed"], device)
    else:
        m = m_override or spec["m"]
        spec["m"] = m
        hb = min(spec["half_band"], max(1, m // 4))
        a = banded_poisson(m, spec["lam"], spec["lo"], spec["hi"], hb, spec["seed"], device)
    x = dense(a.n, spec["d"], spec["seed"], spec["x_dist"], device)
    spec["name"] = name
    return a, x, spec


def algorithmic_bytes(m: int, n: int, nnz: int, d: int) -> int:
    """Compulsory bytes of one SpMM (BASELINE.json north_star / SURVEY.md §8d):
    8*nnz + 4*(M+1) + 4*N*d + 4*M*d."""
    return 8 * nnz + 4 * (m + 1) + 4 * n * d + 4 * m * d
