"""Generates tests/golden/*.npz by running the UNMODIFIED reference library
(oracle/_ref/libspmx_ref.so, built from /root/reference by oracle/Makefile) in
this container. /root/reference does not exist on the GPU box, so the outputs
are committed; re-run this script to regenerate them:

    python tests/golden/make_golden.py

Files:
  ref_instances.npz  the first 40 instances of the reference's acceptance stream
                     (tests/acceptance.cpp:69-124: mt19937_64(2026), m,n <= 200,
                     density 0.5-20 %, d from its pool, X = random_dense(n, d, rng()))
                     with: Y of run_spmm (native JIT, bitwise == interpreter), Y of
                     spmm_reference (unfused), and split_nnz / split_merge /
                     split_rows_static for several T, merge_path_search on every diagonal.
  ref_executor.npz   test_executor.cpp:67-87 instance (200x200, density 0.05, seed 51,
                     d=45, X seed 9): checksum of run_spmm, invariant over strategies/T.
  ref_configs.npz    scaled-down siblings of BASELINE configs c1..c5 from
                     paper_2312_05639_b200.workloads: checksums of the reference's
                     run_spmm result and partition boundaries for T in {7, 64}.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import RefLib  # noqa: E402
from paper_2312_05639_b200 import workloads as W  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
D_POOL = [1, 2, 3, 4, 5, 7, 8, 15, 16, 17, 31, 32, 45, 64, 100]
PARTS = [1, 2, 3, 4, 7, 8, 16, 61]


def instances(ref, count):
    rng = ref.rng(2026)
    for _ in range(count):
        m = 1 + rng() % 200
        n = 1 + rng() % 200
        density = 0.005 + 0.195 * float(rng() % 1000) / 1000.0
        a = ref.random_csr_rect(rng, m, n, density)
        d = D_POOL[rng() % len(D_POOL)]
        x = ref.random_dense(n, d, rng())
        yield a, x


def main():
    ref = RefLib()
    out = {}
    for idx, (a, x) in enumerate(instances(ref, 40)):
        rp, col, vals = a.arrays()
        y_native, _ = ref.run_spmm(a, x, "row", False, 1, "native")
        y_interp, _ = ref.run_spmm(a, x, "merge", False, 3, "interp")
        assert np.array_equal(y_native, y_interp)
        p = f"i{idx}_"
        out[p + "dims"] = np.array([a.m, a.n, a.nnz, x.shape[1]], np.int64)
        out[p + "row_ptr"], out[p + "col"], out[p + "vals"], out[p + "x"] = rp, col, vals, x
        out[p + "y_fused"] = y_native
        out[p + "y_unfused"] = ref.spmm_reference(a, x)
        for t in PARTS:
            out[p + f"nnz{t}"] = ref.split_nnz(a, t)
            out[p + f"merge{t}"] = ref.split_merge(a, t)
            out[p + f"rows{t}"] = ref.split_rows_static(a.m, t)
        ks = np.arange(a.m + a.nnz + 1, dtype=np.uint64)
        ij = np.array([ref.merge_path_search(a, int(k)) for k in ks], np.uint64)
        out[p + "mp_i"], out[p + "mp_j"] = ij[:, 0].copy(), ij[:, 1].copy()
    np.savez_compressed(os.path.join(OUT, "ref_instances.npz"), **out)

    rng = ref.rng(51)
    a = ref.random_csr_rect(rng, 200, 200, 0.05)
    x = ref.random_dense(200, 45, 9)
    rp, col, vals = a.arrays()
    y, _ = ref.run_spmm(a, x, "row", False, 1, "interp")
    sums = {ref.checksum(ref.run_spmm(a, x, s, dyn, t, "native")[0])
            for s, dyn in (("row", False), ("row", True), ("nnz", False), ("merge", False))
            for t in (1, 2, 4, 7)}
    assert sums == {ref.checksum(y)}
    np.savez_compressed(os.path.join(OUT, "ref_executor.npz"), row_ptr=rp, col=col, vals=vals, x=x,
                        checksum=np.array([ref.checksum(y)], np.uint64))

    cfg = {}
    small = {"c1": {}, "c2": {"scale_override": 12}, "c3": {"m_override": 1 << 12},
             "c4": {"scale_override": 12}, "c5": {"scale_override": 11}}
    for name, kw in small.items():
        a, x, spec = W.make_config(name, **kw)
        rp, col, vals = a.numpy()
        ra = ref.csr(a.m, a.n, rp, col, vals)
        y, _ = ref.run_spmm(ra, x.numpy(), "nnz", False, 0, "native")
        cfg[name + "_dims"] = np.array([a.m, a.n, a.nnz, spec["d"]], np.int64)
        cfg[name + "_checksum_fused"] = np.array([ref.checksum(y)], np.uint64)
        cfg[name + "_checksum_unfused"] = np.array(
            [ref.checksum(ref.spmm_reference(ra, x.numpy()))], np.uint64)
        cfg[name + "_row_ptr_checksum"] = np.array([int(rp.sum() % (1 << 63))], np.uint64)
        cfg[name + "_y_head"] = y[:4].copy()
        for t in (7, 64):
            cfg[name + f"_nnz{t}"] = ref.split_nnz(ra, t)
            cfg[name + f"_merge{t}"] = ref.split_merge(ra, t)
    np.savez_compressed(os.path.join(OUT, "ref_configs.npz"), **cfg)
    for f in ("ref_instances.npz", "ref_executor.npz", "ref_configs.npz"):
        print(f, os.path.getsize(os.path.join(OUT, f)) // 1024, "KiB")


if __name__ == "__main__":
    main()
