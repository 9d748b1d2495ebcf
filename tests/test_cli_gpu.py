"""GPU suite: spmx_bench_b200, the reference's bench CLI (tools/bench.cpp) for the B200 path
(SURVEY §8 f1): report fields and order, y_checksum against the reference, exit codes."""
import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "io")

REF_COLUMNS = ("matrix,m,n,nnz,d,strategy,backend,tier,threads,batch_size,trials,times_s,mean_s,codegen_s,"
               "codegen_pct,gflops,memory_loads,stores,branches,vector_arith,scalar_arith,instructions,"
               "y_checksum,max_rel_err,status")  # tools/bench.cpp:109-113


@pytest.fixture(scope="module")
def cli():
    from tools import hostbuild
    return hostbuild.CLI if os.path.exists(hostbuild.CLI) else hostbuild.build_cli()


def run(cli, *args):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=600)


def test_single_run_report_and_checksum(cli):
    """`--synthetic 2000 --cols 32` builds random_csr(2000, 16, 0, 42 ^ 0x5157a7e5) and
    random_dense(2000, 32, 42) exactly as the reference's CLI does; in exact-order mode the
    y_checksum must equal the reference's (fixture produced by the reference library)."""
    z = np.load(os.path.join(GOLD, "rand300.npz"))
    want = int(z["cli_checksum"][0])
    for strategy, dispatch in (("row", "dynamic"), ("row", "static"), ("nnz", "static"), ("merge", "static")):
        r = run(cli, "--synthetic", 2000, "--cols", 32, "--strategy", strategy, "--dispatch", dispatch,
                "--backend", "interp", "--trials", 2, "--verify")
        assert r.returncode == 0, r.stderr
        j = json.loads(r.stdout)
        assert [j["m"], j["n"], j["nnz"]] == z["cli_dims"].tolist()
        assert j["y_checksum"] == want
        assert j["strategy"] == strategy + ("+dynamic" if strategy == "row" and dispatch == "dynamic" else "")
        assert j["backend"] == "interp" and j["d"] == 32 and j["trials"] == 2 and len(j["times_s"]) == 2
        assert j["max_rel_err"] <= 1e-5
        assert abs(j["gflops"] - 2.0 * j["nnz"] * 32 / j["mean_s"] / 1e9) <= 1e-6 * j["gflops"]
        want_bytes = 8 * j["nnz"] + 4 * (j["m"] + 1) + 4 * j["n"] * 32 + 4 * j["m"] * 32
        assert j["bytes_algorithmic"] == want_bytes and j["gpus"] == 1
        # field order of the reference's report, GPU fields after it
        keys = [k for k in j]
        ref_order = [k for k in REF_COLUMNS.split(",") if k in j]
        assert keys[:len(ref_order)] == ref_order
    r = run(cli, "--synthetic", 2000, "--cols", 32, "--strategy", "merge", "--dispatch", "static")
    assert r.returncode == 0 and json.loads(r.stdout)["backend"] == "native"


def test_csv_sweep_files_and_exit_codes(cli, tmp_path):
    rep = tmp_path / "sweep.csv"
    r = run(cli, "sweep", "--matrix", os.path.join(GOLD, "rand300.jspm"), "--d-list", 8, 45,
            "--strategies", "row", "merge", "--backends", "native", "interp", "--dispatch", "static",
            "--verify", "--format", "csv", "--report", rep)
    assert r.returncode == 0, r.stderr
    lines = rep.read_text().strip().split("\n")
    assert lines[0].startswith(REF_COLUMNS + ",")
    assert len(lines) == 1 + 2 * 2 * 2
    cols = lines[0].split(",")
    sums = set()
    for ln in lines[1:]:
        f = dict(zip(cols, ln.split(",")))
        assert f["status"] == "ok" and f["m"] == "300" and float(f["max_rel_err"]) <= 1e-5
        if f["backend"] == "interp":
            sums.add((f["d"], f["y_checksum"]))
    assert len(sums) == 2  # exact-order checksum depends on d only, not on the strategy
    # Matrix Market input, cache output
    cache = tmp_path / "out.jspm"
    r = run(cli, "--matrix", os.path.join(GOLD, "general_dups.mtx"), "--cols", 4, "--save-cache", cache)
    assert r.returncode == 0 and cache.exists() and json.loads(r.stdout)["nnz"] == 6
    # usage errors -> 1 (bench.cpp:294-309)
    assert run(cli, "--cols", 0, "--synthetic", 10).returncode == 1
    assert run(cli, "--strategy", "diagonal", "--synthetic", 10).returncode == 1
    assert run(cli).returncode == 1
    assert run(cli, "--matrix", tmp_path / "absent.mtx").returncode == 1
    assert run(cli, "--tier", "avx2", "--synthetic", 10).returncode == 1
    # dynamic dispatch is silently limited to the row strategy, as in the reference (bench.cpp:155)
    r = run(cli, "--synthetic", 500, "--strategy", "nnz", "--dispatch", "dynamic")
    assert r.returncode == 0 and json.loads(r.stdout)["strategy"] == "nnz"


def test_baseline_configs_from_the_cli(cli, oracle):
    """--config cN: the CLI generates BASELINE.json's configurations itself (host C++ generators,
    host/spmx_workloads.hpp) — the same arrays as workloads.py, so the exact-order y_checksum
    equals the oracle's on the Python-generated sibling, also through the multi-GPU driver."""
    from paper_2312_05639_b200 import workloads as W
    for name, scale in (("c2", 12), ("c5", 11)):
        a, x, spec = W.make_config(name, scale_override=scale)
        rp, col, vals = a.numpy()
        want = oracle.checksum(oracle.spmm_fused(a.m, a.n, rp, col, vals, x.numpy()))
        for extra in ((), ("--gpus", 1, "--shards", 3)):
            r = run(cli, "--config", name, "--scale", scale, "--strategy", "merge", "--dispatch", "static",
                    "--backend", "interp", *extra)  # (no --verify: the reference's relative criterion
            assert r.returncode == 0, r.stderr        #  assumes positive data, X here is U[-1,1))
            j = json.loads(r.stdout[r.stdout.index("{"):])  # (NCCL may print its version line first)
            assert (j["m"], j["nnz"], j["d"]) == (a.m, a.nnz, spec["d"])
            assert j["y_checksum"] == want
    assert run(cli, "--config", "c9").returncode == 1


def test_plain_c_caller_of_the_abi(tmp_path):
    """examples/spmx_minimal.c: the reference's worked example (test_matrix_core.cpp:181-189) from a
    C99 program with malloc'ed arrays, every strategy, both modes, and the reference's shape error."""
    import subprocess
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_abi_cpu import _build_c_example
    out = subprocess.run([_build_c_example(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "worked example ok" in out.stdout
