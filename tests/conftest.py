import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def oracle():
    """The CPU restatement (oracle/spmx_oracle.c) — the checker, never the product."""
    from oracle.pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    """The unmodified reference library, where oracle/_ref was built (optional)."""
    from oracle.pyoracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref/libspmx_ref.so not built here")
    return RefLib()


@pytest.fixture(scope="session")
def golden_instances():
    z = np.load(os.path.join(GOLDEN, "ref_instances.npz"))
    n = len([k for k in z.files if k.endswith("_dims")])
    out = []
    for i in range(n):
        p = f"i{i}_"
        out.append({k[len(p):]: z[k] for k in z.files if k.startswith(p)})
    return out


@pytest.fixture(scope="session")
def ctx():
    """A context on cuda:0 through the C ABI. Fails loudly (no CPU fallback)."""
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2312_05639_b200.binding import Context
    # library kernels and the tests' torch work (fills, slices, generators) share one
    # explicit stream, so they are ordered without host synchronisation
    c = Context.on_torch_stream(0)
    yield c
    c.close()


def pytest_sessionfinish(session, exitstatus):
    """tools/bounds_check.py runs the GPU suite against a library built with
    -DSPMX_DEBUG_BOUNDS=1 and sets SPMX_BOUNDS_REPORT: the per-site counts of out-of-bounds
    accesses the kernels would have made are written there (all zero = clean)."""
    path = os.environ.get("SPMX_BOUNDS_REPORT")
    if not path:
        return
    import ctypes as C
    from paper_2312_05639_b200.binding import Lib
    lib = Lib.get()
    lib.lib.spmx_debug_bounds.argtypes = [C.POINTER(C.c_uint64)]
    out = (C.c_uint64 * 16)()
    rc = lib.lib.spmx_debug_bounds(out)
    with open(path, "w") as f:
        f.write(f"library {lib.path}\nrc {rc} launches {lib.launch_count()} pytest_exit {int(exitstatus)}\n")
        f.write("violations per site: " + " ".join(str(int(v)) for v in out) + "\n")
