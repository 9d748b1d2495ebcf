"""Golden files for the data formats either side of the path, produced by
the UNMODIFIED reference library in this container (oracle/_ref):

  io/sym_pattern.mtx, io/general_dups.mtx, io/integer_sym.mtx   hand-written inputs (our own)
  io/*.mtx.npz               what the reference's load_matrix_market makes of them
  io/rand300.jspm            save_csr_cache(random_csr(300, 8, 0.5, 7)) written by the reference
  io/rand300.mtx             write_matrix_market of the same matrix, written by the reference
  io/rand300.npz             the matrix arrays, random_dense(300, 5, 11), and for the CLI test:
                             random_csr(2000, 16, 0, 42 ^ 0x5157a7e5) / random_dense(2000, 32, 42)
                             run_spmm checksum (what `spmx_bench --synthetic 2000 --cols 32`
                             reports as y_checksum)

    python tests/golden/make_golden_io.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import RefLib  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")

MTX = {
    "sym_pattern.mtx": """%%MatrixMarket matrix coordinate pattern symmetric
% a comment line
5 5 6
1 1
2 1
3 2

5 1
5 5
4 3
""",
    "general_dups.mtx": """%%MatrixMarket matrix coordinate real general
%
4 6 8
1 2 1.5
3 1 -2
1 2 0.25
4 6 1e-3
2 5 7
4 6 2e-3
4 1 3.5
1 6 -0.125
""",
    "integer_sym.mtx": """%%MatrixMarket matrix coordinate integer symmetric
3 3 4
1 1 2
2 1 -3
3 1 4
3 3 5
""",
}


def main():
    ref = RefLib()
    os.makedirs(OUT, exist_ok=True)
    for name, text in MTX.items():
        path = os.path.join(OUT, name)
        with open(path, "w") as f:
            f.write(text)
        a = ref.load_matrix_market(path)
        rp, col, vals = a.arrays()
        np.savez(path + ".npz", dims=np.array([a.m, a.n, a.nnz]), row_ptr=rp, col=col, vals=vals)
    a = ref.random_csr(300, 8.0, 0.5, 7)
    ref.save_csr_cache(a, os.path.join(OUT, "rand300.jspm"))
    ref.write_matrix_market(a, os.path.join(OUT, "rand300.mtx"))
    back = ref.load_matrix_market(os.path.join(OUT, "rand300.mtx"))  # duplicates get summed
    brp, bcol, bvals = back.arrays()
    np.savez(os.path.join(OUT, "rand300.mtx.npz"), dims=np.array([back.m, back.n, back.nnz]),
             row_ptr=brp, col=bcol, vals=bvals)
    rp, col, vals = a.arrays()
    cli_a = ref.random_csr(2000, 16.0, 0.0, 42 ^ 0x5157a7e5)
    cli_x = ref.random_dense(2000, 32, 42)
    y, _ = ref.run_spmm(cli_a, cli_x, "row", True, 0, "native")
    np.savez(os.path.join(OUT, "rand300.npz"), dims=np.array([a.m, a.n, a.nnz]), row_ptr=rp, col=col,
             vals=vals, dense=ref.random_dense(300, 5, 11),
             cli_dims=np.array([cli_a.m, cli_a.n, cli_a.nnz]),
             cli_checksum=np.array([ref.checksum(y)], np.uint64),
             cli_row_ptr_tail=cli_a.arrays()[0][-3:])
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
