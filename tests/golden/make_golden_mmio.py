"""Golden fixtures for MatrixMarket ingestion: small .mtx / vector / mask files
and the reference's own parse of each (``deflamg.mmio``, run in the build
container):

    python tests/golden/make_golden_mmio.py [--ref /tmp/refbuild/src]

Outputs (committed): tests/golden/mmio/*, tests/golden/golden_mmio.npz.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import ensure_ref  # noqa: E402

OUT = os.path.join(HERE, "mmio")

FILES = {
    "sym_comments.mtx": (
        "%%MatrixMarket matrix coordinate real symmetric\n"
        "% a 4x4 SPD matrix, lower triangle, scattered comments\n"
        "\n"
        "4 4 7\n"
        "1 1 4.0\n"
        "% in-between comment\n"
        "2 1 -1.25\n"
        "2 2 4.5\n"
        "3 2 -0.5e0\n"
        "3 3 3.0\n"
        "4 1 1e-3\n"
        "4 4 2.0\n"
    ),
    "dup_integer.mtx": (
        "%%MatrixMarket matrix coordinate integer general\n"
        "3 4 6\n"
        "1 1 3\n1 1 -1\n2 4 7\n3 2 5\n1 1 10\n3 2 -5\n"
    ),
    "upper_case_header.mtx": "%%MatrixMarket MATRIX Coordinate REAL General\n2 2 2\n1 2 0.1\n2 1 0.2\n",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/tmp/refbuild/src")
    args = ap.parse_args()
    os.environ["DEFLAMG_KERNELS"] = "c"
    sys.path.insert(0, ensure_ref(args.ref))
    from deflamg.mmio import read_mask, read_matrix_market, read_vector, write_matrix_market, write_vector
    from deflamg.problems import poisson3d

    os.makedirs(OUT, exist_ok=True)
    for name, text in FILES.items():
        with open(os.path.join(OUT, name), "w") as fh:
            fh.write(text)
    write_matrix_market(poisson3d(6).matrix, os.path.join(OUT, "poisson6.mtx"))
    x = np.sin(np.arange(11) * 0.7) * 10.0 ** np.arange(-5, 6)
    write_vector(x, os.path.join(OUT, "vec.txt"))
    with open(os.path.join(OUT, "mask.txt"), "w") as fh:
        fh.write("% pressure mask\n1\n0\n\n1\n1\n0\n")
    arrs = {}
    for name in list(FILES) + ["poisson6.mtx"]:
        A = read_matrix_market(os.path.join(OUT, name))
        arrs[name + "/shape"] = np.array([A.nrows, A.ncols])
        arrs[name + "/ptr"], arrs[name + "/col"], arrs[name + "/val"] = A.row_ptr, A.col_idx, A.values
    arrs["vec.txt"] = read_vector(os.path.join(OUT, "vec.txt"))
    arrs["mask.txt"] = read_mask(os.path.join(OUT, "mask.txt"))
    np.savez_compressed(os.path.join(HERE, "golden_mmio.npz"), **arrs)
    print(sorted(arrs))


if __name__ == "__main__":
    main()
