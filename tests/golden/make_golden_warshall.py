"""Golden fixtures for the Warshall backend, made by EXECUTING THE REFERENCE.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_warshall.py

Runs only in the build container (/root/reference exists there). Records, for
reference merge.py:169-238:
  adjacency cases   build_core_adjacency(nbr, valid) of fused_build_algebraic
                    outputs on small blob sets and the reference test-suite's
                    collinear / complete / isolated cases: input bits + valid,
                    output core_indices + bits
  closure cases     warshall_closure of random symmetric relations (the tests'
                    generator style), of identity, chain and of random DIRECTED
                    relations (no symmetry assumed), input and output bits
  merge cases       merge_warshall labels for a valid vector that is NOT
                    counts >= min_pts (the reference never checks it)
Output: tests/golden/warshall.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from densescan import (KernelVariant, PointSet, ValidVector, VariantId,  # noqa: E402
                       fused_build_algebraic, validate_params)
from densescan._bitmat import pack_rows  # noqa: E402
from densescan.merge import (CoreAdjacency, build_core_adjacency, merge_warshall,  # noqa: E402
                             warshall_closure)

from paper_1506_02226_b200.datasets import generate_blobs  # noqa: E402


def pad3(c):
    c = np.asarray(c, dtype=np.float64)
    out = np.zeros((c.shape[0], 3))
    out[:, : c.shape[1]] = c
    return out


def main():
    out = {}
    rng = np.random.default_rng(1506)
    adj_cases = [
        ("collinear", np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float), 1.2, 2),
        ("complete", np.array([[0, 0, 0], [0.1, 0, 0], [0.2, 0, 0]], float), 1.0, 3),
        ("skip_noncore", np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [50, 0, 0]], float), 1.2, 2),
        ("isolated", rng.normal(size=(5, 3)) * 50, 1e-3, 2),
        ("blobs300", pad3(generate_blobs(300, 3, 0.3, 0.1, 5, 2).coords_aos), 0.25, 4),
        ("blobs1500", pad3(generate_blobs(1500, 5, 0.4, 0.05, 6, 2).coords_aos), 0.2, 6),
        ("blobs3d", generate_blobs(900, 4, 0.2, 0.1, 7, 3).coords_aos, 0.15, 5),
    ]
    names = []
    for name, pts, eps, min_pts in adj_cases:
        params = validate_params(eps, min_pts)
        nbr, valid = fused_build_algebraic(PointSet(pts), params,
                                           KernelVariant(VariantId.FUSED_ALGEBRAIC))
        adj = build_core_adjacency(nbr, valid)
        closed = warshall_closure(adj)
        labels = merge_warshall(nbr, valid).labels
        out[f"adj/{name}/bits"] = nbr.bits
        out[f"adj/{name}/valid"] = valid.valid.astype(np.uint8)
        out[f"adj/{name}/core_indices"] = adj.core_indices
        out[f"adj/{name}/adj"] = adj.bits
        out[f"adj/{name}/closed"] = closed.bits
        out[f"adj/{name}/labels"] = labels
        names.append(name)
    out["adj_names"] = np.array(names)

    cl_names = []

    def closure_case(name, rel):
        m = rel.shape[0]
        adj = CoreAdjacency(m=m, core_indices=np.arange(m, dtype=np.int64), bits=pack_rows(rel))
        out[f"cl/{name}/in"] = adj.bits
        out[f"cl/{name}/out"] = warshall_closure(adj).bits
        cl_names.append(name)

    closure_case("identity9", np.eye(9, dtype=bool))
    closure_case("chain3", np.array([[1, 1, 0], [1, 1, 1], [0, 1, 1]], bool))
    for t in range(8):  # symmetric, reflexive (test_merge.py random_symmetric_adjacency style)
        m = int(rng.integers(1, 300))
        a = rng.random((m, m)) < float(rng.uniform(0.002, 0.05))
        a = a | a.T | np.eye(m, dtype=bool)
        closure_case(f"sym{t}", a)
    for t in range(8):  # directed, no diagonal guarantee: closure = R+ exactly
        m = int(rng.integers(1, 200))
        a = rng.random((m, m)) < float(rng.uniform(0.003, 0.03))
        closure_case(f"dir{t}", a)
    closure_case("dir_cycle70", np.roll(np.eye(70, dtype=bool), 1, axis=1))
    out["cl_names"] = np.array(cl_names)

    # merge_warshall with a valid vector that disagrees with the counts
    pts = pad3(generate_blobs(400, 3, 0.3, 0.1, 8, 2).coords_aos)
    params = validate_params(0.25, 5)
    nbr, valid = fused_build_algebraic(PointSet(pts), params,
                                       KernelVariant(VariantId.FUSED_ALGEBRAIC))
    v = valid.valid.copy()
    flip = rng.choice(v.size, 40, replace=False)
    v[flip] = ~v[flip]
    v &= nbr.neighbor_count >= 2  # keep every "core" with a non-empty core row
    out["mw/bits"] = nbr.bits
    out["mw/valid"] = v.astype(np.uint8)
    out["mw/labels"] = merge_warshall(nbr, ValidVector(valid=v, min_pts=5)).labels
    np.savez_compressed(os.path.join(HERE, "warshall.npz"), **out)
    print("wrote warshall.npz:", len(names), "adjacency cases,", len(cl_names), "closure cases")


if __name__ == "__main__":
    main()
