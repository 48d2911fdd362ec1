"""Golden fixtures for the materialising ladder, by executing the REFERENCE package.

Runs only in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_dist.py

For each case it runs the reference's dist_baseline (kernels.py:177-180), checks
that dist_soa, dist_tiled(TILED) and dist_tiled(TILED_UNROLLED) give bitwise the
same matrix (the reference's own acceptance 2), and records the matrix plus
build_clusters_from_dist (kernels.py:284-308) bits and counts and the labels of
run_variant(BASELINE) -> merge_iterative.

Output: tests/golden/dist.npz
  <case>/points, <case>/params [eps, eps_sq, min_pts], <case>/dist (float32 n x n),
  <case>/bits, <case>/counts, <case>/labels
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from densescan import (DbscanParams, KernelVariant, PointSet, VariantId,  # noqa: E402
                       build_clusters_from_dist, dist_baseline, dist_soa, dist_tiled,
                       merge_iterative, generate_blobs)


def case(store, key, coords, eps, eps_sq, min_pts):
    coords = np.asarray(coords, dtype=np.float64)
    pts = PointSet(coords)
    params = DbscanParams(eps=eps, eps_sq=eps_sq, min_pts=min_pts)
    base = dist_baseline(pts, 2)
    for other in (dist_soa(pts, 3),
                  dist_tiled(pts, KernelVariant(VariantId.TILED, tile_size=64), 2),
                  dist_tiled(pts, KernelVariant(VariantId.TILED_UNROLLED, tile_size=48,
                                                unroll_width=5), 3)):
        assert np.array_equal(base.values.view(np.uint32), other.values.view(np.uint32)), key
    nbr, valid = build_clusters_from_dist(base, params, 2)
    bits, counts = nbr.bits.copy(), nbr.neighbor_count.copy()  # merge_iterative mutates nbr
    labels = merge_iterative(nbr, valid, 2).labels
    store[f"{key}/points"] = coords
    store[f"{key}/params"] = np.array([eps, eps_sq, min_pts], dtype=np.float64)
    store[f"{key}/dist"] = base.values
    store[f"{key}/bits"] = bits
    store[f"{key}/counts"] = counts.astype(np.int64)
    store[f"{key}/labels"] = labels.astype(np.int64)
    print(f"{key}: n={pts.n} clusters={labels.max() + 1} in-range={int(counts.sum())}")


def main():
    s = {}
    # 3-4-5 triangle: d^2 = 25 exactly (test_kernels.py:69-72), inclusive at 25
    case(s, "kat345", [[0, 0, 0], [3, 4, 0], [6, 8, 0], [0, 0, 5]], 5.0, 25.0, 2)
    # integer lattice with exact ties at eps^2 = 4 (test_kernels.py:174-183)
    g = np.array([[x, y, z] for x in range(4) for y in range(4) for z in range(2)], dtype=float)
    case(s, "lattice", g, 2.0, 4.0, 3)
    # ragged n (not a multiple of 4 or 8), blobs + noise, far from the origin
    b = generate_blobs(257, 3, 0.4, 0.2, 11).coords_aos + np.array([100.0, -50.0, 7.0])
    case(s, "blobs257", b, 0.5, 0.25, 4)
    rng = np.random.default_rng(5)
    case(s, "uniform101", rng.uniform(-3, 3, (101, 3)), 1.1, 1.1 * 1.1, 3)
    path = os.path.join(HERE, "dist.npz")
    np.savez_compressed(path, **s)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    sys.exit(main())
