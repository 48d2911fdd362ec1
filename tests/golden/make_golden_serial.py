"""Golden outputs of the reference's float64 oracle serial_dbscan (oracle.py:48-111),
made by EXECUTING THE REFERENCE:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_serial.py

Cases: C1 (2-D, z-padded for the reference; padding is bit-neutral in float64 too),
the 4x4x2 exact-tie lattice, unfiltered random blob sets and the CLI bench shape
generate_blobs(n, 3, 0.03, 0.02, seed). Writes tests/golden/serial.npz with the
inputs' generator arguments, labels and core counts.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from densescan import PointSet, serial_dbscan, validate_params  # noqa: E402

from paper_1506_02226_b200.datasets import generate_blobs  # noqa: E402

# name -> (n, k, spread, noise, seed, d, scale, eps, min_pts)
SPECS = {
    "c1": (10_000, 4, 0.5, 0.0, 1, 2, 1.0, 0.3, 4),
    "bench500": (500, 3, 0.03, 0.02, 0, 3, 1.0, 0.05, 4),
    "bench2000": (2000, 3, 0.03, 0.02, 7, 3, 1.0, 0.02, 5),
    "r2d": (3000, 6, 0.4, 0.1, 11, 2, 1.0, 0.25, 6),
    "r3d_scaled": (2500, 5, 0.3, 0.05, 12, 3, 10.0, 1.5, 5),
    "r1d": (1500, 3, 0.2, 0.1, 13, 1, 1.0, 0.02, 3),
}


def pad3(c):
    out = np.zeros((c.shape[0], 3))
    out[:, : c.shape[1]] = c
    return out


def main():
    out = {"names": np.array(list(SPECS) + ["lattice"])}
    for name, (n, k, spread, noise, seed, d, scale, eps, min_pts) in SPECS.items():
        c = generate_blobs(n, k, spread, noise, seed, d).coords_aos * scale
        lab, tr = serial_dbscan(PointSet(pad3(c)), validate_params(eps, min_pts))
        out[f"{name}/spec"] = np.array([n, k, spread, noise, seed, d, scale, eps, min_pts])
        out[f"{name}/labels"] = lab.labels
        out[f"{name}/cores"] = np.int64(tr.core_count)
    g = np.array([[x, y, z] for x in range(4) for y in range(4) for z in range(2)], float)
    lab, tr = serial_dbscan(PointSet(g), validate_params(2.0, 5))
    out["lattice/points"] = g
    out["lattice/labels"] = lab.labels
    out["lattice/cores"] = np.int64(tr.core_count)
    np.savez_compressed(os.path.join(HERE, "serial.npz"), **out)
    print("wrote serial.npz")


if __name__ == "__main__":
    main()
