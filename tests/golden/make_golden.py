"""Generate golden fixtures by executing the REFERENCE densescan package.

Runs only in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--c2]

Every fixture records the reference's own outputs (fused_build /
fused_build_algebraic bits + counts, run_dbscan labels) for inputs that are
either stored verbatim or regenerated bit-exactly by
paper_1506_02226_b200.datasets.generate_blobs (verified equal to the
reference's generate_blobs at d=3 by this script before anything is written).

The fixtures pin the oracle (tests/test_oracle_golden.py) and the GPU path
(tests/test_gpu_parity.py). Nothing at test time reads /root/reference.

Outputs (all under tests/golden/):
  kat.npz       the reference test-suite's known-answer cases
  c1.npz        C1 (2-D, z-padded for the reference): counts, labels, bits sha256
  lattice.npz   exact-tie integer lattices and 0.1-pitch near-tie lattices
  random.npz    unfiltered random blob sets incl. offset/scaled data
  blob23040.npz the acceptance fixture generate_blobs(23040, 3, .03, .02, 1)
  c2.npz        (--c2, ~10 min) C2 at full size, ALGEBRAIC
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import densescan as ref  # noqa: E402  (the reference, via PYTHONPATH)
from densescan import (DbscanParams, KernelVariant, PointSet, VariantId,  # noqa: E402
                       fused_build, fused_build_algebraic, merge_iterative)

from paper_1506_02226_b200.datasets import generate_blobs  # noqa: E402

FORMULAS = {"alg": VariantId.FUSED_ALGEBRAIC, "dir": VariantId.FUSED}


def pad3(c: np.ndarray) -> np.ndarray:
    c = np.asarray(c, dtype=np.float64)
    if c.shape[1] == 3:
        return c
    out = np.zeros((c.shape[0], 3), dtype=np.float64)
    out[:, : c.shape[1]] = c
    return out


def ref_run(coords: np.ndarray, eps: float, eps_sq: float, min_pts: int, vid: VariantId,
            mem_cap=None):
    """bits, counts, labels exactly as the reference computes them."""
    points = PointSet(pad3(coords))
    params = DbscanParams(eps=eps, eps_sq=eps_sq, min_pts=min_pts)
    variant = KernelVariant(vid)
    threads = os.cpu_count() or 1
    build = fused_build_algebraic if vid is VariantId.FUSED_ALGEBRAIC else fused_build
    nbr, valid = build(points, params, variant, threads, mem_cap)
    counts = nbr.neighbor_count.copy()
    bits = nbr.bits.copy()
    labels = merge_iterative(nbr, valid, threads).labels
    return bits, counts, labels


def sha(bits: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(bits).tobytes()).hexdigest()


def check_generator():
    for args in [(1000, 3, 0.05, 0.1, 42), (23040, 3, 0.03, 0.02, 1), (777, 5, 0.2, 0.3, 9),
                 (10, 1, 0.0, 0.0, 1), (4000, 27, 0.1, 0.05, 3)]:
        a = ref.generate_blobs(*args).coords_aos
        b = generate_blobs(*args, d=3).coords_aos
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), args
    print("generator: bit-identical to reference generate_blobs at d=3")


def save(name: str, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def add_case(store: dict, key: str, coords, eps, eps_sq, min_pts, keep_bits=True):
    coords = np.asarray(coords, dtype=np.float64)
    store[f"{key}/points"] = coords
    store[f"{key}/params"] = np.array([eps, eps_sq, min_pts], dtype=np.float64)
    for fname, vid in FORMULAS.items():
        bits, counts, labels = ref_run(coords, eps, eps_sq, min_pts, vid)
        if keep_bits:
            store[f"{key}/{fname}/bits"] = bits
        store[f"{key}/{fname}/bits_sha"] = np.array(sha(bits))
        store[f"{key}/{fname}/counts"] = counts.astype(np.int32)
        store[f"{key}/{fname}/labels"] = labels.astype(np.int32)


def make_kat():
    s = {}
    # test_kernels.py:69-72, 124-137 — 3-4-5 triangle, inclusive / exclusive
    add_case(s, "tri345_in", [[0, 0, 0], [3, 4, 0]], 5.0, 25.0, 2)
    add_case(s, "tri345_out", [[0, 0, 0], [3, 4, 0]], 4.9, 24.0, 2)
    # test_kernels.py:139-144 — MinPts met exactly
    add_case(s, "minpts_exact", [[0, 0, 0], [1, 0, 0]], 1.0, 1.0, 2)
    # test_kernels.py:174-183 — integer lattice, exact ties at eps^2 = 4
    grid = np.stack(np.meshgrid(range(4), range(4), range(2)), axis=-1).reshape(-1, 3)
    add_case(s, "lattice_ties", grid.astype(float), 2.0, 4.0, 3)
    # test_kernels.py:192-202 — algebraic identity pair
    add_case(s, "alg_pair_in", [[1, 2, 3], [4, 6, 3]], 5.0, 25.0, 2)
    add_case(s, "alg_pair_out", [[1, 2, 3], [4, 6, 3]], 4.99, 24.99, 2)
    # test_merge.py:46-58, test_pipeline.py:40-52 — chains, groups, singleton
    add_case(s, "collinear", [[0, 0, 0], [1, 0, 0], [2, 0, 0]], 1.2, 1.2 * 1.2, 2)
    add_case(s, "two_groups", [[0, 0, 0], [1, 0, 0], [20, 0, 0], [21, 0, 0]], 1.5, 2.25, 2)
    add_case(s, "single", [[4.0, 5.0, 6.0]], 3.0, 9.0, 1)
    add_case(s, "all_noise", [[0, 0, 0], [10, 0, 0]], 1.0, 1.0, 2)
    # test_oracle.py:64-82 — border ties to its lowest-indexed core
    border = [[0.0, 0, 0], [-0.1, 0, 0], [-0.2, 0, 0], [-0.3, 0, 0],
              [2.0, 0, 0], [2.1, 0, 0], [2.2, 0, 0], [2.3, 0, 0], [1.0, 0, 0]]
    add_case(s, "border_tie", border, 1.0, 1.0, 4)
    # test_merge.py:195-206 and test_core.py:174-179 — 3-blob goldens
    add_case(s, "blobs3_a", generate_blobs(1000, 3, 0.03, 0.0, 42).coords_aos, 0.6, 0.36, 5,
             keep_bits=False)
    add_case(s, "blobs3_b", generate_blobs(1000, 3, 0.05, 0.1, 42).coords_aos, 0.1, 0.01, 5,
             keep_bits=False)
    rng = np.random.default_rng(20240817)
    add_case(s, "isolated", rng.normal(size=(12, 3)) * 100, 1e-3, 1e-6, 2)
    s["names"] = np.array(sorted({k.split("/")[0] for k in s}))
    save("kat.npz", **s)


def make_c1():
    pts = generate_blobs(10_000, 4, 0.5, 0.0, 1, 2).coords_aos
    out = {"gen": np.array([10_000, 4, 0.5, 0.0, 1, 2], dtype=np.float64),
           "params": np.array([0.3, 0.3 * 0.3, 4])}
    for fname, vid in FORMULAS.items():
        t0 = time.perf_counter()
        bits, counts, labels = ref_run(pts, 0.3, 0.3 * 0.3, 4, vid)
        print(f"C1 {fname}: {time.perf_counter() - t0:.1f}s, clusters="
              f"{len(set(labels.tolist()) - {-1})} noise={(labels == -1).sum()}")
        out[f"{fname}/bits_sha"] = np.array(sha(bits))
        out[f"{fname}/counts"] = counts.astype(np.int32)
        out[f"{fname}/labels"] = labels.astype(np.int32)
        # a row sample of the reference bits, to locate a mismatch quickly
        out[f"{fname}/bits_rows0_64"] = bits[:64]
    save("c1.npz", **out)


def make_lattice():
    s = {}
    # exact ties: integer lattices, eps^2 on lattice distances
    g2 = np.stack(np.meshgrid(np.arange(30), np.arange(30)), axis=-1).reshape(-1, 2)
    for k, e2 in enumerate([1.0, 2.0, 4.0, 5.0]):
        add_case(s, f"int_e{k}", g2.astype(float), float(np.sqrt(e2)), e2, 3, keep_bits=False)
    # the same lattice far from the origin: algebraic cancellation regime
    add_case(s, "int_far", g2.astype(float) + 1000.0, 1.0, 1.0, 3, keep_bits=False)
    # 0.1-pitch lattice: pair distances straddle eps^2 after float32 rounding
    g01 = g2.astype(float) * 0.1
    for k, eps in enumerate([0.1, 0.2, np.sqrt(0.02), 0.3]):
        add_case(s, f"dec_e{k}", g01, float(eps), float(eps) * float(eps), 4, keep_bits=False)
        add_case(s, f"dec_far_e{k}", g01 + 37.3, float(eps), float(eps) * float(eps), 4,
                 keep_bits=False)
    s["names"] = np.array(sorted({k.split("/")[0] for k in s}))
    save("lattice.npz", **s)


def make_random(count=48):
    rng = np.random.default_rng(1506_02226)
    s = {}
    specs = []
    for t in range(count):
        n = int(np.exp(rng.uniform(0.0, np.log(1500))))
        n = max(1, n)
        k = int(rng.integers(1, min(5, n) + 1))
        spread = float(rng.uniform(0.02, 0.3))
        noise = float(rng.uniform(0.0, 0.3))
        seed = int(rng.integers(2**31))
        d = int(rng.choice([2, 3]))
        scale = float(rng.choice([1.0, 10.0]))
        offset = float(rng.choice([0.0, 3.0, 100.0]))
        eps = float(rng.uniform(0.02, 0.4)) * scale
        min_pts = int(rng.integers(1, 9))
        specs.append([n, k, spread, noise, seed, d, scale, offset, eps, min_pts])
        coords = generate_blobs(n, k, spread, noise, seed, d).coords_aos * scale + offset
        add_case(s, f"r{t:03d}", coords, eps, eps * eps, min_pts, keep_bits=n <= 200)
        del s[f"r{t:03d}/points"]  # regenerated from the spec at test time
    s["specs"] = np.array(specs, dtype=np.float64)
    save("random.npz", **s)


def make_blob23040():
    pts = generate_blobs(23040, 3, 0.03, 0.02, 1).coords_aos
    out = {"params": np.array([0.1, 0.01, 8])}
    for fname, vid in FORMULAS.items():
        bits, counts, labels = ref_run(pts, 0.1, 0.1 * 0.1, 8, vid)
        out[f"{fname}/bits_sha"] = np.array(sha(bits))
        out[f"{fname}/counts"] = counts.astype(np.int32)
        out[f"{fname}/labels"] = labels.astype(np.int32)
    save("blob23040.npz", **out)


def make_c2():
    pts = generate_blobs(200_000, 16, 1.0, 0.10, 2, 2).coords_aos
    t0 = time.perf_counter()
    bits, counts, labels = ref_run(pts, 0.3, 0.3 * 0.3, 8, VariantId.FUSED_ALGEBRAIC,
                                   mem_cap=6 * 10**9)
    dt = time.perf_counter() - t0
    print(f"C2 alg: {dt:.1f}s clusters={len(set(labels.tolist()) - {-1})} "
          f"noise={(labels == -1).sum()}")
    save("c2.npz", counts=counts.astype(np.int32), labels=labels.astype(np.int32),
         bits_sha=np.array(sha(bits)), seconds=np.array(dt),
         threads=np.array(os.cpu_count()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2", action="store_true", help="only the long C2 run")
    args = ap.parse_args()
    check_generator()
    if args.c2:
        make_c2()
        return
    make_kat()
    make_c1()
    make_lattice()
    make_random()
    make_blob23040()


if __name__ == "__main__":
    main()
