"""ctypes wrapper of the C oracle (ds_oracle.c) — TEST INFRASTRUCTURE ONLY.

Same contract as densescan_oracle.dbscan / neighborhood counts, multithreaded,
for sizes the numpy oracle cannot reach in seconds. Builds itself with `make`
when the library is missing (gcc is on both the build and the GPU box).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libds_oracle.so")
_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        lib = ctypes.CDLL(LIB)
        vp, i64, c_int, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.dso_counts.argtypes = [vp, i64, c_int, dbl, c_int, c_int, vp]
        lib.dso_dbscan.argtypes = [vp, i64, c_int, dbl, i64, c_int, c_int, vp, vp]
        _lib = lib
    return _lib


def threads() -> int:
    return int(os.environ.get("DSO_THREADS", os.cpu_count() or 1))


def counts(coords, eps_sq: float, formula: int = 1, nthreads: int | None = None) -> np.ndarray:
    c = np.ascontiguousarray(coords, dtype=np.float64)
    out = np.empty(c.shape[0], dtype=np.int64)
    load().dso_counts(c.ctypes.data, c.shape[0], c.shape[1], float(eps_sq), int(formula),
                      int(nthreads or threads()), out.ctypes.data)
    return out


def dbscan(coords, eps_sq: float, min_pts: int, formula: int = 1, nthreads: int | None = None):
    c = np.ascontiguousarray(coords, dtype=np.float64)
    labels = np.empty(c.shape[0], dtype=np.int64)
    cnt = np.empty(c.shape[0], dtype=np.int64)
    load().dso_dbscan(c.ctypes.data, c.shape[0], c.shape[1], float(eps_sq), int(min_pts),
                      int(formula), int(nthreads or threads()), labels.ctypes.data, cnt.ctypes.data)
    return labels, cnt
