"""Golden outcomes of the reference's argument validation — made by EXECUTING THE
REFERENCE (reference core.py:86-93 validate_params, pipeline.py:30-41 PipelineConfig).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_params.py

Writes tests/golden/params.json: for every (type, value) descriptor of
`descriptors()` the reference's outcome — accepted (eps, eps_sq, min_pts /
threads) or the InvalidParams field / ValueError it raised. tests/test_api.py
rebuilds the same inputs and checks the drop-in against it.
"""

from __future__ import annotations

import json
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

KINDS = {
    "int": int, "float": float, "bool": bool, "str": str,
    "none": lambda v: None,
    "np.float64": np.float64, "np.float32": np.float32, "np.float16": np.float16,
    "np.int64": np.int64, "np.int32": np.int32, "np.uint8": np.uint8, "np.bool_": np.bool_,
}


def make(kind, value):
    return KINDS[kind](value)


def descriptors():
    vals = []
    for kind in ("int", "float", "bool", "np.float64", "np.float32", "np.float16", "np.int64",
                 "np.int32", "np.uint8", "np.bool_"):
        for v in (1, 0, 3):
            vals.append((kind, v))
    vals += [("float", 0.3), ("float", -1.0), ("float", math.inf), ("float", math.nan),
             ("float", 2.5), ("np.float64", 0.3), ("np.float32", 0.3), ("str", "1"),
             ("none", 0), ("bool", False)]
    return vals


def outcome(fn):
    try:
        return {"ok": fn()}
    except Exception as e:  # noqa: BLE001
        return {"error": type(e).__name__, "field": getattr(e, "field", None)}


def main():
    from densescan import KernelVariant, PipelineConfig, VariantId, validate_params
    rows = []
    for kind, v in descriptors():
        x = make(kind, v)

        def eps_case(x=x):
            p = validate_params(x, 4)
            return [p.eps, p.eps_sq, p.min_pts]

        def pts_case(x=x):
            p = validate_params(1.0, x)
            return [p.eps, p.eps_sq, p.min_pts]

        def thr_case(x=x):
            return int(PipelineConfig(variant=KernelVariant(VariantId.FUSED), threads=x).threads)

        rows.append({"kind": kind, "value": v if not (isinstance(v, float) and not math.isfinite(v))
                     else repr(v), "eps": outcome(eps_case), "min_pts": outcome(pts_case),
                     "threads": outcome(thr_case)})
    with open(os.path.join(HERE, "params.json"), "w") as fh:
        json.dump(rows, fh, indent=0)
    print(f"wrote params.json ({len(rows)} cases)")


if __name__ == "__main__":
    main()
