"""CPU oracle for the densescan hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module, and only as the checker or the timed
CPU baseline. The product package (paper_1506_02226_b200) never imports it
and has no CPU fallback.

What it restates (reference = /root/reference/pkg/src/densescan):
  * narrowing:  float64 -> float32 round-to-nearest once, kernels.py:148-150
  * threshold:  thr32 = float32(eps_sq), eps_sq = float64(eps) * float64(eps),
                core.py:93 + kernels.py:355/385
  * ALGEBRAIC:  P = ((x0*x0 + x1*x1) + x2*x2) ...  (kernels.py:388-391)
                X = 2*x                            (kernels.py:392-395)
                cross = ((X0*x0 + X1*x1) + X2*x2) ...,
                d2 = (T + P) - cross, bit = d2 <= eps32  (kernels.py:409-417)
  * DIRECT:     dx = x_col - x_row, d2 = ((dx0^2 + dx1^2) + dx2^2) ...
                (kernels.py:197-210, 367-371)
    every operation a separately rounded float32 op (numpy ufuncs: no FMA);
    the d-dim forms extend the 3-term sums left to right.
  * counts:     row popcount incl. self, int64; core = counts >= min_pts
                (kernels.py:331-335)
  * merge:      labels of merge_iterative (merge.py:133-166): clusters are the
                connected components of the core-core in-range relation
                (SPEC.md merge contract), non-core points take
                the label of their lowest-indexed in-range core
                (_attach_borders, merge.py:116-130), then canonicalize
                (core.py:116-132).
  * bit layout: reference NeighborhoodMatrix rows, numpy packbits MSB-first,
                ceil(n/8) bytes per row (_bitmat.py:4-7, 13-27).

Parity pinning: tests/golden/make_golden.py runs the reference itself on the
KATs of its own test-suite, on C1, on exact-tie lattices, on large-offset data
and on unfiltered random instances; tests/test_oracle_golden.py checks this
oracle bit-for-bit against those fixtures (bits, counts, labels).
"""

from __future__ import annotations

import numpy as np

ALGEBRAIC = 1
DIRECT = 0
NOISE = -1


def narrow(coords) -> np.ndarray:
    """float64 (n, d) -> float32 (n, d), round-to-nearest-even (kernels.py:148-150)."""
    return np.ascontiguousarray(np.asarray(coords, dtype=np.float64).astype(np.float32))


def thr32(eps_sq: float) -> np.float32:
    """float32(float64 eps*eps): DbscanParams.eps_sq narrowed (kernels.py:355/385)."""
    return np.float32(float(eps_sq))


def sq_norms(p32: np.ndarray) -> np.ndarray:
    """P[j] = ((c0*c0 + c1*c1) + c2*c2) ... in float32 (kernels.py:388-391)."""
    acc = p32[:, 0] * p32[:, 0]
    for k in range(1, p32.shape[1]):
        acc = acc + p32[:, k] * p32[:, k]
    return acc.astype(np.float32)


def block_d2_algebraic(rows: np.ndarray, cols: np.ndarray,
                       norm_rows: np.ndarray, norm_cols: np.ndarray) -> np.ndarray:
    """(T_row + P_col) - ((X0*x0 + X1*x1) + ...) for a rows x cols block (kernels.py:403-417)."""
    two = np.float32(2.0)
    dbl = two * rows
    cross = dbl[:, 0:1] * cols[None, :, 0]
    for k in range(1, rows.shape[1]):
        cross = cross + dbl[:, k:k + 1] * cols[None, :, k]
    return (norm_rows[:, None] + norm_cols[None, :]) - cross


def block_d2_direct(rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """((dx0^2 + dx1^2) + ...) with dx = col - row (kernels.py:197-210)."""
    dx = cols[None, :, 0] - rows[:, 0:1]
    acc = dx * dx
    for k in range(1, rows.shape[1]):
        dx = cols[None, :, k] - rows[:, k:k + 1]
        acc = acc + dx * dx
    return acc


def _blocks(n: int, block: int):
    for r0 in range(0, n, block):
        yield r0, min(r0 + block, n)


def in_range_block(p32, norms, r0, r1, thr, formula, c0=0, c1=None) -> np.ndarray:
    c1 = p32.shape[0] if c1 is None else c1
    if formula == ALGEBRAIC:
        d2 = block_d2_algebraic(p32[r0:r1], p32[c0:c1], norms[r0:r1], norms[c0:c1])
    else:
        d2 = block_d2_direct(p32[r0:r1], p32[c0:c1])
    assert d2.dtype == np.float32
    return d2 <= thr


def neighborhood(coords, eps_sq: float, formula: int = ALGEBRAIC, block: int = 256,
                 want_bits: bool = True):
    """Stage 1+2 (fused_build / fused_build_algebraic, kernels.py:311-337, 420-442).

    Returns (bits, counts): bits in the reference layout (uint8 [n, ceil(n/8)],
    MSB-first) or None, counts int64 incl. self.
    """
    p32 = narrow(coords)
    n = p32.shape[0]
    thr = thr32(eps_sq)
    norms = sq_norms(p32)
    counts = np.empty(n, dtype=np.int64)
    bits = np.empty((n, (n + 7) // 8), dtype=np.uint8) if want_bits else None
    for r0, r1 in _blocks(n, block):
        hit = in_range_block(p32, norms, r0, r1, thr, formula)
        counts[r0:r1] = hit.sum(axis=1)
        if want_bits:
            bits[r0:r1] = np.packbits(hit, axis=-1)
    return bits, counts


def core_edges(coords, eps_sq: float, core: np.ndarray, formula: int = ALGEBRAIC,
               block: int = 256):
    """All in-range (i, j) with i < j and both core, plus the lowest in-range core
    of every non-core point (-1 if none). Recomputes distances row block by
    row block so nothing n x n is stored."""
    p32 = narrow(coords)
    n = p32.shape[0]
    thr = thr32(eps_sq)
    norms = sq_norms(p32)
    src, dst = [], []
    border = np.full(n, -1, dtype=np.int64)
    core_idx = np.nonzero(core)[0]
    if core_idx.size == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64), border
    for r0, r1 in _blocks(n, block):
        hit = in_range_block(p32, norms, r0, r1, thr, formula)
        hit &= core[None, :]
        rows = np.arange(r0, r1)
        rc = core[r0:r1]
        ii, jj = np.nonzero(hit[rc])
        ii = rows[rc][ii]
        keep = jj > ii
        src.append(ii[keep])
        dst.append(jj[keep])
        nc = ~rc
        if nc.any():
            sub = hit[nc]
            has = sub.any(axis=1)
            first = sub.argmax(axis=1)
            border[rows[nc][has]] = first[has]
    return np.concatenate(src), np.concatenate(dst), border


def components(n: int, src: np.ndarray, dst: np.ndarray) -> np.ndarray:
    """Root id (minimum member index) per node of the undirected graph (src, dst)."""
    parent = np.arange(n, dtype=np.int64)

    def find(x):
        root = x
        while parent[root] != root:
            root = parent[root]
        while parent[x] != root:
            parent[x], x = root, parent[x]
        return root

    if src.size:
        try:
            from scipy.sparse import coo_matrix
            from scipy.sparse.csgraph import connected_components
            g = coo_matrix((np.ones(src.size, dtype=np.int8), (src, dst)), shape=(n, n))
            _, comp = connected_components(g, directed=False)
            # re-express each component by its minimum member index
            first = np.full(comp.max() + 1, n, dtype=np.int64)
            np.minimum.at(first, comp, np.arange(n))
            return first[comp]
        except ImportError:  # pragma: no cover - scipy is in the image
            for a, b in zip(src.tolist(), dst.tolist()):
                ra, rb = find(a), find(b)
                if ra != rb:
                    parent[max(ra, rb)] = min(ra, rb)
            return np.array([find(i) for i in range(n)], dtype=np.int64)
    return parent


def canonical(labels: np.ndarray) -> np.ndarray:
    """First-appearance renumbering, NOISE kept (core.py:116-132)."""
    labels = np.asarray(labels, dtype=np.int64)
    out = np.full(labels.shape, NOISE, dtype=np.int64)
    keep = labels != NOISE
    if keep.any():
        vals = labels[keep]
        uniq, first = np.unique(vals, return_index=True)
        rank = np.empty(uniq.size, dtype=np.int64)
        rank[np.argsort(first, kind="stable")] = np.arange(uniq.size)
        out[keep] = rank[np.searchsorted(uniq, vals)]
    return out


def labels_from_core_graph(n, core, src, dst, border) -> np.ndarray:
    root = components(n, src, dst)
    labels = np.full(n, NOISE, dtype=np.int64)
    labels[core] = root[core]
    hit = border >= 0
    labels[hit] = root[border[hit]]
    return canonical(labels)


def merge_labels(bits: np.ndarray, counts: np.ndarray, min_pts: int) -> np.ndarray:
    """Stage 3 from a reference-layout NeighborhoodMatrix (merge.py:133-166)."""
    n = counts.shape[0]
    core = counts >= min_pts
    src, dst = [], []
    border = np.full(n, -1, dtype=np.int64)
    for r0, r1 in _blocks(n, 512):
        hit = np.unpackbits(bits[r0:r1], axis=-1, count=n).view(bool) & core[None, :]
        rows = np.arange(r0, r1)
        rc = core[r0:r1]
        ii, jj = np.nonzero(hit[rc])
        ii = rows[rc][ii]
        keep = jj > ii
        src.append(ii[keep])
        dst.append(jj[keep])
        nc = ~rc
        if nc.any():
            sub = hit[nc]
            has = sub.any(axis=1)
            border[rows[nc][has]] = sub.argmax(axis=1)[has]
    src = np.concatenate(src) if src else np.empty(0, np.int64)
    dst = np.concatenate(dst) if dst else np.empty(0, np.int64)
    return labels_from_core_graph(n, core, src, dst, border)


def dbscan(coords, eps_sq: float, min_pts: int, formula: int = ALGEBRAIC):
    """run_dbscan(points, validate_params(eps, min_pts), config) with the given
    formula (pipeline.py:70-92). Returns (canonical labels int64, counts int64)."""
    _, counts = neighborhood(coords, eps_sq, formula, want_bits=False)
    core = counts >= min_pts
    src, dst, border = core_edges(coords, eps_sq, core, formula)
    return labels_from_core_graph(counts.shape[0], core, src, dst, border), counts


def unpack_ref_bits(bits: np.ndarray, n: int) -> np.ndarray:
    return np.unpackbits(bits, axis=-1, count=n).view(bool)


# ---- Warshall backend (reference merge.py:169-238) --------------------------------

def core_adjacency(bits: np.ndarray, valid: np.ndarray):
    """build_core_adjacency (merge.py:179-188): (core_indices int64, packbits rows of
    the bits restricted to core rows and columns)."""
    valid = np.asarray(valid, dtype=bool)
    n = valid.shape[0]
    ci = np.nonzero(valid)[0].astype(np.int64)
    rows = np.unpackbits(bits[ci], axis=-1, count=n).view(bool)[:, ci]
    return ci, np.packbits(rows, axis=-1)


def warshall_closure_bits(adj_bits: np.ndarray, m: int) -> np.ndarray:
    """warshall_closure (merge.py:191-215): for each pivot k in order, every row with
    bit k set (other than k itself) ORs in row k. Returns packbits rows."""
    rel = np.unpackbits(adj_bits, axis=-1, count=m).view(bool).copy()
    for k in range(m):
        col = rel[:, k].copy()
        col[k] = False
        rows = np.nonzero(col)[0]
        if rows.size:
            rel[rows] |= rel[k]
    return np.packbits(rel, axis=-1)


# ---- the reference's run_dbscan flow, threaded: the CPU baseline of bench.py -------

def dbscan_reference_flow(coords, eps_sq: float, min_pts: int, formula: int = ALGEBRAIC,
                          threads: int = 1, block: int = 256):
    """run_dbscan(points, params, default_config()) as the reference executes it
    (pipeline.py:70-92), for timing on the host's cores: stage 1+2 materialises the
    packbits NeighborhoodMatrix row block by row block of 256 in a fork-join pool over
    contiguous row ranges (kernels.py:311-337, _parallel.py:16-39); stage 3 reads the
    packed rows masked by the core flags, takes core-core pairs as edges and the first
    in-range core of every non-core row (merge.py:116-166 contract), then components
    and first-appearance ids (core.py:116-132). Returns (labels, counts, seconds of
    stage 1+2, seconds of stage 3).
    """
    import time
    from concurrent.futures import ThreadPoolExecutor

    t0 = time.perf_counter()
    p32 = narrow(coords)
    n = p32.shape[0]
    thr = thr32(eps_sq)
    norms = sq_norms(p32)
    rb = (n + 7) // 8
    bits = np.empty((n, rb), dtype=np.uint8)
    counts = np.empty(n, dtype=np.int64)
    bounds = np.linspace(0, n, max(1, min(threads, n)) + 1).astype(np.int64)

    def stage12(w):
        for r0 in range(int(bounds[w]), int(bounds[w + 1]), block):
            r1 = min(r0 + block, int(bounds[w + 1]))
            hit = in_range_block(p32, norms, r0, r1, thr, formula)
            counts[r0:r1] = hit.sum(axis=1)
            bits[r0:r1] = np.packbits(hit, axis=-1)

    with ThreadPoolExecutor(max_workers=len(bounds) - 1) as pool:
        list(pool.map(stage12, range(len(bounds) - 1)))
    t1 = time.perf_counter()

    core = counts >= min_pts
    core_pk = np.packbits(core)
    edges, borders = [], []

    def stage3(r0):
        r1 = min(r0 + 512, n)
        masked = bits[r0:r1] & core_pk[None, :]
        rc = core[r0:r1]
        rows, cols = np.nonzero(masked[rc])
        rows = np.nonzero(rc)[0][rows]
        vals = masked[rows, cols]
        if vals.size:
            unpacked = np.unpackbits(vals[:, None], axis=1).view(bool)
            k, bit = np.nonzero(unpacked)
            i = rows[k] + r0
            j = cols[k].astype(np.int64) * 8 + bit
            keep = j > i
            edges.append((i[keep], j[keep]))
        nc = np.nonzero(~rc)[0]
        if nc.size:
            sub = masked[nc]
            nz = sub != 0
            has = nz.any(axis=1)
            first = nz.argmax(axis=1)
            v = sub[np.arange(nc.size), first]
            lead = np.unpackbits(v[:, None], axis=1).argmax(axis=1)
            borders.append((nc[has] + r0, first[has].astype(np.int64) * 8 + lead[has]))

    with ThreadPoolExecutor(max_workers=max(1, threads)) as pool:
        list(pool.map(stage3, range(0, n, 512)))
    src = np.concatenate([e[0] for e in edges]) if edges else np.empty(0, np.int64)
    dst = np.concatenate([e[1] for e in edges]) if edges else np.empty(0, np.int64)
    border = np.full(n, -1, dtype=np.int64)
    for p, c in borders:
        border[p] = c
    labels = labels_from_core_graph(n, core, src, dst, border)
    t2 = time.perf_counter()
    return labels, counts, t1 - t0, t2 - t1
