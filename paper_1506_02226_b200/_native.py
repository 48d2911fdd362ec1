"""ctypes binding of the sm_100a library (include/densescan_b200.h).

There is no CPU fallback: if the shared library is missing or cannot reach a
CUDA device, every entry point raises. Build it with `make -C
paper_1506_02226_b200/csrc` (or `python -c "import __graft_entry__ as g;
g.build()"`).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .core import DensescanError, DeviceError, InvalidParams

LIB_NAME = "libdensescan_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

DS_OK, DS_EINVAL, DS_ECAPACITY, DS_ECUDA, DS_EINCONSISTENT, DS_ENCCL = range(6)
DS_OPT_TILE_CULL, DS_OPT_SPATIAL_SORT, DS_OPT_CUDA_GRAPH, DS_OPT_EVENT_TIMING = 1, 2, 3, 4
DS_OPT_TEST_CAPACITY = 5
DS_OPT_STABLE_ORDER = 6
FORMULA_DIRECT, FORMULA_ALGEBRAIC = 0, 1

# every symbol the header declares; tests/test_abi.py checks the .so exports them
EXPORTS = (
    "ds_abi_version", "ds_build_info", "ds_last_error", "ds_last_capacity",
    "ds_ctx_create", "ds_ctx_destroy", "ds_ctx_set_option", "ds_ctx_get_option",
    "ds_host_register", "ds_host_unregister",
    "ds_run_dbscan", "ds_run_dbscan_device",
    "ds_fused_build", "ds_merge_bits", "ds_merge_bits_core", "ds_core_adjacency",
    "ds_warshall_closure", "ds_serial_dbscan", "ds_dist_matrix", "ds_dist_threshold", "ds_dist_build",
    "ds_tile_items", "ds_tile_side", "ds_shard_stage12",
    "ds_shard_stage3_local", "ds_shard_stage3_merge", "ds_shard_fold",
)


class Timings(ctypes.Structure):
    """Mirror of ds_timings."""

    _fields_ = [
        ("fused_ms", ctypes.c_double),
        ("merge_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("tile_ms", ctypes.c_double),
        ("h2d_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("pairs_evaluated", ctypes.c_int64),
        ("tiles_total", ctypes.c_int64),
        ("tiles_nonempty", ctypes.c_int64),
        ("words_emitted", ctypes.c_int64),
        ("core_count", ctypes.c_int64),
        ("cluster_count", ctypes.c_int64),
        ("device_bytes", ctypes.c_int64),
        ("unsafe_range", ctypes.c_int32),
        ("tile_launches", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None
_lib_lock = threading.Lock()

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_i64_p = ctypes.POINTER(ctypes.c_int64)
_c_u8_p = ctypes.POINTER(ctypes.c_uint8)


def load_library(path: str = LIB_PATH):
    """Load and prototype the library (no CUDA call is made here)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: the densescan sm_100a library is not built "
                "(run `make -C paper_1506_02226_b200/csrc`); there is no CPU fallback")
        lib = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        lib.ds_abi_version.restype = ctypes.c_int
        lib.ds_build_info.restype = ctypes.c_char_p
        lib.ds_last_error.restype = ctypes.c_char_p
        lib.ds_last_capacity.argtypes = [_c_i64_p, _c_i64_p]
        lib.ds_last_capacity.restype = None
        lib.ds_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
        lib.ds_ctx_create.restype = ctypes.c_int
        lib.ds_ctx_destroy.argtypes = [vp]
        lib.ds_ctx_destroy.restype = None
        lib.ds_host_register.argtypes = [vp, ctypes.c_size_t]
        lib.ds_host_register.restype = ctypes.c_int
        lib.ds_host_unregister.argtypes = [vp]
        lib.ds_host_unregister.restype = ctypes.c_int
        lib.ds_ctx_set_option.argtypes = [vp, ctypes.c_int32, ctypes.c_int64]
        lib.ds_ctx_set_option.restype = ctypes.c_int
        lib.ds_ctx_get_option.argtypes = [vp, ctypes.c_int32]
        lib.ds_ctx_get_option.restype = ctypes.c_int64
        lib.ds_run_dbscan.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_double,
                                      ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, vp, vp,
                                      ctypes.POINTER(Timings)]
        lib.ds_run_dbscan.restype = ctypes.c_int
        lib.ds_run_dbscan_device.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32,
                                             ctypes.c_double, ctypes.c_int64, ctypes.c_int32,
                                             ctypes.c_int64, vp, vp, ctypes.POINTER(Timings)]
        lib.ds_run_dbscan_device.restype = ctypes.c_int
        lib.ds_fused_build.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_double,
                                       ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, vp, vp, vp,
                                       ctypes.POINTER(Timings)]
        lib.ds_fused_build.restype = ctypes.c_int
        lib.ds_merge_bits.argtypes = [vp, vp, vp, vp, ctypes.c_int64, ctypes.c_int64, vp,
                                      ctypes.POINTER(Timings)]
        lib.ds_merge_bits.restype = ctypes.c_int
        lib.ds_merge_bits_core.argtypes = [vp, vp, vp, ctypes.c_int64, vp, ctypes.POINTER(Timings)]
        lib.ds_merge_bits_core.restype = ctypes.c_int
        lib.ds_core_adjacency.argtypes = [vp, vp, vp, ctypes.c_int64, ctypes.c_int64, vp, vp,
                                          ctypes.POINTER(Timings)]
        lib.ds_core_adjacency.restype = ctypes.c_int
        lib.ds_warshall_closure.argtypes = [vp, vp, ctypes.c_int64, vp, ctypes.POINTER(Timings)]
        lib.ds_warshall_closure.restype = ctypes.c_int
        lib.ds_serial_dbscan.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_double,
                                         ctypes.c_int64, vp, vp, ctypes.POINTER(Timings)]
        lib.ds_serial_dbscan.restype = ctypes.c_int
        lib.ds_dist_matrix.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, vp,
                                       ctypes.POINTER(Timings)]
        lib.ds_dist_matrix.restype = ctypes.c_int
        lib.ds_dist_threshold.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_double, ctypes.c_int64,
                                          ctypes.c_int64, vp, vp, vp, ctypes.POINTER(Timings)]
        lib.ds_dist_threshold.restype = ctypes.c_int
        lib.ds_dist_build.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_double,
                                      ctypes.c_int64, ctypes.c_int64, vp, vp, vp,
                                      ctypes.POINTER(Timings)]
        lib.ds_dist_build.restype = ctypes.c_int
        lib.ds_tile_items.argtypes = [ctypes.c_int64]
        lib.ds_tile_items.restype = ctypes.c_int64
        lib.ds_tile_side.restype = ctypes.c_int
        lib.ds_shard_stage12.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_double,
                                         ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int64, vp, vp, ctypes.POINTER(Timings)]
        lib.ds_shard_stage12.restype = ctypes.c_int
        lib.ds_shard_stage3_local.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int64, vp, vp, vp,
                                              ctypes.POINTER(Timings)]
        lib.ds_shard_stage3_local.restype = ctypes.c_int
        lib.ds_shard_stage3_merge.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int64, vp,
                                              ctypes.c_int32, vp, vp, vp, ctypes.POINTER(Timings)]
        lib.ds_shard_stage3_merge.restype = ctypes.c_int
        lib.ds_shard_fold.argtypes = [vp, vp, vp, ctypes.c_int64, vp]
        lib.ds_shard_fold.restype = ctypes.c_int
        if lib.ds_abi_version() != 1:
            raise ImportError(f"{path}: unexpected ABI version {lib.ds_abi_version()}")
        _lib = lib
        return lib


def raise_for(status: int, lib=None) -> None:
    if status == DS_OK:
        return
    lib = lib or load_library()
    msg = (lib.ds_last_error() or b"").decode("utf-8", "replace")
    if status == DS_ECAPACITY:
        from .kernels import CapacityExceeded
        req, cap = ctypes.c_int64(), ctypes.c_int64()
        lib.ds_last_capacity(ctypes.byref(req), ctypes.byref(cap))
        raise CapacityExceeded(int(req.value), int(cap.value))
    if status == DS_EINCONSISTENT:
        from .merge import InconsistentInput
        raise InconsistentInput(msg)
    if status == DS_EINVAL:
        field, _, rest = msg.partition(":")
        raise InvalidParams(field.strip() or "argument", rest.strip() or msg)
    if status in (DS_ECUDA, DS_ENCCL):
        raise DeviceError(msg)
    raise DensescanError(f"densescan status {status}: {msg}")


class Context:
    """One ds_ctx (device workspace + stream) per (host thread, device)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        self.device = int(device)
        handle = ctypes.c_void_p()
        raise_for(self.lib.ds_ctx_create(self.device, ctypes.byref(handle)), self.lib)
        self.handle = handle

    def close(self):
        if getattr(self, "handle", None):
            self.lib.ds_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def set_tile_cull(self, on: bool) -> None:
        """Bounding-box culling of provably empty tile pairs (default on; exact)."""
        self._schedule = None
        raise_for(self.lib.ds_ctx_set_option(self.handle, DS_OPT_TILE_CULL, 1 if on else 0),
                  self.lib)

    def tile_cull(self) -> bool:
        return self.lib.ds_ctx_get_option(self.handle, DS_OPT_TILE_CULL) == 1

    def set_spatial_sort(self, on: bool) -> None:
        """Visit points in Morton order (compact tiles; exact, default on)."""
        self._schedule = None
        raise_for(self.lib.ds_ctx_set_option(self.handle, DS_OPT_SPATIAL_SORT, 1 if on else 0),
                  self.lib)

    def set_event_timing(self, on: bool) -> None:
        """Stage timings from CUDA events between the kernels (default off: from the
        kernels' %globaltimer stamps; events cost device time)."""
        raise_for(self.lib.ds_ctx_set_option(self.handle, DS_OPT_EVENT_TIMING, 1 if on else 0),
                  self.lib)

    def set_cuda_graph(self, on: bool) -> None:
        """Record the device pipeline into a CUDA graph and replay it (default on)."""
        raise_for(self.lib.ds_ctx_set_option(self.handle, DS_OPT_CUDA_GRAPH, 1 if on else 0),
                  self.lib)

    def set_test_capacity(self, entries: int) -> None:
        """Test hook: start the next stage 1+2 from `entries` unit-list / word slots and
        at most double them per re-run (0: normal sizing)."""
        raise_for(self.lib.ds_ctx_set_option(self.handle, DS_OPT_TEST_CAPACITY, int(entries)),
                  self.lib)

    def set_stable_order(self, on: bool) -> None:
        """DS_OPT_STABLE_ORDER: always the stable radix sort for the spatial order (the
        default counting sort of small 1-2-D inputs orders points of one grid cell
        arbitrarily; results are identical, work counters may differ between calls)."""
        raise_for(self.lib.ds_ctx_set_option(self.handle, DS_OPT_STABLE_ORDER, 1 if on else 0),
                  self.lib)

    def configure(self, prune: bool = True, spatial_order: bool = True) -> None:
        """Set both schedule options; a no-op when they are unchanged since the last call
        (run_dbscan calls this every time)."""
        state = (bool(prune), bool(spatial_order))
        if getattr(self, "_schedule", None) == state:
            return
        self._schedule = None
        self.set_tile_cull(prune)
        self.set_spatial_sort(spatial_order)
        self._schedule = state

    def schedule(self) -> tuple[bool, bool]:
        """The current (prune, spatial_order) options of this context."""
        return (self.lib.ds_ctx_get_option(self.handle, DS_OPT_TILE_CULL) == 1,
                self.lib.ds_ctx_get_option(self.handle, DS_OPT_SPATIAL_SORT) == 1)

    # -- entry points --------------------------------------------------------
    def run_dbscan(self, coords: np.ndarray, eps_sq: float, min_pts: int, formula: int,
                   mem_cap: int, want_counts: bool = False):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        n, d = coords.shape
        labels = pinned_empty(n)
        counts = np.empty(n, dtype=np.int64) if want_counts else None
        t = Timings()
        st = self.lib.ds_run_dbscan(self.handle, coords.ctypes.data, n, d, float(eps_sq),
                                    int(min_pts), int(formula), int(mem_cap),
                                    labels.ctypes.data,
                                    counts.ctypes.data if counts is not None else None,
                                    ctypes.byref(t))
        raise_for(st, self.lib)
        return labels, counts, t

    def run_dbscan_device(self, coords_ptr: int, n: int, d: int, eps_sq: float, min_pts: int,
                          formula: int, mem_cap: int, labels_ptr: int, stream_ptr: int = 0):
        t = Timings()
        st = self.lib.ds_run_dbscan_device(self.handle, ctypes.c_void_p(coords_ptr), int(n),
                                           int(d), float(eps_sq), int(min_pts), int(formula),
                                           int(mem_cap), ctypes.c_void_p(labels_ptr),
                                           ctypes.c_void_p(stream_ptr or None), ctypes.byref(t))
        raise_for(st, self.lib)
        return t

    # -- multi-GPU shard stages (device pointers; see distributed.py) -----------
    def shard_stage12(self, coords_ptr, n, d, eps_sq, formula, rank, world, mem_cap,
                      counts_ptr, stream_ptr=0):
        t = Timings()
        st = self.lib.ds_shard_stage12(self.handle, ctypes.c_void_p(coords_ptr), int(n), int(d),
                                       float(eps_sq), int(formula), int(rank), int(world),
                                       int(mem_cap), ctypes.c_void_p(counts_ptr),
                                       ctypes.c_void_p(stream_ptr or None), ctypes.byref(t))
        raise_for(st, self.lib)
        return t

    def shard_stage3_local(self, counts_ptr, n, min_pts, parent_ptr, bmin_ptr, stream_ptr=0):
        t = Timings()
        st = self.lib.ds_shard_stage3_local(self.handle, ctypes.c_void_p(counts_ptr), int(n),
                                            int(min_pts), ctypes.c_void_p(parent_ptr),
                                            ctypes.c_void_p(bmin_ptr),
                                            ctypes.c_void_p(stream_ptr or None), ctypes.byref(t))
        raise_for(st, self.lib)
        return t

    def shard_stage3_merge(self, counts_ptr, n, min_pts, parents_ptr, nparents, bmin_ptr,
                           labels_ptr, stream_ptr=0):
        t = Timings()
        st = self.lib.ds_shard_stage3_merge(self.handle, ctypes.c_void_p(counts_ptr), int(n),
                                            int(min_pts), ctypes.c_void_p(parents_ptr),
                                            int(nparents), ctypes.c_void_p(bmin_ptr),
                                            ctypes.c_void_p(labels_ptr),
                                            ctypes.c_void_p(stream_ptr or None), ctypes.byref(t))
        raise_for(st, self.lib)
        return t

    def shard_fold(self, parent_ptr, other_ptr, n, stream_ptr=0):
        st = self.lib.ds_shard_fold(self.handle, ctypes.c_void_p(parent_ptr),
                                    ctypes.c_void_p(other_ptr), int(n),
                                    ctypes.c_void_p(stream_ptr or None))
        raise_for(st, self.lib)

    def fused_build(self, coords: np.ndarray, eps_sq: float, min_pts: int, formula: int,
                    mem_cap: int, want_bits: bool = True):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        n, d = coords.shape
        bits = np.empty((n, (n + 7) // 8), dtype=np.uint8) if want_bits else None
        counts = np.empty(n, dtype=np.int64)
        valid = np.empty(n, dtype=np.uint8)
        t = Timings()
        st = self.lib.ds_fused_build(self.handle, coords.ctypes.data, n, d, float(eps_sq),
                                     int(min_pts), int(formula), int(mem_cap),
                                     bits.ctypes.data if bits is not None else None,
                                     counts.ctypes.data, valid.ctypes.data, ctypes.byref(t))
        raise_for(st, self.lib)
        return bits, counts, valid.astype(bool), t

    def merge_bits(self, bits: np.ndarray, counts: np.ndarray, valid: np.ndarray, min_pts: int):
        n = counts.shape[0]
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        if bits.shape != (n, (n + 7) // 8):
            raise ValueError(f"bits must have shape {(n, (n + 7) // 8)}, got {bits.shape}")
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        valid8 = np.ascontiguousarray(valid, dtype=np.uint8)
        labels = np.empty(n, dtype=np.int64)
        t = Timings()
        st = self.lib.ds_merge_bits(self.handle, bits.ctypes.data, counts.ctypes.data,
                                    valid8.ctypes.data, n, int(min_pts), labels.ctypes.data,
                                    ctypes.byref(t))
        raise_for(st, self.lib)
        return labels, t


    def merge_bits_core(self, bits: np.ndarray, core: np.ndarray):
        """Union-find merge with the core set taken as given (merge_warshall)."""
        n = core.shape[0]
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        if bits.shape != (n, (n + 7) // 8):
            raise ValueError(f"bits must have shape {(n, (n + 7) // 8)}, got {bits.shape}")
        core8 = np.ascontiguousarray(core, dtype=np.uint8)
        labels = np.empty(n, dtype=np.int64)
        t = Timings()
        st = self.lib.ds_merge_bits_core(self.handle, bits.ctypes.data, core8.ctypes.data, n,
                                         labels.ctypes.data, ctypes.byref(t))
        raise_for(st, self.lib)
        return labels, t

    def serial_dbscan(self, coords: np.ndarray, eps_sq: float, min_pts: int):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        n, d = coords.shape
        labels = np.empty(n, dtype=np.int64)
        counts = np.empty(n, dtype=np.int64)
        t = Timings()
        st = self.lib.ds_serial_dbscan(self.handle, coords.ctypes.data, n, d, float(eps_sq),
                                       int(min_pts), labels.ctypes.data, counts.ctypes.data,
                                       ctypes.byref(t))
        raise_for(st, self.lib)
        return labels, counts, t

    def core_adjacency(self, bits: np.ndarray, valid: np.ndarray):
        """(core_indices int64[m], m x ceil(m/8) packbits rows) of build_core_adjacency."""
        n = valid.shape[0]
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        if bits.shape != (n, (n + 7) // 8):
            raise ValueError(f"bits must have shape {(n, (n + 7) // 8)}, got {bits.shape}")
        valid8 = np.ascontiguousarray(valid, dtype=np.uint8)
        m = int(np.count_nonzero(valid8))
        core_indices = np.empty(m, dtype=np.int64)
        adj = np.empty((m, (m + 7) // 8), dtype=np.uint8)
        t = Timings()
        st = self.lib.ds_core_adjacency(self.handle, bits.ctypes.data, valid8.ctypes.data, n, m,
                                        core_indices.ctypes.data if m else None,
                                        adj.ctypes.data if m else None, ctypes.byref(t))
        raise_for(st, self.lib)
        return core_indices, adj, t

    def warshall_closure(self, adj: np.ndarray, m: int):
        adj = np.ascontiguousarray(adj, dtype=np.uint8)
        if adj.shape != (m, (m + 7) // 8):
            raise ValueError(f"adjacency must have shape {(m, (m + 7) // 8)}, got {adj.shape}")
        out = np.empty_like(adj)
        t = Timings()
        st = self.lib.ds_warshall_closure(self.handle, adj.ctypes.data if m else None, m,
                                          out.ctypes.data if m else None, ctypes.byref(t))
        raise_for(st, self.lib)
        return out, t

    # ---- materialising ladder (kernels.py:153-308) ----
    def dist_matrix(self, coords: np.ndarray, mem_cap: int):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        n, d = coords.shape
        out = np.empty((n, n), dtype=np.float32)
        t = Timings()
        st = self.lib.ds_dist_matrix(self.handle, coords.ctypes.data, n, d, int(mem_cap),
                                     out.ctypes.data, ctypes.byref(t))
        raise_for(st, self.lib)
        return out, t

    def dist_threshold(self, dist: np.ndarray, eps_sq: float, min_pts: int, mem_cap: int):
        dist = np.ascontiguousarray(dist, dtype=np.float32)
        n = dist.shape[0]
        if dist.shape != (n, n):
            raise ValueError(f"distance matrix must be square, got {dist.shape}")
        bits = np.empty((n, (n + 7) // 8), dtype=np.uint8)
        counts = np.empty(n, dtype=np.int64)
        valid = np.empty(n, dtype=np.uint8)
        t = Timings()
        st = self.lib.ds_dist_threshold(self.handle, dist.ctypes.data, n, float(eps_sq),
                                        int(min_pts), int(mem_cap), bits.ctypes.data,
                                        counts.ctypes.data, valid.ctypes.data, ctypes.byref(t))
        raise_for(st, self.lib)
        return bits, counts, valid.astype(bool), t

    def dist_build(self, coords: np.ndarray, eps_sq: float, min_pts: int, mem_cap: int):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        n, d = coords.shape
        bits = np.empty((n, (n + 7) // 8), dtype=np.uint8)
        counts = np.empty(n, dtype=np.int64)
        valid = np.empty(n, dtype=np.uint8)
        t = Timings()
        st = self.lib.ds_dist_build(self.handle, coords.ctypes.data, n, d, float(eps_sq),
                                    int(min_pts), int(mem_cap), bits.ctypes.data,
                                    counts.ctypes.data, valid.ctypes.data, ctypes.byref(t))
        raise_for(st, self.lib)
        return bits, counts, valid.astype(bool), t


def pin_frozen(arr: np.ndarray, owner) -> bool:
    """Page-lock the (read-only) buffer of `arr` for the lifetime of `owner`.

    Used for PointSet coordinates, which are frozen after construction: every
    call still copies them to the device, but at DMA speed. Failure only means
    pageable (slower) copies.
    """
    import weakref
    if getattr(owner, "_ds_pinned", False) or arr.nbytes == 0:
        return getattr(owner, "_ds_pinned", False)
    lib = load_library()
    if lib.ds_host_register(ctypes.c_void_p(arr.ctypes.data), arr.nbytes) != DS_OK:
        return False
    owner._ds_pinned = True
    weakref.finalize(owner, lib.ds_host_unregister, ctypes.c_void_p(arr.ctypes.data))
    return True


_pin_torch = []  # [torch module or None], resolved on first use


def pinned_empty(n: int, dtype=np.int64) -> np.ndarray:
    """Page-locked host array from torch's caching host allocator when available
    (device->host copies into it run at DMA speed); plain numpy otherwise."""
    if not _pin_torch:
        try:
            import torch
            _pin_torch.append(torch if torch.cuda.is_available() else None)
        except Exception:
            _pin_torch.append(None)
    torch = _pin_torch[0]
    dt = np.dtype(dtype)
    if torch is not None and dt in (np.dtype(np.int64), np.dtype(np.int32)):
        try:
            tdt = torch.int64 if dt == np.dtype(np.int64) else torch.int32
            return torch.empty(n, dtype=tdt, pin_memory=True).numpy()
        except Exception:
            pass
    return np.empty(n, dtype=dt)


_ctx_local = threading.local()


def context(device: int | None = None) -> Context:
    """The calling thread's context on `device` (default: $DENSESCAN_DEVICE or 0)."""
    if device is None:
        device = int(os.environ.get("DENSESCAN_DEVICE", "0"))
    cache = getattr(_ctx_local, "ctxs", None)
    if cache is None:
        cache = _ctx_local.ctxs = {}
    ctx = cache.get(device)
    if ctx is None:
        ctx = cache[device] = Context(device)
    return ctx
