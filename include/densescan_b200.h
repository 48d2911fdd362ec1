/*
 * densescan_b200 — C ABI of the sm_100a DBSCAN hot path.
 *
 * This is the drop-in boundary for the reference package's CPU path
 * `run_dbscan(points, validate_params(eps, min_pts), default_config())`
 * (reference pkg/src/densescan/pipeline.py:70-92). The reference has no FFI
 * of its own (it is pure Python); the Python mirror in
 * paper_1506_02226_b200/ binds these symbols with ctypes, and INTEGRATION.md
 * shows the binding a reference maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only. Host buffers are caller-owned; the context
 *    owns device workspaces and streams. Inputs are never written.
 *  - Coordinates are float64, point-major (n x d), exactly the reference
 *    PointSet.coords_aos layout (core.py:43-70). The library narrows them to
 *    float32 round-to-nearest once (kernels.py:148-150).
 *  - eps_sq is the float64 eps*eps of DbscanParams (core.py:93); the kernel
 *    threshold is float32(eps_sq) (kernels.py:355, 385).
 *  - Every entry point returns a ds_status; on failure ds_last_error() gives a
 *    thread-local message and, for DS_ECAPACITY, ds_last_capacity() gives the
 *    (required, cap) byte pair that the Python shim re-raises as
 *    CapacityExceeded(required_bytes, cap_bytes) (kernels.py:55-63).
 *  - Labels are int64, canonical: clusters numbered 0,1,2,... by lowest member
 *    index, noise = -1 (core.py:116-132). Results do not depend on thread
 *    scheduling, atomics order or GPU count.
 *  - A context is not thread-safe; use one context per host thread.
 */
#ifndef DENSESCAN_B200_H
#define DENSESCAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DS_ABI_VERSION 1

typedef struct ds_ctx ds_ctx;

typedef enum {
  DS_OK = 0,
  DS_EINVAL = 1,        /* -> InvalidParams / ValueError (core.py:22-27, 53-58)      */
  DS_ECAPACITY = 2,     /* -> CapacityExceeded(required, cap) (kernels.py:55-79)    */
  DS_ECUDA = 3,         /* -> DeviceError                                            */
  DS_EINCONSISTENT = 4, /* -> InconsistentInput (merge.py:36-37, 141-145)            */
  DS_ENCCL = 5          /* -> DeviceError (multi-GPU exchange)                       */
} ds_status;

typedef enum {
  DS_FORMULA_DIRECT = 0,    /* FUSED and the four materialising rungs (kernels.py:197-210) */
  DS_FORMULA_ALGEBRAIC = 1  /* FUSED_ALGEBRAIC, the default (kernels.py:374-417)          */
} ds_formula;

/* Per-call measurements; mirrors StageTimings (pipeline.py:52-67) plus the
 * counters the benchmark needs. All times are device times except total_ms, which
 * covers the whole call including copies: copies by CUDA events; fused_ms, tile_ms
 * and merge_ms of ds_run_dbscan[_device] by %globaltimer stamps at the kernel
 * boundaries (CUDA events with DS_OPT_EVENT_TIMING), of the other entry points by
 * CUDA events. */
typedef struct {
  double fused_ms;          /* stage 1+2: prep + eps-tile kernel (+ core flags)      */
  double merge_ms;          /* stage 3: union-find, borders, canonical labels        */
  double total_ms;          /* whole call, host wall clock                           */
  double tile_ms;           /* the eps-tile kernel alone                             */
  double h2d_ms;            /* host->device copy of the coordinates                  */
  double d2h_ms;            /* device->host copy of the labels (event timing only,  */
                            /* DS_OPT_EVENT_TIMING; 0 otherwise)                     */
  int64_t pairs_evaluated;  /* ordered pair evaluations executed by the tile kernel  */
  int64_t tiles_total;      /* tile pairs processed (upper triangle incl. diagonal)  */
  int64_t tiles_nonempty;   /* tile pairs with at least one in-range pair            */
  int64_t words_emitted;    /* 32-bit adjacency words kept for stage 3               */
  int64_t core_count;
  int64_t cluster_count;
  int64_t device_bytes;     /* device workspace held by the context after the call   */
  int32_t unsafe_range;     /* 1 if coordinates needed the overflow-safe compare     */
  int32_t tile_launches;    /* eps-tile kernel launches (>1 after a capacity regrow) */
} ds_timings;

/* Library / build identification. */
int ds_abi_version(void);
const char* ds_build_info(void);

/* Last error of the calling thread. */
const char* ds_last_error(void);
void ds_last_capacity(int64_t* required_bytes, int64_t* cap_bytes);

/* Page-lock (and release) a caller-owned host range so the copies of
 * ds_run_dbscan / ds_fused_build run at DMA speed. Frozen inputs (the
 * reference PointSet arrays are read-only after construction, core.py:59-64)
 * are registered once per lifetime. Registering an already registered range
 * succeeds. */
ds_status ds_host_register(const void* ptr, size_t bytes);
ds_status ds_host_unregister(const void* ptr);

/* Context on one CUDA device (ordinal). */
ds_status ds_ctx_create(int device, ds_ctx** out);
void ds_ctx_destroy(ds_ctx* ctx);

/* Context options.
 * DS_OPT_TILE_CULL (default 1): skip tile pairs whose bounding boxes prove every
 * pair out of range, with a float32 rounding-error margin;
 * results are bit-identical with 0 (the paper's dense schedule).
 * DS_OPT_SPATIAL_SORT (default 1): visit points in Morton order of their
 * coordinates so tiles are compact (more tile pairs culled); index-dependent
 * rules still use original indices, results are bit-identical with 0.
 * DS_OPT_CUDA_GRAPH (default 1): record the device pipeline into a CUDA graph
 * on the second call with an identical shape/buffers/options and replay it.
 * DS_OPT_EVENT_TIMING (default 0): time stage 1+2, the eps-tile kernel and stage 3
 * of ds_run_dbscan / ds_run_dbscan_device with CUDA events recorded between the
 * kernels; 0 takes them from %globaltimer stamps the kernels write (events between
 * kernels cost device time: they break the programmatic overlap of the launches).
 * DS_OPT_TEST_CAPACITY (default 0; test hook): > 0 starts the next stage 1+2 from
 * a unit-list and adjacency-word capacity of `value` entries and at most doubles it
 * per re-run, so one call walks through many capacity grow steps. Every launch that
 * overflowed is discarded and re-run; a call never returns results from one.
 * DS_OPT_STABLE_ORDER (default 0): with 0, inputs of 1-2 dimensions up to 2^18 points
 * take the spatial order from a counting sort whose order among points of the same
 * grid cell is arbitrary (the work counters may differ between calls; labels, counts
 * and bits never do); 1 always uses the stable radix sort (the multi-GPU shard stages
 * always do: every rank must build the same order). */
enum { DS_OPT_TILE_CULL = 1, DS_OPT_SPATIAL_SORT = 2, DS_OPT_CUDA_GRAPH = 3, DS_OPT_EVENT_TIMING = 4,
       DS_OPT_TEST_CAPACITY = 5, DS_OPT_STABLE_ORDER = 6 };
ds_status ds_ctx_set_option(ds_ctx* ctx, int32_t option, int64_t value);
int64_t ds_ctx_get_option(ds_ctx* ctx, int32_t option);

/*
 * run_dbscan (pipeline.py:70-92): host float64 coords in, host int64
 * canonical labels out. mem_cap bounds the device workspace in bytes
 * (<= 0: no bound). counts_out (int64[n]) is optional (NULL to skip).
 */
ds_status ds_run_dbscan(ds_ctx* ctx, const double* coords, int64_t n, int32_t d,
                        double eps_sq, int64_t min_pts, int32_t formula, int64_t mem_cap,
                        int64_t* labels_out, int64_t* counts_out, ds_timings* timings);

/*
 * Same pipeline on device-resident buffers: d_coords is a device float64
 * n x d array, d_labels a device int64[n]. `stream` is a cudaStream_t (NULL:
 * the legacy default stream); all work is enqueued on it and the call returns
 * after the stream has completed it.
 */
ds_status ds_run_dbscan_device(ds_ctx* ctx, const double* d_coords, int64_t n, int32_t d,
                               double eps_sq, int64_t min_pts, int32_t formula,
                               int64_t mem_cap, int64_t* d_labels, void* stream,
                               ds_timings* timings);

/*
 * Stage 1+2 in the reference's NeighborhoodMatrix / ValidVector layout
 * (kernels.py:120-145, 311-337, 420-442): bits_out is n x ceil(n/8) bytes,
 * numpy packbits MSB-first rows (_bitmat.py:4-7) or NULL; counts_out int64[n]
 * (incl. self); valid_out uint8[n] (counts >= min_pts).
 */
ds_status ds_fused_build(ds_ctx* ctx, const double* coords, int64_t n, int32_t d,
                         double eps_sq, int64_t min_pts, int32_t formula, int64_t mem_cap,
                         uint8_t* bits_out, int64_t* counts_out, uint8_t* valid_out,
                         ds_timings* timings);

/*
 * Stage 3 from a reference-layout NeighborhoodMatrix (merge_iterative,
 * merge.py:133-166, and merge_warshall, merge.py:218-238, which are
 * label-equivalent): bits n x ceil(n/8) MSB-first, counts int64[n], valid
 * uint8[n]. Checks valid == (counts >= min_pts) first (DS_EINCONSISTENT,
 * merge.py:141-145). Writes canonical int64 labels.
 */
ds_status ds_merge_bits(ds_ctx* ctx, const uint8_t* bits, const int64_t* counts,
                        const uint8_t* valid, int64_t n, int64_t min_pts,
                        int64_t* labels_out, ds_timings* timings);

/*
 * The Warshall backend's merge (merge_warshall, merge.py:218-238): like
 * ds_merge_bits, but the core set is `core` (uint8[n]) exactly as given — the
 * reference reads valid_vec.valid and never checks it against the counts.
 * Label-equivalent to the closure for the symmetric neighbourhood relation
 * stage 1+2 produces (SPEC merge contract).
 */
ds_status ds_merge_bits_core(ds_ctx* ctx, const uint8_t* bits, const uint8_t* core, int64_t n,
                             int64_t* labels_out, ds_timings* timings);

/*
 * build_core_adjacency (merge.py:179-188): the n x ceil(n/8) packbits matrix
 * restricted to the rows and columns of the m valid points. core_indices_out
 * (int64[m], ascending) and adj_out (m x ceil(m/8) packbits rows) are written;
 * m must equal the number of non-zero entries of valid (DS_EINVAL otherwise).
 */
ds_status ds_core_adjacency(ds_ctx* ctx, const uint8_t* bits, const uint8_t* valid, int64_t n,
                            int64_t m, int64_t* core_indices_out, uint8_t* adj_out,
                            ds_timings* timings);

/*
 * warshall_closure (merge.py:191-215): transitive closure of an m x m packbits
 * relation (m x ceil(m/8) bytes) into closed_out (same layout), identical to the
 * reference's pivot recurrence for any input relation (blocked over 32-pivot
 * blocks on the device). The input is not modified.
 */
ds_status ds_warshall_closure(ds_ctx* ctx, const uint8_t* adj, int64_t m, uint8_t* closed_out,
                              ds_timings* timings);

/*
 * serial_dbscan (oracle.py:48-111), the reference's float64 semantic oracle, on the
 * device: d2 = ((x_j - x_i)^2 + (y_j - y_i)^2) + ... in float64 (one IEEE op each, no
 * FMA), in range iff d2 <= eps_sq (float64), counts incl. self, clusters = connected
 * components of core-core pairs, borders to their lowest-indexed in-range core,
 * canonical labels. Used by the CLI's --variant serial and the bench equivalence gate
 * (cli.py:94-122, 152-234). timings: tile_ms = distance + eps stage, fused_ms = core
 * flags, merge_ms = components + borders + labels. Needs n * ceil(n/32) * 4 device bytes.
 */
ds_status ds_serial_dbscan(ds_ctx* ctx, const double* coords, int64_t n, int32_t d, double eps_sq,
                           int64_t min_pts, int64_t* labels_out, int64_t* counts_out,
                           ds_timings* timings);

/* ---- materialising ladder (kernels.py:153-308) ----
 * The BASELINE / SOA / TILED / TILED_UNROLLED rungs all compute the same
 * direct-formula squared distances (kernels.py:21-25, _direct_block 197-210):
 * d2[i][j] = ((x_j - x_i)^2 + (y_j - y_i)^2) + ..., float32, no FMA. */

/* dist_baseline / dist_soa / dist_tiled: the n x n float32 matrix, row-major
 * into out (host). Capacity: 4 n^2 bytes against mem_cap (kernels.py:156). */
ds_status ds_dist_matrix(ds_ctx* ctx, const double* coords, int64_t n, int32_t d,
                         int64_t mem_cap, float* out, ds_timings* timings);

/* build_clusters_from_dist (kernels.py:284-308): threshold a host n x n float32
 * matrix at float32(eps_sq) into the reference layout (bits n x ceil(n/8)
 * MSB-first, int64 counts incl. self, uint8 valid = counts >= min_pts).
 * Capacity: n * ceil(n/8) bytes against mem_cap (kernels.py:293). */
ds_status ds_dist_threshold(ds_ctx* ctx, const float* dist, int64_t n, double eps_sq,
                            int64_t min_pts, int64_t mem_cap, uint8_t* bits_out,
                            int64_t* counts_out, uint8_t* valid_out, ds_timings* timings);

/* run_variant's materialising rungs (kernels.py:445-470): both steps on the
 * device, the matrix materialised in HBM (row blocks of at most 4 GiB) and never
 * copied to the host. timings->tile_ms = distance kernels (dist_ms),
 * timings->merge_ms = threshold kernels (cluster_ms). */
ds_status ds_dist_build(ds_ctx* ctx, const double* coords, int64_t n, int32_t d, double eps_sq,
                        int64_t min_pts, int64_t mem_cap, uint8_t* bits_out,
                        int64_t* counts_out, uint8_t* valid_out, ds_timings* timings);

/* ---- multi-GPU shards (row-block sharding of stage 1 over tile-pair items) ----
 * The upper-triangle tile pairs (TILE = ds_tile_side() points per side) are
 * numbered 0 .. ds_tile_items(n)-1 row-major. Each rank evaluates a share of
 * them (culled: the kept tile pairs dealt cyclically; dense: a contiguous range
 * of work units); exchanges (done by the caller over NCCL, see
 * paper_1506_02226_b200/distributed.py) are: all-reduce(SUM) of the int32
 * counts, all-gather of the int32 parent forests, all-reduce(MIN) of the
 * int32 border minima. Replaces the reference's fork-join over row ranges
 * (_parallel.py:24-39) at GPU granularity. */
int64_t ds_tile_items(int64_t n);
int ds_tile_side(void);

/* Stage 1+2 on rank's share of the tile-pair items (of the culled list when
 * DS_OPT_TILE_CULL is on, of the dense triangle otherwise): partial
 * neighbour counts into d_counts (int32[n], overwritten); the adjacency words
 * stay in the context for ds_shard_stage3_local. */
ds_status ds_shard_stage12(ds_ctx* ctx, const double* d_coords, int64_t n, int32_t d,
                           double eps_sq, int32_t formula, int32_t rank, int32_t world,
                           int64_t mem_cap, int32_t* d_counts, void* stream,
                           ds_timings* timings);

/* Stage 3 on this shard's words with the all-reduced counts (original order):
 * the shard's union-find forest and border minima (int32[n] each, in the
 * context's internal point order, identical on every rank; INT32_MAX = none). */
ds_status ds_shard_stage3_local(ds_ctx* ctx, const int32_t* d_counts, int64_t n, int64_t min_pts,
                                int32_t* d_parent, int32_t* d_bmin, void* stream,
                                ds_timings* timings);

/* One round of the pairwise forest exchange: d_parent (int32[n], a shard forest
 * in the context's internal order) becomes the union of itself and d_other, and is
 * flattened (every entry points at its root). Folding the R shard forests pairwise
 * (recursive doubling, log2 R rounds; paper_1506_02226_b200/distributed.py) gives
 * every rank the forest of all edges with O(n log R) work per rank. */
ds_status ds_shard_fold(ds_ctx* ctx, int32_t* d_parent, const int32_t* d_other, int64_t n,
                        void* stream);

/* Fold nparents forests (nparents x n; 1 after the pairwise exchange) and the
 * min-reduced border minima into canonical int64 labels. */
ds_status ds_shard_stage3_merge(ds_ctx* ctx, const int32_t* d_counts, int64_t n, int64_t min_pts,
                                const int32_t* d_parents, int32_t nparents, const int32_t* d_bmin,
                                int64_t* d_labels, void* stream, ds_timings* timings);

#ifdef __cplusplus
}
#endif

#endif /* DENSESCAN_B200_H */
