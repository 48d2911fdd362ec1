// C ABI of densescan_b200 (include/densescan_b200.h): context, device workspace,
// and the three-stage pipeline composition that replaces the reference's
// run_dbscan (pkg/src/densescan/pipeline.py:70-92), fused_build[_algebraic]
// (kernels.py:420-442) and merge_iterative (merge.py:133-166).
#include <cuda_runtime.h>

#include <atomic>
#include <stdint.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ds_internal.cuh"

namespace ds {

static thread_local std::string g_error;
static thread_local int64_t g_required = 0, g_cap = 0;

void set_error(const std::string& msg) { g_error = msg; }
void set_capacity(int64_t required, int64_t cap) {
  g_required = required;
  g_cap = cap;
}

}  // namespace ds

using namespace ds;

#define DS_CK(expr)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      set_error(std::string(#expr) + " failed: " + cudaGetErrorString(e_));           \
      return DS_ECUDA;                                                                \
    }                                                                                 \
  } while (0)

namespace {

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Scalars {  // a whole number of 8-byte words (the label kernel copies it by words)
  unsigned long long work_ctr;
  unsigned long long words_count;
  unsigned long long nonempty_count;
  unsigned long long kept;  // tile pairs surviving the culling test
  unsigned long long ncore;
  unsigned long long pairs_done;
  unsigned long long unit_count;  // units in the culled unit list
  int32_t kept32;
  uint32_t unsafe_flag;
  int32_t nclusters;
  unsigned int label_blocks;                // label_kernel blocks finished
  unsigned long long stamps[ST_COUNT];      // device stage boundaries (Stamp)
};
static_assert(sizeof(Scalars) % 8 == 0 && sizeof(Scalars) / 8 <= 1024, "Scalars is copied in 8-byte words, one per label-kernel thread");

// The per-call zero region: one memset clears the scalars, the spatial-sort bounding
// box, the diagonal directory index and the label scan's look-back state.
constexpr size_t ZR_ALIGN = 256;
inline size_t zr_round(size_t b) { return (b + ZR_ALIGN - 1) / ZR_ALIGN * ZR_ALIGN; }
inline size_t zr_bbox() { return zr_round(sizeof(Scalars)); }
inline size_t zr_diag() { return zr_bbox() + ZR_ALIGN; }
inline size_t zr_scan(int64_t n) { return zr_diag() + zr_round((size_t)n_tiles(n) * 8); }
// the tile-root link table of union_links (one CAS slot per linked pair of tile roots)
inline int link_tab_bits(int64_t n) {
  int b = 8;
  while (b < 14 && ((int64_t)1 << b) < 4 * n_tiles(n)) ++b;
  return b;
}
inline size_t zr_links(int64_t n) { return zr_round(zr_scan(n) + (size_t)scan_partials_len(n) * 4); }
// the super-tile boxes of the hierarchical culling (d <= 4)
inline size_t zr_super(int64_t n) { return zr_round(zr_links(n) + ((size_t)8 << link_tab_bits(n))); }
// the counting sort's 65536 cell counters (inputs up to 2^18 points)
inline size_t zr_bins(int64_t n) {
  return zr_round(zr_super(n) + (size_t)n_supers(n_tiles(n)) * SUPER_BS * 4);
}
inline size_t zr_bytes(int64_t n) {
  return zr_bins(n) + (n <= ((int64_t)1 << 18) ? (size_t)SORT_BINS * 4 + scan_zeroed_bytes(SORT_BINS)
                                                : 0);
}

}  // namespace

struct ds_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[8] = {};
  Buf troot;  // per-block uniform roots of the diagonal union pass (single GPU)
  Buf coords64, rec, cnt, core, corew, parent, bmin, cmin, root, flag, partials, labels, counts64,
      words, chunks, scalars, dense, tbox, items, iflags, ipartials, rec_sorted, perm, inv, keys,
      keys_alt, kidx, sort_temp, blk, ulist, uchunks, ucnt, dist, dbits, adjm, ci32, ci64, cws, soa64;
  int cull = 1;          // DS_OPT_TILE_CULL
  int use_graph = 1;     // DS_OPT_CUDA_GRAPH
  // CUDA graph of the device pipeline, replayed while the key matches
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t graph = nullptr;  // kept alive: its memcpy nodes are re-pointed per launch
  cudaGraphNode_t gn_h2d = nullptr, gn_labels = nullptr, gn_counts = nullptr;
  unsigned long long gkey[12] = {};
  unsigned long long seen_key[12] = {};
  bool capturing = false;  // events become external graph nodes while recording
  bool stamp_timing = false;  // stage timings from device stamps: no events inside
  int sort = 1;          // DS_OPT_SPATIAL_SORT
  int event_timing = 0;  // DS_OPT_EVENT_TIMING
  int stable = 0;        // DS_OPT_STABLE_ORDER
  bool sorted = false;   // perm / inv describe the last stage 1+2
  unsigned long long words_cap = 0;  // in words (8-byte records)
  unsigned long long units_cap = 0;  // culled unit list capacity (units)
  UnitArgs units{};                  // the last eps-tile launch (read by stage 3)
  int unit_lb = 4;                   // its lane blocks per tile
  Scalars* h_scalars = nullptr;      // pinned
  unsigned long long* h_scalars_dev = nullptr;  // its device (mapped) alias
  // DS_OPT_TEST_CAPACITY (test hook): > 0 forces this initial unit-list and word
  // capacity on the next stage 1+2 and limits every regrow to x2, so one call walks
  // through many grow steps; 0 (default) = normal sizing
  int64_t test_cap = 0;
  bool test_cap_pending = false;
  bool no_graph_key = false;         // the recorded graph lacked a host-copy node
};

namespace {

// bumped whenever a buffer moves (any context, any thread): recorded graphs compare it
static std::atomic<unsigned long long> g_alloc_generation{0};

cudaError_t ensure(Buf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return cudaSuccess;
  ++g_alloc_generation;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return e;
  }
  b.bytes = bytes;
  return cudaSuccess;
}

size_t held_bytes(const ds_ctx* c) {
  const Buf* all[] = {&c->coords64, &c->rec, &c->cnt,   &c->core,     &c->corew,   &c->parent,
                      &c->bmin,     &c->cmin, &c->root, &c->flag,     &c->partials, &c->labels,
                      &c->counts64, &c->words, &c->chunks, &c->scalars, &c->dense,
                      &c->tbox,     &c->items,  &c->iflags, &c->ipartials,
                      &c->rec_sorted, &c->perm, &c->inv, &c->keys, &c->keys_alt, &c->kidx,
                      &c->sort_temp, &c->blk, &c->ulist, &c->uchunks, &c->ucnt,
                      &c->dist, &c->dbits, &c->troot, &c->adjm, &c->ci32, &c->ci64, &c->cws, &c->soa64};
  size_t s = 0;
  for (const Buf* b : all) s += b->bytes;
  return s;
}

double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

ds_status check_args(int64_t n, int32_t d, int64_t min_pts, int32_t formula) {
  if (n < 1) {
    set_error("n: a PointSet needs at least one point");
    return DS_EINVAL;
  }
  if (n >= (int64_t)0x7fffffff - 1024) {
    set_error("n: more than 2^31 points is not supported");
    return DS_EINVAL;
  }
  if (d < 1 || d > MAX_D) {
    set_error("d: dimension must be in [1, 64]");
    return DS_EINVAL;
  }
  if (min_pts < 1) {
    set_error("min_pts: threshold must be an integer >= 1");
    return DS_EINVAL;
  }
  if (formula != DS_FORMULA_DIRECT && formula != DS_FORMULA_ALGEBRAIC) {
    set_error("formula: must be 0 (direct) or 1 (algebraic)");
    return DS_EINVAL;
  }
  return DS_OK;
}

constexpr size_t WORD_BYTES = 8;  // one adjacency record

// Bytes of every device buffer the pipeline needs except the adjacency words.
size_t base_bytes(int64_t n, int d) {
  const size_t N = (size_t)n;
  return N * rec_stride(d) * 4      // rec
         + (size_t)n_items(n_tiles(n)) * (16 + 4 + 4 + 4)  // dir + item list + flags + units
         + (size_t)n_tiles(n) * (2 * padded_dim(d) + 1) * 4  // tile boxes
         + N * rec_stride(d) * 4 + N * (4 + 4 + 8 + 8 + 4)  // spatial order
         + ((N + 31) / 32) * (2 * padded_dim(d) + 1) * 4      // 32-point block boxes
         + N * 4 * 6                // cnt parent bmin cmin root flag
         + N                        // core
         + ((N + 31) / 32) * 4      // corew
         + (size_t)scan_partials_len(n) * 4 + sizeof(Scalars) + N * 8;  // labels
}

// the diagonal tile pairs' unit ranges (zero region; written by the unit list)
uint2* diag_range(ds_ctx* c) { return (uint2*)((char*)c->scalars.p + zr_diag()); }

MergeWs merge_ws(ds_ctx* c, int64_t n) {
  MergeWs w;
  Scalars* sc = (Scalars*)c->scalars.p;
  w.n = n;
  w.cnt = (const int32_t*)c->cnt.p;
  w.core = (uint8_t*)c->core.p;
  w.corew = (uint32_t*)c->corew.p;
  w.parent = (int32_t*)c->parent.p;
  w.bmin = (int32_t*)c->bmin.p;
  w.cmin = (int32_t*)c->cmin.p;
  w.root = (int32_t*)c->root.p;
  w.flag = (int32_t*)c->flag.p;
  w.partials = (int32_t*)c->partials.p;
  w.scan_state = (int32_t*)((char*)c->scalars.p + zr_scan(n));  // zeroed per call
  w.nclusters = &sc->nclusters;
  w.ncore = &sc->ncore;
  if (c->sorted) {
    w.perm = (const int32_t*)c->perm.p;
    w.inv = (const int32_t*)c->inv.p;
  }
  return w;
}

// core_init's job for the diagonal union pass (single GPU)
CoreInit core_init_args(const MergeWs& w, int64_t min_pts) {
  CoreInit ci;
  ci.cnt = w.cnt;
  ci.n = w.n;
  ci.min_pts = min_pts;
  ci.core = w.core;
  ci.corew = w.corew;
  ci.parent = w.parent;
  ci.bmin = w.bmin;
  ci.cmin = w.cmin;
  ci.ncore = w.ncore;
  return ci;
}

ds_status alloc_common(ds_ctx* c, int64_t n, int d) {
  const size_t N = (size_t)n;
  DS_CK(ensure(c->rec, N * rec_stride(d) * 4));
  DS_CK(ensure(c->cnt, N * 4));
  DS_CK(ensure(c->core, N));
  DS_CK(ensure(c->corew, ((N + 31) / 32) * 4));
  DS_CK(ensure(c->parent, N * 4));
  DS_CK(ensure(c->troot, (size_t)((n + 31) / 32) * 4));
  DS_CK(ensure(c->bmin, N * 4));
  DS_CK(ensure(c->cmin, N * 4));
  DS_CK(ensure(c->root, N * 4));
  DS_CK(ensure(c->flag, N * 4));
  DS_CK(ensure(c->partials, (size_t)scan_partials_len(n) * 4));
  DS_CK(ensure(c->scalars, zr_bytes(n)));
  DS_CK(ensure(c->chunks, (size_t)n_items(n_tiles(n)) * 16));  // tile-pair directory
  return DS_OK;
}

cudaError_t record(ds_ctx* c, cudaEvent_t e, cudaStream_t s) {
  return c->capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                      : cudaEventRecord(e, s);
}

// device bytes per row unit: chunk entries (WPR x 8 B) + the culled list entry (8 B)
inline size_t unit_bytes(bool cull) { return (size_t)WPR * 8 + (cull ? 8 : 0); }

struct Plan {
  int64_t T = 0, all_items = 0, item_lo = 0, item_hi = 0, dense_units = 0;
  unsigned long long units_cap = 0;
  bool cull = false;
  size_t base = 0;
  int rank = 0, world = 1;
};

// Stage 1+2 enqueue (prep, spatial order, culling, eps-tile kernel). Nothing here
// waits for the device: the adjacency-word buffer is sized from what earlier calls
// needed, and an overflow (detected by check_words after the caller's single sync)
// triggers one re-run with the exact size.
// want_dir: also build the directory of tile pairs with words (the reference-layout
// export reads it; stage 3 walks the units directly).
ds_status stage12_enqueue(ds_ctx* c, const double* d_coords, int64_t n, int d, double eps_sq,
                          int formula, int64_t mem_cap, cudaStream_t s, Plan& pl, int rank = 0,
                          int world = 1, bool want_dir = false) {
  ds_status st = alloc_common(c, n, d);
  if (st != DS_OK) return st;
  if (world < 1 || rank < 0 || rank >= world) {
    set_error("shard: rank must be in [0, world)");
    return DS_EINVAL;
  }
  pl.T = n_tiles(n);
  if (pl.T > 65536) {  // tile pairs are packed as a << 16 | b
    set_error("n: more than 2^25 points per call is not supported");
    return DS_EINVAL;
  }
  pl.all_items = n_items(pl.T);
  pl.cull = c->cull != 0 && pl.T > 1;
  pl.rank = rank;
  pl.world = world;
  // dense schedule: contiguous equal slice of the triangle; culled schedule: the
  // slice of the device-side kept list is taken inside the kernel
  pl.item_lo = pl.all_items * rank / world;
  pl.item_hi = pl.all_items * (rank + 1) / world;
  const int64_t T = pl.T;
  pl.dense_units = pl.all_items * lane_blocks(d);
  if (c->test_cap_pending) {  // test hook: start from a tiny capacity (see ds_ctx)
    c->units_cap = (unsigned long long)c->test_cap;
    c->words_cap = (unsigned long long)c->test_cap;
    c->test_cap_pending = false;
  }
  if (pl.cull) {  // row-unit list + chunk table sized from earlier calls (lazy, like the words)
    const unsigned long long guess = c->test_cap > 0 ? 1 : (unsigned long long)n / 8 + 4096;
    pl.units_cap = std::max<unsigned long long>(c->units_cap, guess);
  } else {
    pl.units_cap = (unsigned long long)pl.dense_units;
  }
  pl.base = base_bytes(n, d) + (size_t)pl.units_cap * unit_bytes(pl.cull);

  const unsigned long long run_slack = (unsigned long long)c->sm_count * 16 * WORD_RUN;
  unsigned long long want = std::max<unsigned long long>(
      c->words_cap, c->test_cap > 0 ? 1 : (unsigned long long)n * 8 + (1ull << 20) + run_slack);
  if (mem_cap > 0) {
    const int64_t room = mem_cap - (int64_t)pl.base;
    if (room < 16 * 1024) {
      set_capacity((int64_t)pl.base + 16 * 1024, mem_cap);
      set_error("device workspace exceeds the memory cap");
      return DS_ECAPACITY;
    }
    want = std::min<unsigned long long>(want, (unsigned long long)(room / WORD_BYTES));
  }
  if (c->words.bytes < want * WORD_BYTES) DS_CK(ensure(c->words, want * WORD_BYTES));
  c->words_cap = c->test_cap > 0 ? want : c->words.bytes / WORD_BYTES;
  if (mem_cap > 0) {  // a buffer kept from an earlier, larger call must not bypass the cap
    const unsigned long long room_words =
        (unsigned long long)((mem_cap - (int64_t)pl.base) / WORD_BYTES);
    c->words_cap = std::min(c->words_cap, room_words);
  }

  Scalars* sc = (Scalars*)c->scalars.p;
  const float eps32 = (float)eps_sq;  // float32(float64 eps^2), RN (kernels.py:355/385)

  DS_CK(cudaMemsetAsync(c->scalars.p, 0, zr_bytes(n), s));  // the zero region (cnt: prep)
  const bool do_sort = c->sort && T > 1;
  unsigned int* bbox = (unsigned int*)((char*)c->scalars.p + zr_bbox());
  DS_CK(launch_prep(d_coords, n, d, (float*)c->rec.p, &sc->unsafe_flag, sc->stamps,
                    do_sort ? bbox : nullptr, (int32_t*)c->cnt.p, s));
  const float* rec = (const float*)c->rec.p;
  c->sorted = false;
  const int dp = padded_dim(d);
  SortBounds bnd;  // with culling on, the sort's permute pass also reduces the boxes
  if (pl.cull) {
    DS_CK(ensure(c->tbox, (size_t)T * (2 * dp + 1) * 4));
    DS_CK(ensure(c->blk, (size_t)((n + 31) / 32) * (2 * dp + 1) * 4));
    if (do_sort) {
      bnd.lo = (float*)c->tbox.p;
      bnd.hi = bnd.lo + (size_t)T * dp;
      bnd.maxnorm = bnd.lo + (size_t)T * 2 * dp;
      bnd.blk = dp <= 4 ? (float*)c->blk.p : nullptr;  // block boxes only pay off at d <= 4
      bnd.super = (unsigned int*)((char*)c->scalars.p + zr_super(n));
    }
  }
  if (do_sort) {  // Morton order: compact tiles (ds_sort.cu)
    const size_t N = (size_t)n;
    DS_CK(ensure(c->rec_sorted, N * rec_stride(d) * 4));
    DS_CK(ensure(c->perm, N * 4));
    DS_CK(ensure(c->inv, N * 4));
    DS_CK(ensure(c->keys, N * 8));
    DS_CK(ensure(c->keys_alt, N * 8));
    DS_CK(ensure(c->kidx, N * 4));
    DS_CK(ensure(c->sort_temp, sort_temp_bytes(n)));
    DS_CK(launch_spatial_sort(rec, n, d, (float*)c->rec_sorted.p, (int32_t*)c->perm.p,
                              (int32_t*)c->inv.p, (unsigned long long*)c->keys.p,
                              (unsigned long long*)c->keys_alt.p, (int32_t*)c->kidx.p,
                              c->sort_temp.p, c->sort_temp.bytes, bbox, bnd,
                              // one GPU: the counting sort where it applies (16-bit keys)
                              (world == 1 && !c->stable && n <= ((int64_t)1 << 18))
                                  ? (unsigned int*)((char*)c->scalars.p + zr_bins(n))
                                  : nullptr,
                              s));
    rec = (const float*)c->rec_sorted.p;
    c->sorted = true;
  }
  if (pl.cull) {
    DS_CK(ensure(c->items, (size_t)pl.all_items * 4));
    DS_CK(ensure(c->iflags, (size_t)pl.all_items * 4));
    DS_CK(ensure(c->ipartials, (size_t)scan_partials_len(pl.all_items) * 4));
    float* lo = (float*)c->tbox.p;
    DS_CK(launch_cull(rec, n, d, eps32, formula, &sc->unsafe_flag, lo, lo + (size_t)T * dp,
                      lo + (size_t)T * 2 * dp, (unsigned int*)((char*)c->scalars.p + zr_super(n)),
                      (int32_t*)c->iflags.p, (int32_t*)c->ipartials.p, &sc->kept32,
                      (uint32_t*)c->items.p, &sc->kept, bnd.lo != nullptr,
                      /*ordered: every rank reads the same list*/ world > 1, s));
  }
  UnitArgs a;
  a.rec = rec;
  a.n = n;
  a.T = (int32_t)T;
  a.eps32 = eps32;
  a.cnt = (int32_t*)c->cnt.p;
  a.words = (uint2*)c->words.p;
  a.words_cap = c->words_cap;
  a.words_count = &sc->words_count;
  a.item_list = pl.cull ? (const uint32_t*)c->items.p : nullptr;
  a.unit_count = &sc->unit_count;
  a.units_cap = pl.units_cap;
  a.dense_units = pl.dense_units;
  a.shard_rank = rank;
  a.shard_world = world;
  a.unsafe_flag = &sc->unsafe_flag;
  a.pairs_done = &sc->pairs_done;
  a.work_ctr = &sc->work_ctr;
  a.stamps = sc->stamps;
  a.unit_list = nullptr;
  if (pl.cull) {
    if (!bnd.lo && dp <= 4) DS_CK(launch_block_bounds(rec, n, d, (float*)c->blk.p, s));
    DS_CK(ensure(c->ucnt, (size_t)pl.all_items * 8));  // item_units
    DS_CK(ensure(c->ulist, (size_t)pl.units_cap * 8));
    c->units_cap = pl.units_cap;
    DS_CK(launch_unit_list((const float*)c->blk.p, n, d, eps32, formula, &sc->unsafe_flag,
                           (const uint32_t*)c->items.p, &sc->kept, pl.all_items, rank, world,
                           (uint2*)c->ulist.p, pl.units_cap, &sc->unit_count, (uint2*)c->ucnt.p,
                           diag_range(c), s));
    a.unit_list = (const uint2*)c->ulist.p;
  }
  DS_CK(ensure(c->uchunks, (size_t)pl.units_cap * WPR * 8));
  a.uchunks = (uint2*)c->uchunks.p;
  c->units = a;
  c->unit_lb = lane_blocks(d);
  // an event record between two kernels breaks their programmatic overlap (a few us
  // of device time each): with stamp timing the tile kernel is timed by its stamps
  if (!c->stamp_timing) DS_CK(record(c, c->ev[1], s));
  DS_CK(launch_units_kernel(a, d, formula, c->sm_count, s));
  if (!c->stamp_timing) DS_CK(record(c, c->ev[2], s));
  if (want_dir)
    DS_CK(launch_unit_dir(a, d, pl.all_items, pl.cull ? (const uint2*)c->ucnt.p : nullptr,
                          &sc->kept, (uint4*)c->chunks.p, &sc->nonempty_count, s));
  return DS_OK;
}

// After the caller's sync (h_scalars copied): did the unit list or the adjacency
// words overflow? If so grow what overflowed and ask for a re-run (*retry). A
// launch that overflowed dropped work, so its results must never be returned: the
// callers loop while *retry is set (every re-run has strictly larger capacities)
// and fail with DS_ECAPACITY once the cap, or the attempt budget, is exhausted.
constexpr int MAX_ATTEMPTS = 40;

ds_status check_words(ds_ctx* c, const Plan& pl, int64_t mem_cap, bool* retry) {
  *retry = false;
  const bool limited = c->test_cap > 0;  // test hook: at most x2 per grow step
  const unsigned long long nu = c->h_scalars->unit_count;
  const unsigned long long need = c->h_scalars->words_count;  // reserved slots (runs)
  unsigned long long units_next = c->units_cap, words_next = c->words_cap;
  if (pl.cull && nu > pl.units_cap) {  // the unit list overflowed: grow it
    units_next = nu + nu / 16 + 1024;
    if (limited) units_next = std::min<unsigned long long>(units_next, 2 * pl.units_cap + 1);
    // the launch evaluated only the first units_cap units: its word count scales
    // with the share of units it saw, so grow the words in the same step
    const double share = (double)nu / (double)std::max<unsigned long long>(pl.units_cap, 1);
    const unsigned long long est = (unsigned long long)((double)need * share);
    if (est > c->words_cap) words_next = est + est / 4;
  } else if (need > c->words_cap) {
    // reservations of a re-run differ only by warp scheduling (need >= words); +25%
    // and a run per resident warp covers that in practice
    words_next = need + need / 4;
  } else {
    return DS_OK;
  }
  if (words_next > c->words_cap) {
    words_next += (unsigned long long)c->sm_count * 16 * WORD_RUN + 1024;
    if (limited) words_next = std::min<unsigned long long>(words_next, 2 * c->words_cap + 1);
  }
  const int64_t required = (int64_t)(pl.base + (units_next - pl.units_cap) * unit_bytes(pl.cull) +
                                     words_next * WORD_BYTES);
  if (mem_cap > 0 && required > mem_cap) {
    set_capacity(required, mem_cap);
    set_error(units_next > c->units_cap ? "work-unit list exceeds the memory cap"
                                        : "adjacency words exceed the memory cap");
    return DS_ECAPACITY;
  }
  if (words_next > c->words_cap && c->words.bytes < words_next * WORD_BYTES) {
    if (c->words.p) cudaFree(c->words.p);
    ++g_alloc_generation;
    c->words.p = nullptr;
    c->words.bytes = 0;
    DS_CK(ensure(c->words, words_next * WORD_BYTES));
  }
  c->units_cap = units_next;
  c->words_cap = words_next;
  *retry = true;
  return DS_OK;
}

// A re-run was requested by check_words: fail instead of looping forever.
ds_status retry_budget(int attempt) {
  if (attempt < MAX_ATTEMPTS) return DS_OK;
  set_error("adjacency capacity did not converge after " + std::to_string(attempt) +
            " stage 1+2 launches");
  set_capacity(0, 0);
  return DS_ECAPACITY;
}

void stage12_timings(const ds_ctx* c, const Plan& pl, int launches, ds_timings* t) {
  if (!t) return;
  t->tile_launches = launches;
  int64_t evaluated = pl.item_hi - pl.item_lo;
  if (pl.cull) {
    const int64_t kept = (int64_t)c->h_scalars->kept;  // dealt cyclically to the shards
    evaluated = kept > pl.rank ? (kept - pl.rank + pl.world - 1) / pl.world : 0;
  }
  t->tiles_total = evaluated;
  t->tiles_nonempty = (int64_t)c->h_scalars->nonempty_count;
  t->words_emitted = (int64_t)c->h_scalars->words_count;
  t->unsafe_range = c->h_scalars->unsafe_flag ? 1 : 0;
  // pairs the tile kernel actually evaluated (skipped 32-column groups excluded)
  t->pairs_evaluated = (int64_t)c->h_scalars->pairs_done;
}

// Device part of the pipeline: stage 1+2, core flags, merge, labels (+ counts).
// Host buffers of ds_run_dbscan: the coordinates copied in and the labels / counts
// copied out are part of the enqueued (and graph-recorded) work.
struct HostIO {
  const double* coords = nullptr;
  size_t in_bytes = 0;
  int64_t* labels = nullptr;
  int64_t* counts = nullptr;
  bool time_h2d = false;  // ev5 -> ev0 brackets the caller's coordinate copy
  float h2d_ms = 0.f;     // measured while the rest of the pipeline runs
};

bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

ds_status enqueue_device(ds_ctx* c, const double* d_coords, int64_t n, int d, double eps_sq,
                         int64_t min_pts, int formula, int64_t mem_cap, int64_t* d_labels,
                         int64_t* d_counts64, cudaStream_t s, Plan& pl, bool captured,
                         const HostIO* io) {
  c->capturing = captured;
  c->stamp_timing = !c->event_timing;
  struct Reset {
    ds_ctx* c;
    ~Reset() { c->stamp_timing = false; }
  } reset{c};
  auto rec = [&](cudaEvent_t e) { return record(c, e, s); };
  if (io && io->coords) {
    DS_CK(rec(c->ev[5]));
    DS_CK(cudaMemcpyAsync((void*)d_coords, io->coords, io->in_bytes, cudaMemcpyHostToDevice, s));
  }
  DS_CK(rec(c->ev[0]));
  ds_status st = stage12_enqueue(c, d_coords, n, d, eps_sq, formula, mem_cap, s, pl);
  if (st != DS_OK) return st;
  MergeWs w = merge_ws(c, n);
  w.scan_zeroed = true;
  w.stamps = ((Scalars*)c->scalars.p)->stamps;
  w.label_blocks = &((Scalars*)c->scalars.p)->label_blocks;
  w.blk_root = (int32_t*)c->troot.p;
  w.link_tab = (unsigned long long*)((char*)c->scalars.p + zr_links(n));
  w.link_mask = (1u << link_tab_bits(n)) - 1u;
  // the scalars (final once the label kernel is done) are copied into page-locked
  // memory by the label kernel's last block: no device-to-host copy node after it
  w.dev_scalars = (const unsigned long long*)c->scalars.p;
  w.host_scalars = c->h_scalars_dev;
  w.scalar_words = (int)(sizeof(Scalars) / 8);
  if (c->event_timing) DS_CK(rec(c->ev[3]));
  DS_CK(launch_union_chunks(w, c->units, c->unit_lb, diag_range(c), core_init_args(w, min_pts), s));
  DS_CK(launch_finalize(w, d_labels, s));
  if (d_counts64) DS_CK(launch_counts_i64((const int32_t*)c->cnt.p, n, w.perm, d_counts64, s));
  if (c->event_timing) DS_CK(rec(c->ev[4]));
  if (!c->h_scalars_dev)
    DS_CK(cudaMemcpyAsync(c->h_scalars, c->scalars.p, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  // no event nodes around the copies out: an event-record node between the label
  // kernel and the copy cost ~10 us of device time per call (C2; ev7 is recorded on the
  // stream after the launch instead)
  if (io && io->labels)
    DS_CK(cudaMemcpyAsync(io->labels, d_labels, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
  if (io && io->counts && d_counts64)
    DS_CK(cudaMemcpyAsync(io->counts, d_counts64, (size_t)n * 8, cudaMemcpyDeviceToHost, s));

  c->capturing = false;
  return DS_OK;
}

// memcpy node of `g` whose host end is `host` (source or destination), or nullptr
cudaGraphNode_t find_copy_node(cudaGraph_t g, const void* host) {
  if (!host) return nullptr;
  size_t count = 0;
  if (cudaGraphGetNodes(g, nullptr, &count) != cudaSuccess || count == 0) return nullptr;
  std::vector<cudaGraphNode_t> nodes(count);
  if (cudaGraphGetNodes(g, nodes.data(), &count) != cudaSuccess) return nullptr;
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess || ty != cudaGraphNodeTypeMemcpy) continue;
    cudaMemcpy3DParms pr{};
    if (cudaGraphMemcpyNodeGetParams(nd, &pr) != cudaSuccess) continue;
    if (pr.srcPtr.ptr == host || pr.dstPtr.ptr == host) return nd;
  }
  return nullptr;
}

// The whole pipeline, enqueued without host round trips; the optional host
// copies of labels / counts are enqueued before the single final sync. The
// device part is recorded into a CUDA graph on the second call with the same
// shape, buffers and options, and replayed from then on (no per-kernel launch
// cost); an adjacency-word overflow invalidates the graph.
ds_status pipeline(ds_ctx* c, const double* d_coords, int64_t n, int d, double eps_sq,
                   int64_t min_pts, int formula, int64_t mem_cap, int64_t* d_labels,
                   int64_t* d_counts64, cudaStream_t s, ds_timings* t, HostIO* io = nullptr) {
  Plan pl;
  // host copies are recorded into the graph (and re-pointed per launch) when every
  // host buffer is page-locked; pageable buffers run the pipeline eagerly
  const bool io_graphable =
      !io || ((!io->coords || host_pinned(io->coords)) && (!io->labels || host_pinned(io->labels)) &&
              (!io->counts || host_pinned(io->counts)));
  for (int attempt = 1;; ++attempt) {
    unsigned long long key[12];
    uint64_t eps_bits;
    std::memcpy(&eps_bits, &eps_sq, 8);
    key[0] = (unsigned long long)n;
    key[1] = (unsigned long long)d | ((unsigned long long)formula << 8) |
             ((unsigned long long)c->cull << 16) | ((unsigned long long)c->sort << 17) |
             ((unsigned long long)c->event_timing << 18) | ((unsigned long long)c->stable << 19) |
             1ull << 40;
    key[2] = eps_bits;
    key[3] = (unsigned long long)min_pts;
    key[4] = (unsigned long long)(uintptr_t)d_coords;
    key[5] = (unsigned long long)(uintptr_t)d_labels;
    key[6] = (unsigned long long)(uintptr_t)d_counts64;
    key[7] = c->words_cap;
    key[8] = g_alloc_generation.load();
    key[9] = (unsigned long long)mem_cap;
    key[10] = (unsigned long long)c->device;
    key[11] = c->units_cap;
    key[1] |= (unsigned long long)(io && io->coords) << 41 | (unsigned long long)(io && io->labels) << 42 |
              (unsigned long long)(io && io->counts) << 43;
    const bool use_graph = c->use_graph && io_graphable && !c->no_graph_key;

    const bool graph_hit = use_graph && c->gexec && std::memcmp(key, c->gkey, sizeof key) == 0;
    if (graph_hit) {
      if (io && io->coords && c->gn_h2d)
        DS_CK(cudaGraphExecMemcpyNodeSetParams1D(c->gexec, c->gn_h2d, (void*)d_coords, io->coords,
                                                 io->in_bytes, cudaMemcpyHostToDevice));
      if (io && io->labels && c->gn_labels)
        DS_CK(cudaGraphExecMemcpyNodeSetParams1D(c->gexec, c->gn_labels, io->labels, d_labels,
                                                 (size_t)n * 8, cudaMemcpyDeviceToHost));
      if (io && io->counts && c->gn_counts)
        DS_CK(cudaGraphExecMemcpyNodeSetParams1D(c->gexec, c->gn_counts, io->counts, d_counts64,
                                                 (size_t)n * 8, cudaMemcpyDeviceToHost));
      DS_CK(cudaGraphLaunch(c->gexec, s));
      // plan fields the timings need (no device work)
      pl.T = n_tiles(n);
      pl.all_items = n_items(pl.T);
      pl.cull = c->cull != 0 && pl.T > 1;
      pl.item_lo = 0;
      pl.item_hi = pl.all_items;
      pl.dense_units = pl.all_items * lane_blocks(d);
      pl.units_cap = pl.cull ? c->units_cap : (unsigned long long)pl.dense_units;
      pl.base = base_bytes(n, d) + (size_t)pl.units_cap * unit_bytes(pl.cull);
    } else if (use_graph && std::memcmp(key, c->seen_key, sizeof key) == 0) {
      // second call with this key: record the device pipeline and replay it
      if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
      }
      if (c->graph) {
        cudaGraphDestroy(c->graph);
        c->graph = nullptr;
      }
      const unsigned long long gen0 = g_alloc_generation.load();
      // the legacy default stream cannot be captured: record on the context's own
      // stream (nothing executes while recording) and launch on the caller's
      cudaStream_t cap = (s == nullptr || s == cudaStreamLegacy || s == cudaStreamPerThread)
                             ? c->stream
                             : s;
      DS_CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      ds_status st = enqueue_device(c, d_coords, n, d, eps_sq, min_pts, formula, mem_cap,
                                    d_labels, d_counts64, cap, pl, true, io);
      c->capturing = false;
      cudaGraph_t graph = nullptr;
      cudaError_t ce = cudaStreamEndCapture(cap, &graph);
      if (st != DS_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
      }
      DS_CK(ce);
      if (gen0 != g_alloc_generation.load()) {  // a buffer moved while recording: run eagerly
        cudaGraphDestroy(graph);
        st = enqueue_device(c, d_coords, n, d, eps_sq, min_pts, formula, mem_cap, d_labels,
                            d_counts64, s, pl, false, io);
        if (st != DS_OK) return st;
      } else {
        DS_CK(cudaGraphInstantiate(&c->gexec, graph, 0));
        c->graph = graph;
        c->gn_h2d = io ? find_copy_node(graph, io->coords) : nullptr;
        c->gn_labels = io ? find_copy_node(graph, io->labels) : nullptr;
        c->gn_counts = io ? find_copy_node(graph, io->counts) : nullptr;
        DS_CK(cudaGraphLaunch(c->gexec, s));
        const bool nodes_ok = !io || ((!io->coords || c->gn_h2d) && (!io->labels || c->gn_labels) &&
                                      (!io->counts || c->gn_counts));
        if (nodes_ok) {
          std::memcpy(c->gkey, key, sizeof key);
        } else {
          // a host copy could not be re-pointed on replay: this key runs eagerly from
          // now on (the launch above used this call's own buffers, so it is correct)
          std::memset(c->gkey, 0, sizeof key);
          c->no_graph_key = true;
        }
      }
    } else {
      ds_status st = enqueue_device(c, d_coords, n, d, eps_sq, min_pts, formula, mem_cap,
                                    d_labels, d_counts64, s, pl, false, io);
      if (st != DS_OK) return st;
      // key after this call's allocations: the next identical call records the graph
      key[7] = c->words_cap;
      key[8] = g_alloc_generation.load();
      key[11] = c->units_cap;
      std::memcpy(c->seen_key, key, sizeof key);
    }
    if (io && io->time_h2d) {  // the copy is done long before the pipeline: time it meanwhile
      DS_CK(cudaEventSynchronize(c->ev[0]));
      DS_CK(cudaEventElapsedTime(&io->h2d_ms, c->ev[5], c->ev[0]));
    }
    DS_CK(cudaEventRecord(c->ev[7], s));  // end of the device span (after the graph)
    DS_CK(cudaStreamSynchronize(s));
    bool retry = false;
    ds_status st = check_words(c, pl, mem_cap, &retry);
    if (st != DS_OK) return st;
    if (retry) {
      if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
      }
      st = retry_budget(attempt);
      if (st != DS_OK) return st;
      continue;
    }
    stage12_timings(c, pl, attempt, t);
    break;
  }
  if (t) {
    float f = 0, m = 0, k = 0, o = 0;
    // stage 1+2 / tile / stage 3 from the device stamps (copied back with the
    // scalars); events only if a stamp is missing or out of order
    const unsigned long long* st = c->h_scalars->stamps;
    if (c->event_timing) {
      DS_CK(cudaEventElapsedTime(&f, c->ev[0], c->ev[3]));
      DS_CK(cudaEventElapsedTime(&m, c->ev[3], c->ev[4]));
      DS_CK(cudaEventElapsedTime(&k, c->ev[1], c->ev[2]));
    } else if (st[ST_PREP] && st[ST_PREP] <= st[ST_TILE] && st[ST_TILE] <= st[ST_MERGE] &&
               st[ST_MERGE] <= st[ST_LABELS_DONE]) {
      f = (float)((st[ST_MERGE] - st[ST_PREP]) * 1e-6);
      k = (float)((st[ST_MERGE] - st[ST_TILE]) * 1e-6);
      m = (float)((st[ST_LABELS_DONE] - st[ST_MERGE]) * 1e-6);
    } else {  // no split available: the whole device part as stage 1+2
      DS_CK(cudaEventElapsedTime(&f, c->ev[0], c->ev[7]));
    }
    // the host copies after the label kernel: timed only with event timing (one more
    // cudaEventElapsedTime, a few us of host time after the sync, otherwise)
    if (c->event_timing && io && (io->labels || io->counts))
      DS_CK(cudaEventElapsedTime(&o, c->ev[4], c->ev[7]));
    t->fused_ms = f;
    t->merge_ms = m;
    t->tile_ms = k;
    t->d2h_ms = o;
    t->core_count = (int64_t)c->h_scalars->ncore;
    t->cluster_count = c->h_scalars->nclusters;
    t->device_bytes = (int64_t)held_bytes(c);
  }
  return DS_OK;
}

}  // namespace

extern "C" {

int ds_abi_version(void) { return DS_ABI_VERSION; }

const char* ds_build_info(void) {
  return "densescan_b200 sm_100a; eps-unit kernel TILE=512, warp units + cp.async staging, exact culling; "
         "union-find merge; built with nvcc " __DATE__;
}

const char* ds_last_error(void) { return g_error.c_str(); }

void ds_last_capacity(int64_t* required_bytes, int64_t* cap_bytes) {
  if (required_bytes) *required_bytes = g_required;
  if (cap_bytes) *cap_bytes = g_cap;
}

ds_status ds_ctx_create(int device, ds_ctx** out) {
  if (!out) {
    set_error("out: NULL");
    return DS_EINVAL;
  }
  *out = nullptr;
  int count = 0;
  DS_CK(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) {
    set_error("device: ordinal out of range");
    return DS_EINVAL;
  }
  DS_CK(cudaSetDevice(device));
  ds_ctx* c = new ds_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  for (int i = 0; e == cudaSuccess && i < 8; ++i) e = cudaEventCreate(&c->ev[i]);
  if (e == cudaSuccess) e = cudaMallocHost((void**)&c->h_scalars, sizeof(Scalars));
  if (e == cudaSuccess) {
    // device (mapped) alias of the page-locked scalar block: the label kernel's last
    // block writes it; without one the pipeline copies the scalars with a copy node
    void* p = nullptr;
    if (cudaHostGetDevicePointer(&p, c->h_scalars, 0) == cudaSuccess)
      c->h_scalars_dev = (unsigned long long*)p;
    cudaGetLastError();
  }
  if (e != cudaSuccess) {
    set_error(std::string("context creation failed: ") + cudaGetErrorString(e));
    ds_ctx_destroy(c);
    return DS_ECUDA;
  }
  *out = c;
  return DS_OK;
}

void ds_ctx_destroy(ds_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  Buf* all[] = {&c->coords64, &c->rec,    &c->cnt,    &c->core,   &c->corew,    &c->parent,
                &c->bmin,     &c->cmin,   &c->root,   &c->flag,   &c->partials, &c->labels,
                &c->counts64, &c->words,  &c->chunks, &c->scalars, &c->dense,
                &c->tbox,     &c->items,  &c->iflags, &c->ipartials,
                &c->rec_sorted, &c->perm, &c->inv, &c->keys, &c->keys_alt, &c->kidx,
                &c->sort_temp, &c->blk, &c->ulist, &c->uchunks, &c->ucnt,
                &c->dist, &c->dbits, &c->troot, &c->adjm, &c->ci32, &c->ci64, &c->cws, &c->soa64};
  for (Buf* b : all)
    if (b->p) cudaFree(b->p);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->h_scalars) cudaFreeHost(c->h_scalars);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->graph) cudaGraphDestroy(c->graph);
  delete c;
}

ds_status ds_run_dbscan_device(ds_ctx* c, const double* d_coords, int64_t n, int32_t d,
                               double eps_sq, int64_t min_pts, int32_t formula, int64_t mem_cap,
                               int64_t* d_labels, void* stream, ds_timings* t) {
  if (!c || !d_coords || !d_labels) {
    set_error("ctx, d_coords and d_labels must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, d, min_pts, formula);
  if (st != DS_OK) return st;
  DS_CK(cudaSetDevice(c->device));
  const double t0 = now_ms();
  ds_timings local{};
  st = pipeline(c, d_coords, n, d, eps_sq, min_pts, formula, mem_cap, d_labels, nullptr,
                (cudaStream_t)stream, &local);
  local.total_ms = now_ms() - t0;
  if (t) *t = local;
  return st;
}

ds_status ds_run_dbscan(ds_ctx* c, const double* coords, int64_t n, int32_t d, double eps_sq,
                        int64_t min_pts, int32_t formula, int64_t mem_cap, int64_t* labels_out,
                        int64_t* counts_out, ds_timings* t) {
  if (!c || !coords || !labels_out) {
    set_error("ctx, coords and labels_out must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, d, min_pts, formula);
  if (st != DS_OK) return st;
  DS_CK(cudaSetDevice(c->device));
  const double t0 = now_ms();
  ds_timings local{};
  const size_t in_bytes = (size_t)n * d * 8;
  DS_CK(ensure(c->coords64, in_bytes));
  DS_CK(ensure(c->labels, (size_t)n * 8));
  if (counts_out) DS_CK(ensure(c->counts64, (size_t)n * 8));
  cudaStream_t s = c->stream;
  // the coordinates go in before the graph launch, so the copy overlaps the launch;
  // the label / count copies out are part of the recorded pipeline
  DS_CK(cudaEventRecord(c->ev[5], s));
  DS_CK(cudaMemcpyAsync(c->coords64.p, coords, in_bytes, cudaMemcpyHostToDevice, s));
  HostIO io;
  io.labels = labels_out;
  io.counts = counts_out;
  io.time_h2d = true;
  st = pipeline(c, (const double*)c->coords64.p, n, d, eps_sq, min_pts, formula, mem_cap,
                (int64_t*)c->labels.p, counts_out ? (int64_t*)c->counts64.p : nullptr, s, &local,
                &io);
  if (st != DS_OK) return st;
  local.h2d_ms = io.h2d_ms;
  local.total_ms = now_ms() - t0;
  if (t) *t = local;
  return DS_OK;
}

ds_status ds_fused_build(ds_ctx* c, const double* coords, int64_t n, int32_t d, double eps_sq,
                         int64_t min_pts, int32_t formula, int64_t mem_cap, uint8_t* bits_out,
                         int64_t* counts_out, uint8_t* valid_out, ds_timings* t) {
  if (!c || !coords || !counts_out) {
    set_error("ctx, coords and counts_out must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, d, min_pts, formula);
  if (st != DS_OK) return st;
  DS_CK(cudaSetDevice(c->device));
  const double t0 = now_ms();
  ds_timings local{};
  cudaStream_t s = c->stream;
  const size_t in_bytes = (size_t)n * d * 8;
  DS_CK(ensure(c->coords64, in_bytes));
  DS_CK(ensure(c->counts64, (size_t)n * 8));
  DS_CK(cudaMemcpyAsync(c->coords64.p, coords, in_bytes, cudaMemcpyHostToDevice, s));
  Plan pl;
  for (int attempt = 1;; ++attempt) {
    DS_CK(cudaEventRecord(c->ev[0], s));
    st = stage12_enqueue(c, (const double*)c->coords64.p, n, d, eps_sq, formula, mem_cap, s, pl, 0,
                         1, bits_out != nullptr);
    if (st != DS_OK) return st;
    const int32_t* perm = c->sorted ? (const int32_t*)c->perm.p : nullptr;
    DS_CK(launch_counts_i64((const int32_t*)c->cnt.p, n, perm, (int64_t*)c->counts64.p, s));
    DS_CK(cudaEventRecord(c->ev[3], s));
    DS_CK(cudaMemcpyAsync(counts_out, c->counts64.p, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
    if (bits_out) {
      const int64_t stride = (n + 31) / 32;  // words per row
      const size_t dense = (size_t)n * stride * 4;
      DS_CK(ensure(c->dense, dense));
      DS_CK(cudaMemsetAsync(c->dense.p, 0, dense, s));
      Scalars* sc = (Scalars*)c->scalars.p;
      DS_CK(launch_export_bits((const uint2*)c->words.p, c->words_cap,
                               (const uint2*)c->uchunks.p, (const uint4*)c->chunks.p,
                               &sc->nonempty_count, perm, (uint32_t*)c->dense.p, stride, s));
      DS_CK(launch_bswap_rows((uint32_t*)c->dense.p, n, stride, s));
      const size_t row_bytes = (size_t)(n + 7) / 8;
      DS_CK(cudaMemcpy2DAsync(bits_out, row_bytes, c->dense.p, stride * 4, row_bytes, (size_t)n,
                              cudaMemcpyDeviceToHost, s));
    }
    DS_CK(cudaMemcpyAsync(c->h_scalars, c->scalars.p, sizeof(Scalars), cudaMemcpyDeviceToHost,
                          s));
    DS_CK(cudaStreamSynchronize(s));
    bool retry = false;
    st = check_words(c, pl, mem_cap, &retry);
    if (st != DS_OK) return st;
    if (retry) {
      st = retry_budget(attempt);
      if (st != DS_OK) return st;
      continue;
    }
    stage12_timings(c, pl, attempt, &local);
    break;
  }
  if (valid_out)
    for (int64_t i = 0; i < n; ++i) valid_out[i] = counts_out[i] >= min_pts ? 1 : 0;
  float f = 0, k = 0;
  DS_CK(cudaEventElapsedTime(&f, c->ev[0], c->ev[3]));
  DS_CK(cudaEventElapsedTime(&k, c->ev[1], c->ev[2]));
  local.fused_ms = f;
  local.tile_ms = k;
  local.device_bytes = (int64_t)held_bytes(c);
  local.total_ms = now_ms() - t0;
  if (t) *t = local;
  return DS_OK;
}

ds_status ds_ctx_set_option(ds_ctx* c, int32_t option, int64_t value) {
  if (!c) {
    set_error("ctx: NULL");
    return DS_EINVAL;
  }
  if (option == DS_OPT_TILE_CULL) {
    c->cull = value ? 1 : 0;
    return DS_OK;
  }
  if (option == DS_OPT_SPATIAL_SORT) {
    c->sort = value ? 1 : 0;
    return DS_OK;
  }
  if (option == DS_OPT_CUDA_GRAPH) {
    c->use_graph = value ? 1 : 0;
    return DS_OK;
  }
  if (option == DS_OPT_EVENT_TIMING) {
    c->event_timing = value ? 1 : 0;
    return DS_OK;
  }
  if (option == DS_OPT_STABLE_ORDER) {
    c->stable = value ? 1 : 0;
    return DS_OK;
  }
  if (option == DS_OPT_TEST_CAPACITY) {
    if (value < 0) {
      set_error("DS_OPT_TEST_CAPACITY: value must be >= 0");
      return DS_EINVAL;
    }
    c->test_cap = value;
    c->test_cap_pending = value > 0;
    if (c->gexec) {
      cudaGraphExecDestroy(c->gexec);
      c->gexec = nullptr;
    }
    std::memset(c->seen_key, 0, sizeof c->seen_key);
    return DS_OK;
  }
  set_error("option: unknown option id");
  return DS_EINVAL;
}

int64_t ds_ctx_get_option(ds_ctx* c, int32_t option) {
  if (c && option == DS_OPT_TILE_CULL) return c->cull;
  if (c && option == DS_OPT_SPATIAL_SORT) return c->sort;
  if (c && option == DS_OPT_CUDA_GRAPH) return c->use_graph;
  if (c && option == DS_OPT_EVENT_TIMING) return c->event_timing;
  if (c && option == DS_OPT_TEST_CAPACITY) return c->test_cap;
  if (c && option == DS_OPT_STABLE_ORDER) return c->stable;
  return -1;
}

ds_status ds_host_register(const void* ptr, size_t bytes) {
  if (!ptr || !bytes) {
    set_error("ptr/bytes: empty range");
    return DS_EINVAL;
  }
  cudaError_t e = cudaHostRegister(const_cast<void*>(ptr), bytes, cudaHostRegisterDefault);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    return DS_OK;
  }
  DS_CK(e);
  return DS_OK;
}

ds_status ds_host_unregister(const void* ptr) {
  cudaError_t e = cudaHostUnregister(const_cast<void*>(ptr));
  if (e != cudaSuccess) cudaGetLastError();  // not registered / already gone: nothing to do
  return DS_OK;
}

int64_t ds_tile_items(int64_t n) { return n < 1 ? 0 : n_items(n_tiles(n)); }

int ds_tile_side(void) { return TILE; }

ds_status ds_shard_stage12(ds_ctx* c, const double* d_coords, int64_t n, int32_t d, double eps_sq,
                           int32_t formula, int32_t rank, int32_t world, int64_t mem_cap,
                           int32_t* d_counts, void* stream, ds_timings* t) {
  if (!c || !d_coords || !d_counts) {
    set_error("ctx, d_coords and d_counts must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, d, 1, formula);
  if (st != DS_OK) return st;
  DS_CK(cudaSetDevice(c->device));
  const double t0 = now_ms();
  ds_timings local{};
  cudaStream_t s = (cudaStream_t)stream;
  Plan pl;
  for (int attempt = 1;; ++attempt) {
    DS_CK(cudaEventRecord(c->ev[0], s));
    st = stage12_enqueue(c, d_coords, n, d, eps_sq, formula, mem_cap, s, pl, rank, world);
    if (st != DS_OK) return st;
    // partial counts leave in original point order (the internal order is spatial)
    DS_CK(launch_permute_i32((const int32_t*)c->cnt.p, n,
                             c->sorted ? (const int32_t*)c->perm.p : nullptr, 1, d_counts, s));
    DS_CK(cudaEventRecord(c->ev[3], s));
    DS_CK(cudaMemcpyAsync(c->h_scalars, c->scalars.p, sizeof(Scalars), cudaMemcpyDeviceToHost,
                          s));
    DS_CK(cudaStreamSynchronize(s));
    bool retry = false;
    st = check_words(c, pl, mem_cap, &retry);
    if (st != DS_OK) return st;
    if (retry) {
      st = retry_budget(attempt);
      if (st != DS_OK) return st;
      continue;
    }
    stage12_timings(c, pl, attempt, &local);
    break;
  }
  float f = 0, k = 0;
  DS_CK(cudaEventElapsedTime(&f, c->ev[0], c->ev[3]));
  DS_CK(cudaEventElapsedTime(&k, c->ev[1], c->ev[2]));
  local.fused_ms = f;
  local.tile_ms = k;
  local.device_bytes = (int64_t)held_bytes(c);
  local.total_ms = now_ms() - t0;
  if (t) *t = local;
  return DS_OK;
}

ds_status ds_shard_stage3_local(ds_ctx* c, const int32_t* d_counts, int64_t n, int64_t min_pts,
                                int32_t* d_parent, int32_t* d_bmin, void* stream, ds_timings* t) {
  if (!c || !d_counts || !d_parent || !d_bmin) {
    set_error("ctx, d_counts, d_parent and d_bmin must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, 1, min_pts, DS_FORMULA_DIRECT);
  if (st != DS_OK) return st;
  if (!c->cnt.p || c->cnt.bytes < (size_t)n * 4 || !c->chunks.p) {
    set_error("ds_shard_stage3_local needs a preceding ds_shard_stage12 on this context");
    return DS_EINVAL;
  }
  DS_CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  DS_CK(cudaEventRecord(c->ev[3], s));
  DS_CK(launch_permute_i32(d_counts, n, c->sorted ? (const int32_t*)c->perm.p : nullptr, 0,
                           (int32_t*)c->cnt.p, s));
  MergeWs w = merge_ws(c, n);
  // per-block uniform roots of this shard's diagonal tiles (-1 elsewhere) and the
  // tile-root link table (zeroed by the stage 1+2 call): union_links' shortcuts
  w.blk_root = (int32_t*)c->troot.p;
  w.link_tab = (unsigned long long*)((char*)c->scalars.p + zr_links(n));
  w.link_mask = (1u << link_tab_bits(n)) - 1u;
  Scalars* sc = (Scalars*)c->scalars.p;
  DS_CK(cudaMemsetAsync(&sc->ncore, 0, sizeof(unsigned long long), s));
  DS_CK(launch_core_init(w, min_pts, s));
  DS_CK(launch_union_chunks(w, c->units, c->unit_lb, diag_range(c), CoreInit{}, s));
  DS_CK(cudaMemcpyAsync(d_parent, c->parent.p, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
  DS_CK(cudaMemcpyAsync(d_bmin, c->bmin.p, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
  DS_CK(cudaEventRecord(c->ev[4], s));
  DS_CK(cudaEventSynchronize(c->ev[4]));
  if (t) {
    float m = 0;
    DS_CK(cudaEventElapsedTime(&m, c->ev[3], c->ev[4]));
    t->merge_ms = m;
  }
  return DS_OK;
}

ds_status ds_shard_stage3_merge(ds_ctx* c, const int32_t* d_counts, int64_t n, int64_t min_pts,
                                const int32_t* d_parents, int32_t nparents, const int32_t* d_bmin,
                                int64_t* d_labels, void* stream, ds_timings* t) {
  if (!c || !d_counts || !d_parents || nparents < 1 || !d_bmin || !d_labels) {
    set_error("ctx, d_counts, d_parents (nparents >= 1), d_bmin and d_labels are required");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, 1, min_pts, DS_FORMULA_DIRECT);
  if (st != DS_OK) return st;
  DS_CK(cudaSetDevice(c->device));
  st = alloc_common(c, n, 1);
  if (st != DS_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  DS_CK(cudaEventRecord(c->ev[3], s));
  Scalars* sc = (Scalars*)c->scalars.p;
  DS_CK(cudaMemsetAsync(&sc->ncore, 0, sizeof(unsigned long long), s));
  DS_CK(launch_permute_i32(d_counts, n, c->sorted ? (const int32_t*)c->perm.p : nullptr, 0,
                           (int32_t*)c->cnt.p, s));
  MergeWs w = merge_ws(c, n);
  DS_CK(launch_core_init(w, min_pts, s));
  DS_CK(cudaMemcpyAsync(c->bmin.p, d_bmin, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
  DS_CK(launch_merge_forests(w, d_parents, nparents, s));
  DS_CK(launch_finalize(w, d_labels, s));
  DS_CK(cudaEventRecord(c->ev[4], s));
  DS_CK(cudaMemcpyAsync(c->h_scalars, c->scalars.p, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  DS_CK(cudaStreamSynchronize(s));
  if (t) {
    float m = 0;
    DS_CK(cudaEventElapsedTime(&m, c->ev[3], c->ev[4]));
    t->merge_ms = m;
    t->core_count = (int64_t)c->h_scalars->ncore;
    t->cluster_count = c->h_scalars->nclusters;
  }
  return DS_OK;
}

ds_status ds_shard_fold(ds_ctx* c, int32_t* d_parent, const int32_t* d_other, int64_t n,
                        void* stream) {
  if (!c || !d_parent || !d_other) {
    set_error("ctx, d_parent and d_other must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, 1, 1, DS_FORMULA_DIRECT);
  if (st != DS_OK) return st;
  DS_CK(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  DS_CK(launch_fold_forest(d_parent, d_other, n, s));
  DS_CK(cudaStreamSynchronize(s));
  return DS_OK;
}

// ---- materialising ladder (ds_dist.cu) ---------------------------------------------
namespace {

constexpr size_t DIST_BLOCK_BYTES = (size_t)4 << 30;  // device row block of the matrix

int64_t dist_rows_per_block(int64_t n) {
  const int64_t r = (int64_t)(DIST_BLOCK_BYTES / ((size_t)dist_pitch(n) * 4));
  return r < 1 ? 1 : (r > n ? n : r);
}

ds_status ladder_capacity(int64_t required, int64_t mem_cap, const char* what) {
  if (mem_cap > 0 && required > mem_cap) {
    set_capacity(required, mem_cap);
    set_error(std::string(what) + " exceeds the memory cap");
    return DS_ECAPACITY;
  }
  return DS_OK;
}

// coords (host float64 n x d) -> narrowed records on the device
ds_status ladder_prep(ds_ctx* c, const double* coords, int64_t n, int32_t d) {
  cudaStream_t s = c->stream;
  const size_t in_bytes = (size_t)n * d * 8;
  DS_CK(ensure(c->coords64, in_bytes));
  DS_CK(ensure(c->rec, (size_t)n * rec_stride(d) * 4));
  DS_CK(ensure(c->scalars, sizeof(Scalars)));
  DS_CK(cudaMemcpyAsync(c->coords64.p, coords, in_bytes, cudaMemcpyHostToDevice, s));
  DS_CK(cudaMemsetAsync(c->scalars.p, 0, sizeof(Scalars), s));
  DS_CK(launch_prep((const double*)c->coords64.p, n, d, (float*)c->rec.p,
                    &((Scalars*)c->scalars.p)->unsafe_flag, nullptr, nullptr, nullptr, s));
  return DS_OK;
}

}  // namespace

ds_status ds_dist_matrix(ds_ctx* c, const double* coords, int64_t n, int32_t d, int64_t mem_cap,
                         float* out, ds_timings* t) {
  if (!c || !coords || !out) {
    set_error("ctx, coords and out must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, d, 1, DS_FORMULA_DIRECT);
  if (st != DS_OK) return st;
  st = ladder_capacity(4 * n * n, mem_cap, "the n x n float32 distance matrix");  // kernels.py:156
  if (st != DS_OK) return st;
  DS_CK(cudaSetDevice(c->device));
  const double t0 = now_ms();
  cudaStream_t s = c->stream;
  st = ladder_prep(c, coords, n, d);
  if (st != DS_OK) return st;
  const int64_t pitch = dist_pitch(n), rows = dist_rows_per_block(n);
  DS_CK(ensure(c->dist, (size_t)rows * pitch * 4));
  float kernel_ms = 0.f;
  for (int64_t r0 = 0; r0 < n; r0 += rows) {
    const int64_t rb = std::min(rows, n - r0);
    DS_CK(cudaEventRecord(c->ev[1], s));
    DS_CK(launch_dist((const float*)c->rec.p, n, d, r0, rb, (float*)c->dist.p, s));
    DS_CK(cudaEventRecord(c->ev[2], s));
    DS_CK(cudaMemcpy2DAsync(out + r0 * n, (size_t)n * 4, c->dist.p, (size_t)pitch * 4,
                            (size_t)n * 4, (size_t)rb, cudaMemcpyDeviceToHost, s));
    DS_CK(cudaStreamSynchronize(s));
    float k = 0.f;
    DS_CK(cudaEventElapsedTime(&k, c->ev[1], c->ev[2]));
    kernel_ms += k;
  }
  if (t) {
    ds_timings local{};
    local.tile_ms = kernel_ms;
    local.pairs_evaluated = n * n;
    local.device_bytes = (int64_t)held_bytes(c);
    local.total_ms = now_ms() - t0;
    *t = local;
  }
  return DS_OK;
}

ds_status ds_dist_threshold(ds_ctx* c, const float* dist, int64_t n, double eps_sq, int64_t min_pts,
                            int64_t mem_cap, uint8_t* bits_out, int64_t* counts_out,
                            uint8_t* valid_out, ds_timings* t) {
  if (!c || !dist || !bits_out || !counts_out) {
    set_error("ctx, dist, bits_out and counts_out must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, 1, min_pts, DS_FORMULA_DIRECT);
  if (st != DS_OK) return st;
  const int64_t rb_bytes = (n + 7) / 8;
  st = ladder_capacity(n * rb_bytes, mem_cap, "the n x ceil(n/8) neighbourhood matrix");
  if (st != DS_OK) return st;
  DS_CK(cudaSetDevice(c->device));
  const double t0 = now_ms();
  cudaStream_t s = c->stream;
  const float eps32 = (float)eps_sq;  // kernels.py:297
  const int64_t pitch = dist_pitch(n), rows = dist_rows_per_block(n);
  DS_CK(ensure(c->dist, (size_t)rows * pitch * 4));
  DS_CK(ensure(c->dbits, (size_t)rows * rb_bytes));
  DS_CK(ensure(c->counts64, (size_t)n * 8));
  float kernel_ms = 0.f;
  for (int64_t r0 = 0; r0 < n; r0 += rows) {
    const int64_t rb = std::min(rows, n - r0);
    DS_CK(cudaMemcpy2DAsync(c->dist.p, (size_t)pitch * 4, dist + r0 * n, (size_t)n * 4,
                            (size_t)n * 4, (size_t)rb, cudaMemcpyHostToDevice, s));
    DS_CK(cudaEventRecord(c->ev[1], s));
    DS_CK(launch_threshold((const float*)c->dist.p, n, rb, eps32, (uint8_t*)c->dbits.p,
                           (int64_t*)c->counts64.p + r0, s));
    DS_CK(cudaEventRecord(c->ev[2], s));
    DS_CK(cudaMemcpyAsync(bits_out + r0 * rb_bytes, c->dbits.p, (size_t)rb * rb_bytes,
                          cudaMemcpyDeviceToHost, s));
    DS_CK(cudaStreamSynchronize(s));
    float k = 0.f;
    DS_CK(cudaEventElapsedTime(&k, c->ev[1], c->ev[2]));
    kernel_ms += k;
  }
  DS_CK(cudaMemcpy(counts_out, c->counts64.p, (size_t)n * 8, cudaMemcpyDeviceToHost));
  if (valid_out)
    for (int64_t i = 0; i < n; ++i) valid_out[i] = counts_out[i] >= min_pts ? 1 : 0;
  if (t) {
    ds_timings local{};
    local.merge_ms = kernel_ms;
    local.device_bytes = (int64_t)held_bytes(c);
    local.total_ms = now_ms() - t0;
    *t = local;
  }
  return DS_OK;
}

ds_status ds_dist_build(ds_ctx* c, const double* coords, int64_t n, int32_t d, double eps_sq,
                        int64_t min_pts, int64_t mem_cap, uint8_t* bits_out, int64_t* counts_out,
                        uint8_t* valid_out, ds_timings* t) {
  if (!c || !coords || !bits_out || !counts_out) {
    set_error("ctx, coords, bits_out and counts_out must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, d, min_pts, DS_FORMULA_DIRECT);
  if (st != DS_OK) return st;
  const int64_t rb_bytes = (n + 7) / 8;
  st = ladder_capacity(4 * n * n, mem_cap, "the n x n float32 distance matrix");
  if (st != DS_OK) return st;
  st = ladder_capacity(n * rb_bytes, mem_cap, "the n x ceil(n/8) neighbourhood matrix");
  if (st != DS_OK) return st;
  DS_CK(cudaSetDevice(c->device));
  const double t0 = now_ms();
  cudaStream_t s = c->stream;
  st = ladder_prep(c, coords, n, d);
  if (st != DS_OK) return st;
  const float eps32 = (float)eps_sq;
  const int64_t pitch = dist_pitch(n), rows = dist_rows_per_block(n);
  DS_CK(ensure(c->dist, (size_t)rows * pitch * 4));
  DS_CK(ensure(c->dbits, (size_t)n * rb_bytes));
  DS_CK(ensure(c->counts64, (size_t)n * 8));
  float dist_ms = 0.f, thr_ms = 0.f;
  for (int64_t r0 = 0; r0 < n; r0 += rows) {
    const int64_t rb = std::min(rows, n - r0);
    DS_CK(cudaEventRecord(c->ev[1], s));
    DS_CK(launch_dist((const float*)c->rec.p, n, d, r0, rb, (float*)c->dist.p, s));
    DS_CK(cudaEventRecord(c->ev[2], s));
    DS_CK(launch_threshold((const float*)c->dist.p, n, rb, eps32,
                           (uint8_t*)c->dbits.p + r0 * rb_bytes, (int64_t*)c->counts64.p + r0, s));
    DS_CK(cudaEventRecord(c->ev[3], s));
    DS_CK(cudaEventSynchronize(c->ev[3]));
    float a = 0.f, b = 0.f;
    DS_CK(cudaEventElapsedTime(&a, c->ev[1], c->ev[2]));
    DS_CK(cudaEventElapsedTime(&b, c->ev[2], c->ev[3]));
    dist_ms += a;
    thr_ms += b;
  }
  DS_CK(cudaMemcpyAsync(bits_out, c->dbits.p, (size_t)n * rb_bytes, cudaMemcpyDeviceToHost, s));
  DS_CK(cudaMemcpyAsync(counts_out, c->counts64.p, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
  DS_CK(cudaStreamSynchronize(s));
  if (valid_out)
    for (int64_t i = 0; i < n; ++i) valid_out[i] = counts_out[i] >= min_pts ? 1 : 0;
  if (t) {
    ds_timings local{};
    local.tile_ms = dist_ms;
    local.merge_ms = thr_ms;
    local.pairs_evaluated = n * n;
    local.device_bytes = (int64_t)held_bytes(c);
    local.total_ms = now_ms() - t0;
    *t = local;
  }
  return DS_OK;
}

}  // extern "C"

namespace {

// Stage 3 from a reference-layout matrix: union-find over (bits AND core x core) with
// core = cnt32 >= min_pts, lowest-core borders, canonical labels.
ds_status merge_bits_impl(ds_ctx* c, const uint8_t* bits, const std::vector<int32_t>& cnt32,
                          int64_t n, int64_t min_pts, int64_t* labels_out, ds_timings* t) {
  DS_CK(cudaSetDevice(c->device));
  const double t0 = now_ms();
  ds_timings local{};
  cudaStream_t s = c->stream;
  ds_status st = alloc_common(c, n, 1);
  if (st != DS_OK) return st;
  c->sorted = false;  // the reference-layout matrix is in original order
  const int64_t stride = (n + 31) / 32;
  const size_t dense = (size_t)n * stride * 4;
  const size_t row_bytes = (size_t)(n + 7) / 8;
  DS_CK(ensure(c->dense, dense));
  DS_CK(ensure(c->labels, (size_t)n * 8));
  DS_CK(cudaEventRecord(c->ev[0], s));
  DS_CK(cudaMemsetAsync(c->scalars.p, 0, sizeof(Scalars), s));
  DS_CK(cudaMemsetAsync(c->dense.p, 0, dense, s));
  DS_CK(cudaMemcpy2DAsync(c->dense.p, stride * 4, bits, row_bytes, row_bytes, (size_t)n,
                          cudaMemcpyHostToDevice, s));
  DS_CK(cudaMemcpyAsync(c->cnt.p, cnt32.data(), (size_t)n * 4, cudaMemcpyHostToDevice, s));
  DS_CK(launch_bswap_rows((uint32_t*)c->dense.p, n, stride, s));
  MergeWs w = merge_ws(c, n);
  DS_CK(launch_core_init(w, min_pts, s));
  DS_CK(cudaEventRecord(c->ev[3], s));
  DS_CK(launch_union_dense(w, (const uint32_t*)c->dense.p, stride, s));
  DS_CK(launch_finalize(w, (int64_t*)c->labels.p, s));
  DS_CK(cudaEventRecord(c->ev[4], s));
  DS_CK(cudaMemcpyAsync(labels_out, c->labels.p, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
  DS_CK(cudaMemcpyAsync(c->h_scalars, c->scalars.p, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  DS_CK(cudaStreamSynchronize(s));
  float m = 0;
  DS_CK(cudaEventElapsedTime(&m, c->ev[3], c->ev[4]));
  local.merge_ms = m;
  local.core_count = (int64_t)c->h_scalars->ncore;
  local.cluster_count = c->h_scalars->nclusters;
  local.device_bytes = (int64_t)held_bytes(c);
  local.total_ms = now_ms() - t0;
  if (t) *t = local;
  return DS_OK;
}

// reference-layout rows (n x ceil(n/8) bytes) -> native words on the device (c->dense)
ds_status upload_rows(ds_ctx* c, const uint8_t* bits, int64_t n, int64_t* stride_out) {
  cudaStream_t s = c->stream;
  const int64_t stride = (n + 31) / 32;
  const size_t dense = (size_t)n * stride * 4;
  const size_t row_bytes = (size_t)(n + 7) / 8;
  DS_CK(ensure(c->dense, dense));
  DS_CK(cudaMemsetAsync(c->dense.p, 0, dense, s));
  DS_CK(cudaMemcpy2DAsync(c->dense.p, stride * 4, bits, row_bytes, row_bytes, (size_t)n,
                          cudaMemcpyHostToDevice, s));
  DS_CK(launch_bswap_rows((uint32_t*)c->dense.p, n, stride, s));
  *stride_out = stride;
  return DS_OK;
}

// native words (m rows of stride words in buf) -> reference-layout rows on the host
ds_status download_rows(ds_ctx* c, uint32_t* words, int64_t m, int64_t stride, uint8_t* out) {
  cudaStream_t s = c->stream;
  DS_CK(launch_bswap_rows(words, m, stride, s));
  const size_t row_bytes = (size_t)(m + 7) / 8;
  DS_CK(cudaMemcpy2DAsync(out, row_bytes, words, stride * 4, row_bytes, (size_t)m,
                          cudaMemcpyDeviceToHost, s));
  return DS_OK;
}

}  // namespace

extern "C" {

ds_status ds_merge_bits(ds_ctx* c, const uint8_t* bits, const int64_t* counts, const uint8_t* valid,
                        int64_t n, int64_t min_pts, int64_t* labels_out, ds_timings* t) {
  if (!c || !bits || !counts || !valid || !labels_out) {
    set_error("ctx, bits, counts, valid and labels_out must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, 1, min_pts, DS_FORMULA_DIRECT);
  if (st != DS_OK) return st;
  for (int64_t i = 0; i < n; ++i) {
    if ((counts[i] >= min_pts) != (valid[i] != 0)) {  // merge.py:141-145
      set_error("valid[" + std::to_string(i) + "] disagrees with neighbor_count[" +
                std::to_string(i) + "] >= min_pts");
      return DS_EINCONSISTENT;
    }
  }
  std::vector<int32_t> cnt32((size_t)n);
  for (int64_t i = 0; i < n; ++i) cnt32[i] = (int32_t)std::min<int64_t>(counts[i], 0x7fffffff);
  return merge_bits_impl(c, bits, cnt32, n, min_pts, labels_out, t);
}

ds_status ds_merge_bits_core(ds_ctx* c, const uint8_t* bits, const uint8_t* core, int64_t n,
                             int64_t* labels_out, ds_timings* t) {
  if (!c || !bits || !core || !labels_out) {
    set_error("ctx, bits, core and labels_out must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, 1, 1, DS_FORMULA_DIRECT);
  if (st != DS_OK) return st;
  // the core set is taken as given (merge_warshall, merge.py:218-238, reads
  // valid_vec.valid and never checks it against the counts): core <=> 1 >= 1
  std::vector<int32_t> flag((size_t)n);
  for (int64_t i = 0; i < n; ++i) flag[i] = core[i] ? 1 : 0;
  return merge_bits_impl(c, bits, flag, n, 1, labels_out, t);
}

ds_status ds_core_adjacency(ds_ctx* c, const uint8_t* bits, const uint8_t* valid, int64_t n,
                            int64_t m, int64_t* core_indices_out, uint8_t* adj_out,
                            ds_timings* t) {
  if (!c || !bits || !valid || (m > 0 && (!core_indices_out || !adj_out))) {
    set_error("ctx, bits, valid (and core_indices_out, adj_out when m > 0) must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, 1, 1, DS_FORMULA_DIRECT);
  if (st != DS_OK) return st;
  if (m < 0 || m > n) {
    set_error("m: must be the number of valid points");
    return DS_EINVAL;
  }
  DS_CK(cudaSetDevice(c->device));
  const double t0 = now_ms();
  cudaStream_t s = c->stream;
  ds_status a = alloc_common(c, n, 1);
  if (a != DS_OK) return a;
  int64_t stride_n = 0;
  st = upload_rows(c, bits, n, &stride_n);
  if (st != DS_OK) return st;
  DS_CK(ensure(c->core, (size_t)n));
  DS_CK(cudaMemcpyAsync(c->core.p, valid, (size_t)n, cudaMemcpyHostToDevice, s));
  DS_CK(ensure(c->ci32, (size_t)std::max<int64_t>(m, 1) * 4));
  DS_CK(ensure(c->ci64, (size_t)std::max<int64_t>(m, 1) * 8));
  Scalars* sc = (Scalars*)c->scalars.p;
  DS_CK(cudaEventRecord(c->ev[3], s));
  DS_CK(launch_core_index((const uint8_t*)c->core.p, n, (int32_t*)c->flag.p,
                          (int32_t*)c->partials.p, &sc->kept32, (int32_t*)c->ci32.p,
                          (int64_t*)c->ci64.p, s));
  const int64_t stride_m = (m + 31) / 32;
  if (m > 0) {
    DS_CK(ensure(c->adjm, (size_t)m * stride_m * 4));
    DS_CK(launch_core_gather((const uint32_t*)c->dense.p, stride_n, (const int32_t*)c->ci32.p, m,
                             (uint32_t*)c->adjm.p, stride_m, s));
  }
  DS_CK(cudaEventRecord(c->ev[4], s));
  int32_t m_dev = 0;
  DS_CK(cudaMemcpyAsync(&c->h_scalars->kept32, &sc->kept32, 4, cudaMemcpyDeviceToHost, s));
  DS_CK(cudaStreamSynchronize(s));
  m_dev = c->h_scalars->kept32;
  if (m_dev != m) {
    set_error("m: " + std::to_string(m) + " given but valid has " + std::to_string(m_dev) +
              " set entries");
    return DS_EINVAL;
  }
  if (m > 0) {
    DS_CK(cudaMemcpyAsync(core_indices_out, c->ci64.p, (size_t)m * 8, cudaMemcpyDeviceToHost, s));
    st = download_rows(c, (uint32_t*)c->adjm.p, m, stride_m, adj_out);
    if (st != DS_OK) return st;
    DS_CK(cudaStreamSynchronize(s));
  }
  if (t) {
    ds_timings local{};
    float k = 0;
    DS_CK(cudaEventElapsedTime(&k, c->ev[3], c->ev[4]));
    local.merge_ms = k;
    local.core_count = m;
    local.device_bytes = (int64_t)held_bytes(c);
    local.total_ms = now_ms() - t0;
    *t = local;
  }
  return DS_OK;
}

ds_status ds_serial_dbscan(ds_ctx* c, const double* coords, int64_t n, int32_t d, double eps_sq,
                           int64_t min_pts, int64_t* labels_out, int64_t* counts_out,
                           ds_timings* t) {
  if (!c || !coords || !labels_out) {
    set_error("ctx, coords and labels_out must be non-NULL");
    return DS_EINVAL;
  }
  ds_status st = check_args(n, d, min_pts, DS_FORMULA_DIRECT);
  if (st != DS_OK) return st;
  DS_CK(cudaSetDevice(c->device));
  const double t0 = now_ms();
  cudaStream_t s = c->stream;
  st = alloc_common(c, n, 1);
  if (st != DS_OK) return st;
  c->sorted = false;
  const int64_t stride = (n + 31) / 32;
  const size_t in_bytes = (size_t)n * d * 8;
  DS_CK(ensure(c->coords64, in_bytes));
  DS_CK(ensure(c->soa64, in_bytes));
  DS_CK(ensure(c->dense, (size_t)n * stride * 4));
  DS_CK(ensure(c->labels, (size_t)n * 8));
  DS_CK(ensure(c->counts64, (size_t)n * 8));
  DS_CK(cudaMemcpyAsync(c->coords64.p, coords, in_bytes, cudaMemcpyHostToDevice, s));
  DS_CK(cudaMemsetAsync(c->scalars.p, 0, sizeof(Scalars), s));
  DS_CK(cudaEventRecord(c->ev[0], s));
  DS_CK(launch_serial_words((const double*)c->coords64.p, n, d, eps_sq, (double*)c->soa64.p,
                            (uint32_t*)c->dense.p, stride, (int32_t*)c->cnt.p, s));
  DS_CK(cudaEventRecord(c->ev[1], s));
  MergeWs w = merge_ws(c, n);
  DS_CK(launch_core_init(w, min_pts, s));
  DS_CK(cudaEventRecord(c->ev[2], s));
  DS_CK(launch_union_dense(w, (const uint32_t*)c->dense.p, stride, s));
  DS_CK(launch_finalize(w, (int64_t*)c->labels.p, s));
  DS_CK(cudaEventRecord(c->ev[3], s));
  DS_CK(cudaMemcpyAsync(labels_out, c->labels.p, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
  if (counts_out) {
    DS_CK(launch_counts_i64((const int32_t*)c->cnt.p, n, nullptr, (int64_t*)c->counts64.p, s));
    DS_CK(cudaMemcpyAsync(counts_out, c->counts64.p, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
  }
  DS_CK(cudaMemcpyAsync(c->h_scalars, c->scalars.p, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  DS_CK(cudaStreamSynchronize(s));
  if (t) {
    ds_timings local{};
    float a = 0, b = 0, m = 0;
    DS_CK(cudaEventElapsedTime(&a, c->ev[0], c->ev[1]));
    DS_CK(cudaEventElapsedTime(&b, c->ev[1], c->ev[2]));
    DS_CK(cudaEventElapsedTime(&m, c->ev[2], c->ev[3]));
    local.tile_ms = a;   // dist_sq stage (fused with the eps test and counts)
    local.fused_ms = b;  // core flags
    local.merge_ms = m;
    local.pairs_evaluated = n * n;
    local.core_count = (int64_t)c->h_scalars->ncore;
    local.cluster_count = c->h_scalars->nclusters;
    local.device_bytes = (int64_t)held_bytes(c);
    local.total_ms = now_ms() - t0;
    *t = local;
  }
  return DS_OK;
}

ds_status ds_warshall_closure(ds_ctx* c, const uint8_t* adj, int64_t m, uint8_t* closed_out,
                              ds_timings* t) {
  if (!c || (m > 0 && (!adj || !closed_out))) {
    set_error("ctx, adj and closed_out must be non-NULL");
    return DS_EINVAL;
  }
  if (m < 0 || m >= (int64_t)0x7fffffff) {
    set_error("m: must be in [0, 2^31)");
    return DS_EINVAL;
  }
  if (m == 0) {
    if (t) *t = ds_timings{};
    return DS_OK;
  }
  DS_CK(cudaSetDevice(c->device));
  const double t0 = now_ms();
  cudaStream_t s = c->stream;
  int64_t stride = 0;
  ds_status st = upload_rows(c, adj, m, &stride);
  if (st != DS_OK) return st;
  DS_CK(ensure(c->cws, (size_t)(m + 32) * 4));
  DS_CK(cudaEventRecord(c->ev[3], s));
  uint32_t* C = (uint32_t*)c->dense.p;
  DS_CK(launch_closure(C, m, stride, (uint32_t*)c->cws.p + m, (uint32_t*)c->cws.p, s));
  DS_CK(cudaEventRecord(c->ev[4], s));
  st = download_rows(c, C, m, stride, closed_out);
  if (st != DS_OK) return st;
  DS_CK(cudaStreamSynchronize(s));
  if (t) {
    ds_timings local{};
    float k = 0;
    DS_CK(cudaEventElapsedTime(&k, c->ev[3], c->ev[4]));
    local.merge_ms = k;
    local.device_bytes = (int64_t)held_bytes(c);
    local.total_ms = now_ms() - t0;
    *t = local;
  }
  return DS_OK;
}

}  // extern "C"
