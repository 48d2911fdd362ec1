// Internal declarations shared by the densescan_b200 translation units.
//
// Data layout in HBM:
//   rec      float32 [n][S]      S = roundup4(d+1): d narrowed coordinates, then the
//                                squared norm P (algebraic formula), zero pad.
//   cnt      int32   [n]         neighbour counts incl. self (kernels.py:331)
//   core     uint8   [n]         cnt >= min_pts            (kernels.py:335)
//   corew    uint32  [ceil(n/32)] core flags as adjacency words (bit 31-t <-> point 32w+t)
//   words    uint2   [cap]       {32-bit adjacency word, local row << 4 | column word}: the
//                                non-zero words of the upper-triangle tile pairs, i.e. the
//                                bit-packed neighbourhood matrix without its empty part,
//                                grouped in one contiguous chunk per work unit
//   uchunks  uint2   [units]     {first word lo, count | first word hi << 16}
//   dir      uint4   [items]     tile pairs with words: {a << 16 | b, first unit, units, hi}
//   parent   int32   [n]         union-find forest over core points (root = min index)
//   bmin     int32   [n]         lowest in-range core of each non-core point
//   root/cmin/flag/id int32 [n]  canonical relabel workspace
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/densescan_b200.h"

namespace ds {

// ---- tile geometry of the eps-tile kernel ---------------------------------------
constexpr int TILE = 512;             // points per tile side
constexpr int NT = 128;               // threads per CTA
constexpr int KPT = TILE / NT;        // lane points owned by one thread
constexpr int WPR = TILE / 32;        // adjacency words per point per tile
constexpr int BSTRIDE = TILE + 8;     // smem stride of one word column (bank padding)
constexpr int MAX_D = 64;
constexpr int DS_MAX_DEVICES = 64;    // per-device launch configuration caches
constexpr int32_t NONE = 0x7fffffff;  // "no core" marker in bmin / cmin

int padded_dim(int d);  // tile kernels are instantiated for d in {1,2,3,4,8,16,32,64}
inline int rec_stride(int d) { return ((padded_dim(d) + 1) + 3) / 4 * 4; }
inline int64_t n_tiles(int64_t n) { return (n + TILE - 1) / TILE; }
inline int64_t n_items(int64_t T) { return T * (T + 1) / 2; }

// coordinates beyond this magnitude could overflow float32 inside the pair
// arithmetic (|d2| <= 4*d*max|c|^2); such inputs take the compare-based path
constexpr float SAFE_ABS = 1.0e17f;

// Row unit of the eps-tile kernel: (a block of 32*KP consecutive points of tile a,
// held in registers by one warp) x (a mask of the 32-point column blocks of tile b
// it evaluates, staged through shared memory one block at a time). KP = 4 / 2 / 1
// lane points per lane for d <= 8 / 32 / 64; each column block of a row unit owns
// one chunk entry (unit * WPR + column block).
inline int unit_kp(int d) { return padded_dim(d) <= 16 ? 4 : (padded_dim(d) <= 32 ? 2 : 1); }
inline int lane_blocks(int d) { return TILE / (32 * unit_kp(d)); }
// chunk entries per tile pair: one per (lane block, column block)
inline int units_per_tile(int d) { return lane_blocks(d) * WPR; }
// Each warp of the eps-tile kernel reserves adjacency-word slots WORD_RUN at a time
// (one global atomic per run instead of one per unit); a unit emits at most 32*KP
// <= 128 words, so a run's unused tail is < 128 slots. Bound on the reserved total:
// words * WORD_RUN / (WORD_RUN - 128) + warps * WORD_RUN.
constexpr int WORD_RUN = 256;

// KP = 4: a (lane block, tile pair) with many kept column blocks is listed as units of
// at most unit_cols column blocks — 2 for inputs up to UNIT_SMALL_N points (few units
// per warp: the end of the eps launch waits on the last ones), else 4 (fewer units, less
// per-unit overhead in the eps and union kernels)
constexpr int64_t UNIT_SMALL_N = (int64_t)1 << 18;

struct UnitArgs {
  const float* rec;
  int64_t n;
  int32_t T;                            // tiles per side
  float eps32;
  float negz = -0.0f;                   // the FFMA2 addend of exact products (ds_tile.cu)
  int32_t* cnt;
  uint2* words;                         // {32-bit word, local row << 4 | column word}
  unsigned long long words_cap;
  unsigned long long* words_count;
  uint2* uchunks;                       // per (unit, column block) {first word lo,
                                        //   count | first word hi << 16}
  const uint32_t* item_list;            // culled tile pairs (a << 16 | b), or nullptr: triangle
  const uint2* unit_list;               // culled row units of this shard {a << 16 | b,
                                        // lb << 16 | column mask}, or nullptr: unit
                                        // q * LB + lb of the triangle
  const unsigned long long* unit_count; // length of unit_list (device)
  unsigned long long units_cap;         // capacity of unit_list (culled); uchunks: * WPR
  int64_t dense_units;                  // all_items * LB (dense schedule)
  int32_t shard_rank, shard_world;      // slice of the units this launch evaluates
  const uint32_t* unsafe_flag;
  unsigned long long* pairs_done;       // ordered pairs evaluated (32 x 32*KP per unit)
  unsigned long long* work_ctr;         // batch counter (zeroed before the launch)
  unsigned long long* stamps = nullptr; // %globaltimer stamps (Stamp), or nullptr
};

// Device-side stage boundaries of one call, in %globaltimer ns, written by thread 0 of
// block 0 after its griddep_wait (i.e. once the preceding kernel has completed):
// the host turns them into the stage timings without cudaEventElapsedTime calls
// (about 3 us of host time each, on the critical path of every call).
enum Stamp { ST_PREP = 0, ST_TILE = 1, ST_MERGE = 2, ST_LABELS_DONE = 3, ST_COUNT = 4 };

// ---- programmatic dependent launch ------------------------------------------------
// Pipeline kernels are launched with programmatic stream serialization: a kernel may
// be scheduled while its predecessor in the stream drains (hiding the launch and
// CTA ramp of ~20 small dependent kernels per call); each such kernel executes
// griddep_wait() first, which returns once the predecessor grid has completed and
// its memory is visible (a no-op for an ordinary launch).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void stamp(unsigned long long* st, int k) {
  if (st && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    st[k] = t;
  }
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// ---- item <-> tile pair: items enumerate the upper triangle a <= b in row order ----
__device__ __forceinline__ int64_t row_offset(int64_t a, int64_t T) {
  return a * T - a * (a - 1) / 2;
}
__device__ __forceinline__ void decode_item(int64_t q, int64_t T, int& a, int& b) {
  const double tt = 2.0 * (double)T + 1.0;
  int64_t r = (int64_t)floor((tt - sqrt(tt * tt - 8.0 * (double)q)) * 0.5);
  if (r < 0) r = 0;
  if (r > T - 1) r = T - 1;
  while (r + 1 <= T - 1 && row_offset(r + 1, T) <= q) ++r;
  while (r > 0 && row_offset(r, T) > q) --r;
  a = (int)r;
  b = (int)(r + (q - row_offset(r, T)));
}

// Units this launch evaluates: the culled list is built per shard (its items), the
// dense triangle order is sliced into equal unit ranges.
__device__ __forceinline__ void unit_range(const UnitArgs& A, long long& lo, long long& hi) {
  if (A.unit_list) {
    const unsigned long long c = *A.unit_count;
    lo = 0;
    hi = (long long)(c < A.units_cap ? c : A.units_cap);
  } else {
    const long long U = A.dense_units;
    lo = U * A.shard_rank / A.shard_world;
    hi = U * (A.shard_rank + 1) / A.shard_world;
  }
}

// order-preserving float -> uint (for atomicMin/Max bounding boxes)
__device__ __forceinline__ unsigned int ord_bits(float f) {
  const unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_bits(unsigned int u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// Super tiles: 32 consecutive tiles (16k points). Their boxes (d <= 4) let the tile
// culling test a tile row against a super tile first (T^2 / 32 instead of T^2 / 2 box
// tests at C5). Layout per super tile (uint, zeroed per call, reduced with atomicMax):
// {~ord lo[dpad], ord hi[dpad], ord maxnorm}; SUPER_BS words per super tile.
constexpr int SUPER = 32;
constexpr int SUPER_BS = 2 * 4 + 1;
inline int64_t n_supers(int64_t T) { return (T + SUPER - 1) / SUPER; }
__device__ __forceinline__ void super_box_add(unsigned int* super, int64_t tile, int dpad, int k,
                                              float mn, float mx) {
  unsigned int* sb = super + (tile / SUPER) * SUPER_BS;
  if (k < dpad) {
    atomicMax(&sb[k], ~ord_bits(mn));
    atomicMax(&sb[dpad + k], ord_bits(mx));
  } else {
    atomicMax(&sb[2 * dpad], ord_bits(mx));
  }
}

// ---- launchers (ds_tile.cu) ---------------------------------------------------
// bbox (nullable): 8 uints {~ord lo[4], ord hi[4]} of the first min(d, 4) dimensions
// (the spatial sort's grid).
// bbox words must be zero on entry (lo is stored as ~ord_bits, hi as ord_bits, so
// both reduce with atomicMax); cnt (nullable): zeroed here for stage 1's counts
cudaError_t launch_prep(const double* coords, int64_t n, int d, float* rec, uint32_t* unsafe_flag,
                        unsigned long long* stamps,
                        unsigned int* bbox, int32_t* cnt, cudaStream_t s);
cudaError_t launch_units_kernel(const UnitArgs& a, int d, int formula, int sm_count,
                                cudaStream_t s);
// culled schedule: the row-unit list of this shard (kept items q = rank + k * world),
// pieces of unit_cols column blocks; item_units[q] = {first unit, units}; for a
// diagonal pair (a, a) also diag_range[a] = {first unit lo, first unit hi << 16 |
// units} (must be zero on entry)
cudaError_t launch_unit_list(const float* blk, int64_t n, int d, float eps32, int formula,
                             const uint32_t* unsafe_flag, const uint32_t* item_list,
                             const unsigned long long* kept, int64_t all_items, int rank, int world,
                             uint2* unit_list, unsigned long long units_cap,
                             unsigned long long* unit_count, uint2* item_units, uint2* diag_range,
                             cudaStream_t s);
// per tile pair with words: {a << 16 | b, first unit lo, units, first unit hi} (atomic append)
// core_init's job (core flags, core words, union-find init), fused into the diagonal
// union pass on one GPU (the counts are complete after the eps-tile kernel)
struct CoreInit {
  const int32_t* cnt = nullptr;  // nullptr: skip
  int64_t n = 0, min_pts = 0;
  uint8_t* core = nullptr;
  uint32_t* corew = nullptr;
  int32_t* parent = nullptr;
  int32_t* bmin = nullptr;
  int32_t* cmin = nullptr;
  unsigned long long* ncore = nullptr;
};
// tile pairs with words (the reference-layout export walks them)
cudaError_t launch_unit_dir(const UnitArgs& a, int d, int64_t all_items, const uint2* item_units,
                            const unsigned long long* kept, uint4* dir,
                            unsigned long long* dir_count, cudaStream_t s);
// 32-point block boxes [block][lo(dpad), hi(dpad), maxnorm] for sub-tile culling
cudaError_t launch_block_bounds(const float* rec, int64_t n, int d, float* blk, cudaStream_t s);
// tile bounding boxes + list of tile pairs that are not provably empty
// bounds_ready: lo / hi / maxnorm were filled by the spatial sort (SortBounds)
// ordered = false (one GPU): the hierarchical cull may append the kept pairs in any order
cudaError_t launch_cull(const float* rec, int64_t n, int d, float eps32, int formula,
                        const uint32_t* unsafe_flag, float* lo, float* hi, float* maxnorm,
                        unsigned int* super, int32_t* flags, int32_t* partials,
                        int32_t* total_kept, uint32_t* list, unsigned long long* count,
                        bool bounds_ready, bool ordered, cudaStream_t s);
// exclusive prefix sum of int32 data in place (3 kernels); *total = sum
cudaError_t launch_exclusive_scan(int32_t* data, int64_t n, int32_t* partials, int32_t* total,
                                  cudaStream_t s);
size_t tile_smem_bytes(int d);

// ---- launchers (ds_merge.cu) --------------------------------------------------
struct MergeWs {
  int64_t n;
  const int32_t* cnt;
  uint8_t* core;
  uint32_t* corew;
  int32_t* parent;
  int32_t* bmin;
  int32_t* cmin;
  int32_t* root;
  int32_t* flag;          // flags, then exclusive scan (cluster ids)
  int32_t* partials;      // scan workspace (scan_partials_len ints)
  int32_t* scan_state = nullptr;  // label-scan look-back state in the per-call zero region
  bool scan_zeroed = false;       // scan_state was zeroed by the call's zero-region memset
  int32_t* nclusters;     // device scalar
  unsigned long long* ncore;
  const int32_t* perm = nullptr;  // sorted -> original index (nullptr: identity)
  const int32_t* inv = nullptr;   // original -> sorted index
  unsigned long long* stamps = nullptr;  // Stamp slots (ST_LABELS_DONE), or nullptr
  unsigned int* label_blocks = nullptr;  // finished label_kernel blocks (zeroed per call)
  int32_t* blk_root = nullptr;  // per 32-point block: the root all its core points share
                                // after the diagonal pass, or -1 (single GPU; nullptr: unused)
  unsigned long long* link_tab = nullptr;  // zeroed per call: tile-root pairs already linked
  unsigned int link_mask = 0;              // slots - 1 (a power of two)
  // single-GPU pipeline: the label kernel's last block copies the scalar block into
  // mapped page-locked memory (no device-to-host copy node for it). Labels written
  // straight to page-locked host memory by the kernel were measured slower than the
  // label kernel + a copy-engine copy (27 vs 47 GB/s at C2; tools/zerocopy_bench.cu).
  const unsigned long long* dev_scalars = nullptr;
  unsigned long long* host_scalars = nullptr;
  int scalar_words = 0;
};
int64_t scan_partials_len(int64_t n);
cudaError_t launch_core_init(const MergeWs& w, int64_t min_pts, cudaStream_t s);
// stage 3 over the stage-1 output, walked per row unit of `units` (the eps-tile
// launch's arguments): diagonal tile pairs by tile (their units: diag_range for the
// culled list, the triangle order otherwise), off-diagonal ones by unit. With ci.cnt
// set, the diagonal pass also initialises the core flags and the union-find of its
// tile (core_init's job; the counts must be complete).
cudaError_t launch_union_chunks(const MergeWs& w, const UnitArgs& units, int lane_blocks,
                                const uint2* diag_range, const CoreInit& ci, cudaStream_t s);
cudaError_t launch_union_dense(const MergeWs& w, const uint32_t* bits32, int64_t stride_words,
                               cudaStream_t s);
cudaError_t launch_merge_forests(const MergeWs& w, const int32_t* parents, int R, cudaStream_t s);
cudaError_t launch_finalize(const MergeWs& w, int64_t* labels, cudaStream_t s);
// parent <- union of the forests parent and other, flattened (multi-GPU fold round)
cudaError_t launch_fold_forest(int32_t* parent, const int32_t* other, int64_t n, cudaStream_t s);
cudaError_t launch_counts_i64(const int32_t* cnt, int64_t n, const int32_t* perm, int64_t* out,
                              cudaStream_t s);
cudaError_t launch_export_bits(const uint2* words, unsigned long long words_cap, const uint2* uchunks,
                               const uint4* dir, const unsigned long long* ndir, const int32_t* perm,
                               uint32_t* bits32, int64_t stride_words, cudaStream_t s);
cudaError_t launch_permute_i32(const int32_t* src, int64_t n, const int32_t* perm, int to_original,
                               int32_t* dst, cudaStream_t s);
// ---- spatial order (ds_sort.cu) -----------------------------------------------
size_t sort_temp_bytes(int64_t n);
// culling bounds computed while permuting (lo == nullptr: plain permute)
struct SortBounds {
  float* lo = nullptr;       // T x dpad tile boxes
  float* hi = nullptr;
  float* maxnorm = nullptr;  // T max squared norms
  float* blk = nullptr;      // 32-point block boxes (nullptr: skip)
  unsigned int* super = nullptr;  // super-tile boxes, zeroed (nullptr: skip; d <= 4)
};
cudaError_t launch_spatial_sort(const float* rec, int64_t n, int d, float* rec_sorted,
                                int32_t* perm, int32_t* inv, unsigned long long* keys,
                                unsigned long long* keys_alt, int32_t* idx, void* temp,
                                size_t temp_bytes, unsigned int* bbox, const SortBounds& bnd,
                                unsigned int* bins, cudaStream_t s);
// bins (nullable, 65536 zeroed words): with 16-bit keys a counting sort whose order
// within a key is arbitrary (one GPU); nullptr: the stable radix sort (same order on
// every rank)
constexpr int SORT_BINS = 1 << 16;
// in-place exclusive scan of n int32 (decoupled look-back) whose look-back state of
// scan_zeroed_bytes(n) bytes is zeroed by the caller (the per-call zero region)
cudaError_t launch_scan_zeroed(int32_t* data, int64_t n, void* state, cudaStream_t s);
size_t scan_zeroed_bytes(int64_t n);
cudaError_t launch_bswap_rows(uint32_t* bits32, int64_t n, int64_t stride_words, cudaStream_t s);

// ---- Warshall backend building blocks (ds_closure.cu) -----------------------------
// core_indices of the valid points (ascending) as int32 and int64; flags / partials:
// scan workspace (n ints, scan_partials_len(n) ints); *total = m
cudaError_t launch_core_index(const uint8_t* valid, int64_t n, int32_t* flags, int32_t* partials,
                              int32_t* total, int32_t* ci32, int64_t* ci64, cudaStream_t s);
// adj (m x stride_m native words) = bits (n x stride_n) restricted to rows and columns ci
cudaError_t launch_core_gather(const uint32_t* bits, int64_t stride_n, const int32_t* ci, int64_t m,
                               uint32_t* adj, int64_t stride_m, cudaStream_t s);
// transitive closure of the m x m native bit matrix C in place (dplus: 32 words,
// W: m words of workspace)
cudaError_t launch_closure(uint32_t* C, int64_t m, int64_t stride, uint32_t* dplus, uint32_t* W,
                           cudaStream_t s);

// ---- float64 serial oracle (ds_serial.cu) ---------------------------------------
// dense MSB-first neighbourhood words (n x stride) and int32 counts of the float64
// direct formula (oracle.py:58-79); soa: n x d doubles of workspace
cudaError_t launch_serial_words(const double* coords, int64_t n, int d, double eps_sq,
                                double* soa, uint32_t* bits, int64_t stride, int32_t* cnt,
                                cudaStream_t s);

// ---- materialising ladder (ds_dist.cu) -----------------------------------------
int64_t dist_pitch(int64_t n);  // floats per device matrix row (roundup4(n))
// rows [row0, row0 + rows) of the direct-formula n x n matrix into out (pitch floats)
cudaError_t launch_dist(const float* rec, int64_t n, int d, int64_t row0, int64_t rows,
                        float* out, cudaStream_t s);
// bits (rows x ceil(n/8), packbits layout) and int64 counts of out-of-pitch rows
cudaError_t launch_threshold(const float* dist, int64_t n, int64_t rows, float eps32, uint8_t* bits,
                             int64_t* counts, cudaStream_t s);

// ---- error plumbing (ds_api.cu) -----------------------------------------------
void set_error(const std::string& msg);
void set_capacity(int64_t required, int64_t cap);

}  // namespace ds
