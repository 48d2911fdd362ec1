// Stage 2-3 of the densescan hot path on sm_100a: core flags, primitive-cluster
// merge and canonical labels.
//
// Replaces merge_iterative (pkg/src/densescan/merge.py:133-166) and the
// border rule _attach_borders (merge.py:116-130) plus canonicalize
// (core.py:116-132). merge_iterative's clusters are the connected components
// of the core-core in-range relation (SPEC.md merge contract),
// so the merge is a lock-free union-find over core-core adjacency words:
// atomicCAS hooks the larger root under the smaller one and finds halve the
// path, hence every root is the minimum core index of its component and the
// result is independent of atomic order. Non-core points take the label of
// their lowest-indexed in-range core (atomicMin), exactly the reference tie
// rule. Canonical ids (first appearance, i.e. lowest member index incl.
// borders) come from an atomicMin per root plus an exclusive prefix scan.
//
// All kernels here are HBM/L2 bound: they stream the adjacency words once and
// touch O(n) int32 arrays that stay L2-resident (4n <= 8 MB at C5).
#include <cuda_runtime.h>

#include <atomic>
#include <stdint.h>

#include "ds_internal.cuh"

namespace ds {
namespace {

constexpr int SCAN_T = 1024;
constexpr int SCAN_PER = 4;
constexpr int SCAN_BLK = SCAN_T * SCAN_PER;

__device__ __forceinline__ int find_root(int32_t* parent, int v) {
  volatile int32_t* p = parent;
  int par = p[v];
  if (par != v) {
    int prev = v, next;
    while (par > (next = p[par])) {  // parents only ever point to smaller indices
      p[prev] = next;                // path halving (benign race: next is an ancestor)
      prev = par;
      par = next;
    }
  }
  return par;
}

// Read-only find (roots pass, after every union is done).
__device__ __forceinline__ int find_root_ro(const int32_t* parent, int v) {
  const volatile int32_t* p = parent;
  int par = p[v];
  while (true) {
    const int next = p[par];
    if (next == par) return par;
    par = next;
  }
}

__device__ __forceinline__ void unite(int32_t* parent, int a, int b) {
  int ra = find_root(parent, a);
  int rb = find_root(parent, b);
  while (ra != rb) {
    if (ra < rb) {
      const int t = ra;
      ra = rb;
      rb = t;
    }
    const int old = atomicCAS(&parent[ra], ra, rb);  // hook the larger root
    if (old == ra) return;
    ra = find_root(parent, old);
    rb = find_root(parent, rb);
  }
}

__global__ void core_init_kernel(const int32_t* __restrict__ cnt, int64_t n, int64_t min_pts,
                                 uint8_t* __restrict__ core, uint32_t* __restrict__ corew,
                                 int32_t* __restrict__ parent, int32_t* __restrict__ bmin,
                                 int32_t* __restrict__ cmin, unsigned long long* ncore) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool c = i < n && (int64_t)cnt[i] >= min_pts;  // kernels.py:335
  const uint32_t ballot = __ballot_sync(0xffffffffu, c);
  if (i < n) {
    core[i] = c ? 1 : 0;
    parent[i] = (int32_t)i;
    bmin[i] = NONE;
    cmin[i] = NONE;
  }
  if ((threadIdx.x & 31) == 0) {
    const int64_t w = i >> 5;
    if (w * 32 < n) corew[w] = __brev(ballot);  // bit 31 - t <-> point 32w + t
    if (ballot) atomicAdd(ncore, (unsigned long long)__popc(ballot));
  }
}

// ---- union over adjacency words ---------------------------------------------------
// Loads here are plain (L1-cacheable). An L1 copy of parent[] may be stale, but a
// stale entry is still an ancestor (parents only move toward smaller indices), so
// equal stale roots imply the same set, and every failed CAS returns a strictly
// smaller fresh root: correctness and termination do not depend on coherence.
__device__ __forceinline__ int find_plain(int32_t* parent, int v) {
  int par = parent[v];
  if (par != v) {
    int prev = v, next;
    while (par > (next = parent[par])) {
      parent[prev] = next;  // path halving
      prev = par;
      par = next;
    }
  }
  return par;
}

// Link the set holding root `r` with the set of node j; returns a root of the union.
__device__ __forceinline__ int link_root(int32_t* parent, int r, int j) {
  int rj = find_plain(parent, j);
  while (r != rj) {
    const int hi = r > rj ? r : rj;
    const int lo = r > rj ? rj : r;
    const int old = atomicCAS(&parent[hi], hi, lo);  // hook the larger root
    if (old == hi) return lo;
    r = find_plain(parent, old);
    rj = find_plain(parent, lo);
  }
  return r;
}

// block-wide exclusive scan of one int per thread; also returns the block total
__device__ __forceinline__ int block_exclusive_scan(int v, int& total) {
  __shared__ int warp_sums[32];
  __shared__ int tot;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int s = lane < nw ? warp_sums[lane] : 0;
    int si = s;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, si, off);
      if (lane >= off) si += y;
    }
    if (lane < nw) warp_sums[lane] = si - s;
    if (lane == nw - 1) tot = si;
  }
  __syncthreads();
  total = tot;
  const int excl = warp_sums[wid] + incl - v;
  __syncthreads();  // the shared slots may be reused by the caller's next call
  return excl;
}

// ---- union over tile-pair chunks (two rounds) --------------------------------------
// Round 1, one CTA per diagonal chunk (tile a with itself, words hold j >= i):
//   * every in-range core pair (u < v) proposes u as v's minimum neighbour
//     (shared-memory atomicMin, no CAS);
//   * pointer jumping on that min-neighbour forest (9 halvings cover 512 nodes);
//   * the few pairs whose endpoints still have different roots are merged with a
//     shared-memory union-find (CAS on the larger root);
//   * every core point gets parent = its local root (the smallest index of its
//     local component) — each tile is owned by one CTA, so no global atomics.
// Round 2 (union_links_kernel, below) walks the off-diagonal units of the eps-tile
// launch, one warp per unit.
// A directory entry names one tile pair with words and its range of unit chunks;
// the words of a tile pair are the concatenation of its units' chunks. ItemWords
// holds the prefix sums of the chunk lengths in shared memory so that a CTA can
// walk the tile pair's words as one flat index space (word k lives in the last
// chunk whose prefix is <= k).
// chunk entries per tile pair: up to 32 units (KP = 4 in pieces of 2 column blocks;
// KP = 1: 16 unsplit) x WPR
constexpr int MAX_UPT = 32 * WPR;
static_assert(MAX_UPT <= 512, "union_diag loads one chunk entry per thread");

struct ItemWords {
  uint32_t pre[MAX_UPT + 1];
  unsigned long long base[MAX_UPT];
  int nunits;
  int total;
  int ok;
};

struct DirInfo {
  int a, b;
  unsigned long long ulo;
  int nunits;
};

__device__ __forceinline__ DirInfo decode_dir(uint4 e) {
  DirInfo di;
  di.a = (int)(e.x >> 16);
  di.b = (int)(e.x & 0xffffu);
  di.ulo = (unsigned long long)e.y | ((unsigned long long)e.w << 32);
  di.nunits = (int)e.z;
  return di;
}

// Called by every thread of the CTA (contains __syncthreads).
__device__ void load_item_words(const DirInfo& di, const uint2* __restrict__ uchunks,
                               unsigned long long words_cap, ItemWords& iw) {
  __syncthreads();  // the previous entry's readers are done with iw
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint32_t run = 0;
    bool bad = false;
    for (int c0 = 0; c0 < di.nunits; c0 += 32) {
      const int c = c0 + lane;
      const uint2 e = c < di.nunits ? uchunks[di.ulo + c] : make_uint2(0u, 0u);
      const uint32_t cnt = e.y & 0xffffu;
      const unsigned long long base = (unsigned long long)e.x | ((unsigned long long)(e.y >> 16) << 32);
      bad |= cnt != 0 && base + cnt > words_cap;  // overflowed run: the host re-runs
      uint32_t incl = cnt;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      if (c < di.nunits) {
        iw.pre[c] = run + incl - cnt;
        iw.base[c] = base;
      }
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    const bool any_bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      iw.pre[di.nunits] = run;
      iw.nunits = di.nunits;
      iw.total = (int)run;
      iw.ok = !any_bad;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ uint2 item_word(const ItemWords& iw, const uint2* __restrict__ words,
                                           uint32_t k) {
  int lo = 0, hi = iw.nunits;  // pre[lo] <= k < pre[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (iw.pre[mid] <= k) lo = mid;
    else hi = mid;
  }
  return words[iw.base[lo] + (k - iw.pre[lo])];
}

// read-only find: the only concurrent writes are unite_local's atomicCAS hooks
__device__ __forceinline__ int find_local(const int* lp, int v) {
  int p = lp[v];
  while (p != v) {
    v = p;
    p = lp[v];
  }
  return v;
}

__device__ __forceinline__ void unite_local(int* lp, int u, int v) {
  for (;;) {
    u = find_local(lp, u);
    v = find_local(lp, v);
    if (u == v) return;
    if (u < v) {
      const int t = u;
      u = v;
      v = t;
    }
    if (atomicCAS(&lp[u], u, v) == u) return;  // hook the larger local root
  }
}

__device__ __forceinline__ int orig_of(const int32_t* perm, int g) { return perm ? perm[g] : g; }

// lowest ORIGINAL index among the core points flagged in `bits` of word column jb0
__device__ __forceinline__ int min_orig(const int32_t* perm, int jb0, uint32_t bits) {
  if (!perm) return jb0 + __clz(bits);
  int best = NONE;
  while (bits) {
    const int t = __clz(bits);
    bits &= ~(0x80000000u >> t);
    best = min(best, perm[jb0 + t]);
  }
  return best;
}

// Round 1. THREADS = 512: thread (w, c) owns column word w and row block c.
// Row stride of union_diag's dense adjacency R (word column ww, row u at ww * DIAG_RS + u):
// one word of padding puts the 16 word columns of a row in different banks, so the
// row-block scans (thread = word column x row block) are conflict-free (a stride of
// TILE made them 16-way conflicts)
constexpr int DIAG_RS = TILE + 1;

__global__ void __launch_bounds__(512, 4) union_diag_kernel(
    const UnitArgs A, int LB, const uint2* __restrict__ diag_range, const CoreInit ci,
    const uint32_t* __restrict__ corew_in, int32_t* parent, int32_t* bmin,
    const int32_t* __restrict__ perm, int32_t* __restrict__ blk_root) {
  griddep_wait();
  stamp(A.stamps, ST_MERGE);  // stage 1+2 complete
  constexpr int THREADS = 512;
  constexpr int RB = TILE / (THREADS / WPR);  // rows per block: 16
  extern __shared__ uint32_t dsm[];
  uint32_t* R = dsm;                         // [WPR][DIAG_RS] core-masked adjacency words
  uint32_t* M = R + WPR * DIAG_RS;           // [THREADS / WPR][WPR] row-block column masks
  int* lp = reinterpret_cast<int*>(M + THREADS);
  int* lb = lp + TILE;
  int* hist = lb + TILE;
  __shared__ uint32_t lcw[WPR];
  __shared__ uint32_t adj[32];
  __shared__ int wroots[WPR], wpre[WPR], slot_root[32];
  __shared__ int ntrees_sh;
  __shared__ int epre[MAX_UPT + 1];                  // chunk-entry prefix of the word counts
  __shared__ unsigned long long ebase_sh[MAX_UPT];   // chunk-entry first word
  const int tid = threadIdx.x;
  const int w = tid % WPR, cblk = tid / WPR;
  const int64_t n = A.n;
  const int64_t ntiles = A.T;
  const int64_t nw = (n + 31) / 32;
  const uint2* __restrict__ uchunks = A.uchunks;
  const uint2* __restrict__ words = A.words;
  const unsigned long long words_cap = A.words_cap;
  long long r_lo, r_hi;
  unit_range(A, r_lo, r_hi);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int base = (int)tile * TILE;
    if (ci.cnt) {  // core_init for the tile's points (kernels.py:335); one word per warp
      const int64_t i = base + tid;
      const bool c = i < n && (int64_t)ci.cnt[i] >= ci.min_pts;
      const uint32_t ballot = __ballot_sync(0xffffffffu, c);
      if (i < n) {
        ci.core[i] = c ? 1 : 0;
        parent[i] = (int32_t)i;
        bmin[i] = NONE;
        ci.cmin[i] = NONE;
      }
      if ((tid & 31) == 0) {
        const int64_t gw = (int64_t)tile * WPR + (tid >> 5);
        if (gw < nw) ci.corew[gw] = __brev(ballot);  // bit 31 - t <-> point 32w + t
        lcw[tid >> 5] = __brev(ballot);
        if (ballot) atomicAdd(ci.ncore, (unsigned long long)__popc(ballot));
      }
    } else if (tid < WPR) {
      const int64_t gw = (int64_t)tile * WPR + tid;
      lcw[tid] = gw < nw ? corew_in[gw] : 0u;
    }
    // the diagonal pair's chunk entries: its units (culled list: diag_range; dense: the
    // triangle order, clipped to this launch's shard) own entries [u * WPR, ...)
    long long u_lo = 0, u_hi = 0;
    if (A.unit_list) {
      const uint2 dr = diag_range[tile];
      u_lo = (long long)dr.x | ((long long)(dr.y >> 16) << 32);
      u_hi = u_lo + (long long)(dr.y & 0xffffu);
      if (u_hi > r_hi) u_hi = r_hi;  // list overflow: the host re-runs
    } else {
      const long long q = row_offset(tile, ntiles);
      u_lo = q * LB > r_lo ? q * LB : r_lo;
      u_hi = (q + 1) * LB < r_hi ? (q + 1) * LB : r_hi;
    }
    if (u_lo >= u_hi) {  // no words on this launch: only the core init (uniform per CTA)
      if (blk_root && (tid & 31) == 0 && (int64_t)tile * WPR + (tid >> 5) < nw)
        blk_root[(int64_t)tile * WPR + (tid >> 5)] = -1;
      __syncthreads();
      continue;
    }
    const long long e_lo = u_lo * WPR;
    const int nentries = (int)((u_hi - u_lo) * WPR);
    // the pair's chunk entries (nentries <= MAX_UPT <= THREADS), loaded before the
    // shared-memory setup so that their latency overlaps it
    uint32_t ecnt = 0;
    unsigned long long ebase = 0;
    if (tid < nentries) {
      const uint2 ce = uchunks[e_lo + tid];
      ecnt = ce.y & 0xffffu;
      ebase = (unsigned long long)ce.x | ((unsigned long long)(ce.y >> 16) << 32);
      if (ebase + ecnt > words_cap) ecnt = 0;  // overflowed run: the host re-runs
    }
    for (int k = tid; k < WPR * DIAG_RS; k += THREADS) R[k] = 0u;
    for (int v = tid; v < TILE; v += THREADS) {
      lp[v] = v;
      lb[v] = NONE;
      hist[v] = 0;
    }
    if (tid == 0) slot_root[0] = -1;  // atomicMax target of the single-root fast path
    __syncthreads();
    auto scatter = [&](const uint2 rec) {
      const int u = (int)(rec.y >> 4);
      const int ww = (int)(rec.y & 15u);
      const uint32_t cw = lcw[ww];
      if ((lcw[u >> 5] >> (31 - (u & 31))) & 1u) {
        R[ww * DIAG_RS + u] = rec.x & cw;
        uint32_t bm = rec.x & ~cw;  // core u in range of non-core v (merge.py:116-130)
        if (bm) {
          const int gu = orig_of(perm, base + u);
          while (bm) {
            const int t = __clz(bm);
            bm &= ~(0x80000000u >> t);
            atomicMin(&lb[ww * 32 + t], gu);
          }
        }
      } else {
        const uint32_t cm = rec.x & cw;
        if (cm) atomicMin(&lb[u], min_orig(perm, base + ww * 32, cm));
      }
    };
    // scatter the tile pair's words into the dense matrix (core rows, core columns
    // only); non-core rows give their own border candidate directly. The pair's words
    // are one flat index space over its chunk entries (a block scan of the entry
    // counts): every thread loads 4 words at a time from independent addresses, so the
    // whole tile pair costs about two L2 round trips instead of one per entry.
    {
      int total;
      const int pre = block_exclusive_scan((int)ecnt, total);
      if (tid < nentries) {
        epre[tid] = pre;
        ebase_sh[tid] = ebase;
      }
      __syncthreads();
      auto locate = [&](int j) -> unsigned long long {  // word j of the pair -> address
        int lo = 0, hi = nentries;  // epre[lo] <= j < epre[hi], epre[nentries] taken as total
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (epre[mid] <= j) lo = mid;
          else hi = mid;
        }
        return ebase_sh[lo] + (unsigned long long)(j - epre[lo]);
      };
      for (int j0 = tid; j0 < total; j0 += 4 * THREADS) {
        uint2 rec[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = j0 + q * THREADS;
          rec[q] = j < total ? words[locate(j)] : make_uint2(0u, 0u);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (j0 + q * THREADS < total) scatter(rec[q]);
      }
    }
    __syncthreads();
    // minimum neighbour of every core column = first row (ascending) holding it (the
    // self bit makes it exist): OR per row block, then warp w takes word column w, lane
    // l column 32 w + l — the first row block whose OR has the column (broadcast reads),
    // then the first row of that block. No atomics, about 32 shared loads per lane
    // (a per-bit atomicMin loop over the fresh bits of every row was 10 us of the
    // kernel at C2).
    uint32_t acc = 0;
    for (int r = 0; r < RB; ++r) acc |= R[w * DIAG_RS + cblk * RB + r];
    M[cblk * WPR + w] = acc;
    __syncthreads();
    static_assert(THREADS / 32 == WPR, "one warp per word column");
    {
      const int ww = tid >> 5, l = tid & 31;
      const uint32_t bit = 0x80000000u >> l;
      int q0 = -1;
#pragma unroll
      for (int q = 0; q < THREADS / WPR; ++q)
        if (q0 < 0 && (M[q * WPR + ww] & bit)) q0 = q;
      if (q0 >= 0) {
        const uint32_t* col = R + ww * DIAG_RS + q0 * RB;
        int r = 0;
        while (r < RB - 1 && !(col[r] & bit)) ++r;
        lp[ww * 32 + l] = q0 * RB + r;
      }
    }
    __syncthreads();
    // Fast path: a core point without a smaller core neighbour is a local minimum. If
    // the tile has at most one, every core point reaches it by following smaller
    // neighbours, so the tile is one component rooted there (the common dense case):
    // no pointer jumping, no tree merge.
    {
      const bool core0 = (lcw[tid >> 5] >> (31 - (tid & 31))) & 1u;
      const bool root0 = core0 && lp[tid] == tid;
      const uint32_t rb0 = __ballot_sync(0xffffffffu, root0);
      if ((tid & 31) == 0) wroots[tid >> 5] = __popc(rb0);
      if (root0) atomicMax(&slot_root[0], tid);  // read only when it is the single root
      __syncthreads();
      int nroots = 0;
#pragma unroll
      for (int q = 0; q < THREADS / 32; ++q) nroots += wroots[q];
      if (nroots <= 1) {  // uniform per CTA
        if (blk_root) {  // every core point of the tile has the root slot_root[0]
          const uint32_t cores = __ballot_sync(0xffffffffu, core0 && (int64_t)base + tid < n);
          const int64_t gw = (int64_t)tile * WPR + (tid >> 5);
          if ((tid & 31) == 0 && gw < nw) blk_root[gw] = cores ? base + slot_root[0] : -1;
        }
        const int64_t g = (int64_t)base + tid;
        if (g < n) {
          if (nroots == 1 && core0 && tid != slot_root[0]) parent[g] = base + slot_root[0];
          if (lb[tid] != NONE) atomicMin(&bmin[g], lb[tid]);
        }
        __syncthreads();  // smem is reused by the next tile
        continue;
      }
      __syncthreads();  // wroots / slot_root are rewritten below
    }
    // synchronous pointer jumping over the min-neighbour forest (every node reads its
    // grandparent, barrier, writes it) until no pointer moves: 9 rounds cover 512 nodes
#pragma unroll 1
    for (int r = 0; r < TILE; ++r) {
      const int cur = lp[tid];
      const int nv = lp[cur];
      __syncthreads();
      if (nv != cur) lp[tid] = nv;
      if (!__syncthreads_or(nv != cur)) break;
    }
    // merge the min-neighbour trees. Roots get slots in index order; with <= 32
    // trees every word ANDs its row's complement mask against the tree masks to
    // find crossing trees, and a 32 x 32 boolean closure (one warp) merges them —
    // no per-bit work. More trees (sparse tiles, few bits) use a shared-memory
    // union-find over the crossing bits.
    const bool is_core = (lcw[tid >> 5] >> (31 - (tid & 31))) & 1u;
    const bool is_root = is_core && lp[tid] == tid;
    const uint32_t rball = __ballot_sync(0xffffffffu, is_root);
    if ((tid & 31) == 0) wroots[tid >> 5] = __popc(rball);
    for (int k = tid; k < 32 * WPR; k += THREADS) M[k] = 0u;  // M becomes T[32][WPR]
    if (tid < 32) adj[tid] = 0u;
    __syncthreads();
    if (tid < 32) {  // exclusive prefix of roots per warp -> slots in index order
      const int cnt = tid < WPR ? wroots[tid] : 0;
      int incl = cnt;
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (tid >= off) incl += y;
      }
      if (tid < WPR) wpre[tid] = incl - cnt;
      if (tid == 31) ntrees_sh = incl;
    }
    __syncthreads();
    const int ntrees = ntrees_sh;
    if (is_root) {
      const int k = wpre[tid >> 5] + __popc(rball & ((1u << (tid & 31)) - 1u));
      hist[tid] = k;                     // root node -> slot
      if (k < 32) slot_root[k] = tid;    // slot -> root node
    }
    __syncthreads();
    if (ntrees <= 32) {
      {  // tree masks: one store per (tree, warp) group instead of 32-way smem atomics
        const int key = is_core ? hist[lp[tid]] : -1;
        const uint32_t grp = __match_any_sync(0xffffffffu, key);
        if (is_core && (tid & 31) == __ffs(grp) - 1) M[key * WPR + (tid >> 5)] = __brev(grp);
        __syncthreads();
        hist[tid] = key;  // hist becomes node -> tree slot (one load less per lookup)
      }
      __syncthreads();
#pragma unroll 4
      for (int r = 0; r < RB; ++r) {
        const int u = cblk * RB + r;
        const uint32_t um = R[w * DIAG_RS + u];  // zero for non-core rows
        const int k = hist[u];
        if (!um) continue;
        const uint32_t cross = um & ~M[k * WPR + w];
        if (!cross) continue;
        // the trees the word crosses into: per iteration the tree of its lowest remaining
        // bit, whose columns are then removed (iterations = distinct crossed trees, not
        // ntrees)
        uint32_t bits = 0, rest = cross;
        while (rest) {
          const int j = hist[w * 32 + __clz(rest)];
          bits |= 1u << j;
          rest &= ~M[j * WPR + w];
        }
        atomicOr(&adj[k], bits);
      }
      __syncthreads();
      if (tid < 32) {  // symmetric transitive closure of the tree graph (one warp)
        uint32_t row = adj[tid] | (1u << tid);
        uint32_t col = 0;
        for (int j = 0; j < ntrees; ++j)  // lanes >= ntrees hold only their self bit
          if ((__shfl_sync(0xffffffffu, row, j) >> tid) & 1u) col |= 1u << j;
        row |= col;
        for (int p = 0; p < ntrees; ++p) {
          const uint32_t rp = __shfl_sync(0xffffffffu, row, p);
          if ((row >> p) & 1u) row |= rp;
        }
        adj[tid] = row;
      }
      __syncthreads();
      if (is_core) {  // lowest slot of the merged component = its smallest root
        const int kmin = __ffs(adj[hist[tid]]) - 1;
        lp[tid] = slot_root[kmin];
      }
    } else {
      for (int r = 0; r < RB; ++r) {
        const int u = cblk * RB + r;
        uint32_t um = R[w * DIAG_RS + u];
        const int ru = lp[u];
        while (um) {
          const int t = __clz(um);
          um &= ~(0x80000000u >> t);
          const int v = w * 32 + t;
          if (lp[v] != ru) unite_local(lp, u, v);
        }
      }
    }
    __syncthreads();
    {
      const int v = tid;
      const int64_t g = (int64_t)base + v;
      int r = -1;
      if (g < n) {
        r = find_local(lp, v);
        if (r != v) parent[g] = base + r;  // r < v: parent[x] <= x holds
        if (lb[v] != NONE) atomicMin(&bmin[g], lb[v]);
      }
      if (blk_root) {  // the 32-point block's common root, if all its core points share one
        const bool cv = g < n && ((lcw[tid >> 5] >> (31 - (tid & 31))) & 1u);
        const uint32_t cores = __ballot_sync(0xffffffffu, cv);
        const uint32_t grp = __match_any_sync(0xffffffffu, cv ? r : -1);
        const int first = cores ? __ffs(cores) - 1 : 0;
        const uint32_t grp0 = __shfl_sync(0xffffffffu, grp, first);
        const int r0 = __shfl_sync(0xffffffffu, r, first);
        const int64_t gw = (int64_t)tile * WPR + (tid >> 5);
        if ((tid & 31) == 0 && gw < nw)
          blk_root[gw] = (cores && (cores & ~grp0) == 0u) ? base + r0 : -1;
      }
    }
    __syncthreads();
  }
}

// Round 2, off-diagonal tile pairs, one warp per row unit of the eps-tile launch
// (lane block lb of tile a x the column blocks of tile b it evaluated). After round
// 1 every core point's parent is its tile-local root. Per unit the warp stages the
// parents and core flags of its 32*KP rows in shared memory and groups the rows of
// each 32-row chunk by root (match_any: a group is named by its first lane); per
// non-empty column block it stages that block's 32 parents and groups the columns the
// same way. Then per word (row u, column block jw, 32 bits), all of a column block's
// words loaded at once:
//   * core u, core columns: the column groups the word touches are OR-ed into the
//     row group's pair mask (shared memory) — after the block, one link per (row
//     group, column group) pair that has a bit, made by the lanes in parallel, instead
//     of a serial chain of per-bit links on one lane (the tail of this kernel);
//   * core u, non-core columns: border candidates, atomicMin of u's ORIGINAL index;
//   * non-core u with core columns: u's border candidate, the lowest ORIGINAL index
//     among those columns (merge.py:116-130).
// Links go through the global lock-free union-find (link_root: CAS hooks the larger
// root under the smaller), so the result does not depend on the order.
constexpr int LINK_WARPS = 8;
#ifndef DS_LINK_MINB
#define DS_LINK_MINB 4
#endif
__global__ void __launch_bounds__(LINK_WARPS * 32, DS_LINK_MINB) union_links_kernel(
    const UnitArgs A, int LB, const uint32_t* __restrict__ corew, int32_t* parent, int32_t* bmin,
    const int32_t* __restrict__ perm, const int32_t* __restrict__ blk_root,
    unsigned long long* link_tab, unsigned int link_mask) {
  griddep_wait();
  constexpr int MAXR = TILE / WPR * 4;  // up to 128 rows per lane block
  __shared__ int rows_sh[LINK_WARPS][MAXR];
  __shared__ int cols_sh[LINK_WARPS][32];
  __shared__ uint8_t rlead_sh[LINK_WARPS][MAXR];     // row -> its group's first row
  __shared__ uint8_t clead_sh[LINK_WARPS][32];       // column -> its group's first column
  __shared__ uint32_t cmask_sh[LINK_WARPS][32];      // group (first column) -> its columns
  __shared__ uint32_t pairs_sh[LINK_WARPS][MAXR];    // row group -> column groups linked
  // links of the current unit, made together at its end (lanes in parallel) instead of
  // per column block: each link is a chain of dependent parent loads + CAS, and made
  // per column block those chains were serial in the unit's column blocks
  constexpr int LKCAP = 64;
  __shared__ int2 lk_sh[LINK_WARPS][LKCAP];
  __shared__ int lkn_sh[LINK_WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* rows = rows_sh[warp];
  int* cols = cols_sh[warp];
  uint8_t* rlead = rlead_sh[warp];
  uint8_t* clead = clead_sh[warp];
  uint32_t* cmask = cmask_sh[warp];
  uint32_t* pairs = pairs_sh[warp];
  for (int k = lane; k < MAXR; k += 32) pairs[k] = 0u;
  int2* lk = lk_sh[warp];
  int* lkn = &lkn_sh[warp];
  if (lane == 0) *lkn = 0;
  __syncwarp();
  auto defer_link = [&](int au, int av) {  // overflow: link now
    const int at = atomicAdd(lkn, 1);
    if (at < LKCAP) lk[at] = make_int2(au, av);
    else link_root(parent, find_plain(parent, au), av);
  };
  const int n = (int)A.n;
  const int KPL = TILE / LB;  // rows per lane block (32 * KP)
  long long r_lo, r_hi;
  unit_range(A, r_lo, r_hi);
  const long long nw = (long long)gridDim.x * LINK_WARPS;
  int last_a = -1, last_b = -1;  // this lane's last linked pair of roots
  // the uniform-tile shortcut (below) pays when warps walk several units each (it
  // saves per-unit load latency); with about one unit per warp (small inputs, e.g.
  // C1) its burst of simultaneous links is slower than the full path
  const bool uniform_ok = blk_root && (r_hi - r_lo) > 2 * nw;
  // loads are issued a step ahead where the data does not depend on them: the next
  // unit's list entry and chunk entries during the current unit, and per column block
  // the core word, the 32 parents and the first 32 words together
  auto unit_entry = [&](long long u, int& a, int& b, int& lb) {
    if (A.unit_list) {
      const uint2 e = __ldg(A.unit_list + u);
      a = (int)(e.x >> 16);
      b = (int)(e.x & 0xffffu);
      lb = (int)((e.y >> 16) & 0xfu);
    } else {
      decode_item(u / LB, A.T, a, b);
      lb = (int)(u % LB);
    }
  };
  long long u = r_lo + (long long)blockIdx.x * LINK_WARPS + warp;
  int na = 0, nb = 0, nlb = 0;
  uint2 nce = make_uint2(0u, 0u);
  if (u < r_hi) {
    unit_entry(u, na, nb, nlb);
    if (lane < WPR) nce = A.uchunks[u * WPR + lane];
  }
  for (; u < r_hi; u += nw) {
    const int a = na, b = nb, lb = nlb;
    const uint2 ce = nce;
    if (u + nw < r_hi) {  // prefetch the next unit
      unit_entry(u + nw, na, nb, nlb);
      nce = lane < WPR ? A.uchunks[(u + nw) * WPR + lane] : make_uint2(0u, 0u);
    }
    if (a == b) continue;  // round 1
    const uint32_t cnt = ce.y & 0xffffu;
    const unsigned long long base = (unsigned long long)ce.x | ((unsigned long long)(ce.y >> 16) << 32);
    const bool ok = cnt != 0u && base + cnt <= A.words_cap;  // overflowed run: the host re-runs
    uint32_t todo = __ballot_sync(0xffffffffu, ok);
    if (!todo) continue;
    // the rows' parents and core words, issued together with the uniform test's loads
    // (one round trip instead of one per 32-row chunk after it)
    const int r0 = a * TILE + lb * KPL;  // a multiple of 32
    int pgs[MAXR / 32];
    uint32_t cws[MAXR / 32];
#pragma unroll
    for (int i = 0; i < MAXR / 32; ++i) {
      const bool chunk = 32 * i < KPL && r0 + 32 * i < n;  // warp-uniform
      pgs[i] = chunk && r0 + 32 * i + lane < n ? parent[r0 + 32 * i + lane] : -1;
      cws[i] = chunk ? corew[(r0 >> 5) + i] : 0u;
    }
    auto load_cb = [&](int jw, uint2 (&rw)[4], int& pr, uint32_t& cwv, uint32_t& wc) {
      wc = __shfl_sync(0xffffffffu, cnt, jw);  // <= 32*KP <= 128 words
      const unsigned long long wbase = __shfl_sync(0xffffffffu, base, jw);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        rw[q] = lane + 32u * q < wc ? A.words[wbase + lane + 32u * q] : make_uint2(0u, 0u);
      const int c = b * TILE + jw * 32 + lane;
      pr = c < n ? parent[c] : -1;
      cwv = corew[(b * TILE >> 5) + jw];
    };
    // Uniform blocks (union_diag: all core points of a 32-point block share one root):
    // when the lane block's row blocks share one root, every column block has a root,
    // and every row and column is core, every word is a core-core word and no border
    // candidates exist — the unit is exactly the links of the row root with the column
    // roots, made without reading parents or words.
    if (uniform_ok) {
      // core words and block roots of the row blocks (lanes 0..) and of the column
      // blocks (lanes 16 + jw), loaded together: one round trip
      const int rw = (a * TILE + lb * KPL) >> 5;  // first row block
      const bool rl = lane < KPL / 32 && (rw + lane) * 32 < n;
      const bool cl = lane >= 32 - WPR && ((todo >> (lane - (32 - WPR))) & 1u);
      const int gw = rl ? rw + lane : (cl ? ((b * TILE) >> 5) + lane - (32 - WPR) : -1);
      uint32_t w = 0u, vm = 0u;
      int br = -1;
      if (gw >= 0) {
        const int g0 = gw * 32;
        w = corew[gw];
        br = blk_root[gw];
        vm = n - g0 >= 32 ? 0xffffffffu : ~(0xffffffffu >> (n - g0));
      }
      const int urow = __shfl_sync(0xffffffffu, br, 0);  // lane 0 holds a row block
      if (__all_sync(0xffffffffu, w == vm && (!rl || br == urow) && (!cl || br >= 0)) && urow >= 0) {
        // one link per distinct column root; many units of a block pair arrive here at
        // once: the first to claim the pair's slot links it, the rest skip (a slot
        // taken by another pair: link anyway)
        const unsigned grp = __match_any_sync(0xffffffffu, cl ? br : -1);
        if (cl && lane == __ffs(grp) - 1 && br != urow && !(urow == last_a && br == last_b)) {
          const unsigned long long key = ((unsigned long long)(unsigned)urow << 32 | (unsigned)br) + 1ull;
          const unsigned slot = (unsigned)((key * 0x9E3779B97F4A7C15ull) >> 40) & link_mask;
          unsigned long long old = link_tab[slot];
          if (old == 0ull) old = atomicCAS(&link_tab[slot], 0ull, key);
          if (old != key) link_root(parent, find_plain(parent, urow), br);
          last_a = urow;
          last_b = br;
        }
        continue;
      }
    }
    // rows of the lane block: parent (= local root, or an ancestor of it) or -1 (not
    // core), grouped by root per 32-row chunk
    // the first column block's loads overlap the row grouping (issued after the uniform
    // test: uniform units, most of a dense region's, never read words)
    int jw = __ffs(todo) - 1;
    todo &= todo - 1u;
    uint2 rec[4];
    int praw;
    uint32_t cw, wcnt;
    load_cb(jw, rec, praw, cw, wcnt);
    int rfirst = -1;  // this lane's first core row root
    bool rsame = true;  // all of this lane's core rows share it
    bool rnoncore = false;  // this lane has a non-core row
#pragma unroll
    for (int i = 0; i < MAXR / 32; ++i) {
      if (32 * i >= KPL) break;  // KPL is a multiple of 32: warp-uniform
      const int k = lane + 32 * i;
      const int g = r0 + k;
      const int pg = pgs[i];
      const bool c = g < n && ((cws[i] >> (31 - lane)) & 1u);
      const int v = c ? pg : -1;
      rows[k] = v;
      const unsigned grp = __match_any_sync(0xffffffffu, v);
      rlead[k] = (uint8_t)((k & ~31) + __ffs(grp) - 1);
      rnoncore |= g < n && !c;
      if (c) {
        if (rfirst < 0) rfirst = pg;
        else rsame &= pg == rfirst;
      }
    }
    const bool rows_allcore = !__any_sync(0xffffffffu, rnoncore);
    // urow: the single root of all core rows of the lane block (the common case inside
    // a cluster), -1 if they differ or there are none
    int urow = -1;
    {
      const unsigned has = __ballot_sync(0xffffffffu, rfirst >= 0);
      if (has) {
        const int r = __shfl_sync(0xffffffffu, rfirst, __ffs(has) - 1);
        if (__all_sync(0xffffffffu, rsame && (rfirst < 0 || rfirst == r))) urow = r;
      }
    }
    for (bool first_cb = true;; first_cb = false) {  // column blocks of the unit
      if (!first_cb) {
        if (!todo) break;
        jw = __ffs(todo) - 1;
        todo &= todo - 1u;
        load_cb(jw, rec, praw, cw, wcnt);
      }
      const int c0 = b * TILE + jw * 32;
      const bool cc = (cw >> (31 - lane)) & 1u;
      const int pv = cc ? praw : -1;
      cols[lane] = pv;
      const unsigned same = __match_any_sync(0xffffffffu, pv);
      const int lead = __ffs(same) - 1;
      clead[31 - lane] = (uint8_t)lead;  // indexed by bit position (bit 31 - l <-> lane l)
      if (lane == lead) cmask[lane] = __brev(same);
      const unsigned corel = __brev(cw);  // bit l <-> lane l
      // uniform: every core lane in one match group
      const int first = corel ? __ffs(corel) - 1 : 0;
      const unsigned grp0 = __shfl_sync(0xffffffffu, same, first);
      const int ub = (corel && (corel & ~grp0) == 0u) ? __shfl_sync(0xffffffffu, pv, first) : -1;
      __syncwarp();
      // uniform rows x uniform columns: the whole column block is at most one link
      // (urow, ub), made once by lane 0 if any core-core bit is set
      const bool one_link = urow >= 0 && ub >= 0;
      bool cc_any = false;
      // all rows and all (valid) columns core: every word is a core-core word and no
      // border candidates exist, so the block is exactly the link — its words need not
      // be read
      const int nvalid = n - c0 < 32 ? n - c0 : 32;
      const uint32_t vmask = nvalid >= 32 ? 0xffffffffu : ~(0xffffffffu >> nvalid);
      const bool skip_words = one_link && rows_allcore && cw == vmask;
      if (skip_words) cc_any = wcnt > 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (skip_words || lane + 32u * q >= wcnt) continue;
        const uint32_t x = rec[q].x;
        const int ul = (int)(rec[q].y >> 4);
        const int kr = ul - lb * KPL;
        const uint32_t cm = x & cw;
        if (rows[kr] >= 0) {
          if (cm) {
            if (one_link) {
              cc_any = true;
            } else {  // the column groups this word touches
              uint32_t bits = cm, m = 0u;
              while (bits) {
                const int g = clead[__clz(bits) ^ 31];
                m |= 1u << g;
                bits &= ~cmask[g];
              }
              atomicOr(&pairs[rlead[kr]], m);
            }
          }
          uint32_t bm = x & ~cw;
          if (bm) {
            const int gu = orig_of(perm, a * TILE + ul);
            while (bm) {
              const int t = __clz(bm);
              bm &= ~(0x80000000u >> t);
              atomicMin(&bmin[c0 + t], gu);
            }
          }
        } else if (cm) {
          atomicMin(&bmin[a * TILE + ul], min_orig(perm, c0, cm));
        }
      }
      if (one_link) {
        if (__any_sync(0xffffffffu, cc_any) && lane == 0 && urow != ub &&
            !(urow == last_a && ub == last_b)) {
          defer_link(urow, ub);
          last_a = urow;
          last_b = ub;
        }
      } else {
        __syncwarp();
        // one link per (row group, column group) pair with a bit; lane l takes the
        // row groups led by rows l, l + 32, ...
        for (int k = lane; k < KPL; k += 32) {
          uint32_t m = pairs[k];
          if (!m) continue;
          pairs[k] = 0u;
          const int au = rows[k];
          while (m) {
            const int g = __ffs(m) - 1;
            m &= m - 1u;
            const int av = cols[g];
            if (av != au && !(au == last_a && av == last_b)) {
              defer_link(au, av);
              last_a = au;
              last_b = av;
            }
          }
        }
      }
      __syncwarp();  // cols / groups / pair masks are rewritten by the next column block
    }
    const int nl = min(*lkn, LKCAP);
    for (int i = lane; i < nl; i += 32) link_root(parent, find_plain(parent, lk[i].x), lk[i].y);
    __syncwarp();
    if (lane == 0) *lkn = 0;
    __syncwarp();
  }
}

// Dense rows (reference NeighborhoodMatrix converted to native words): one warp per row.
__global__ void union_dense_kernel(const uint32_t* __restrict__ bits32, int64_t stride_words,
                                   int64_t n, const uint8_t* __restrict__ core,
                                   const uint32_t* __restrict__ corew, int32_t* parent,
                                   int32_t* bmin) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (n + 31) / 32;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint32_t* row = bits32 + i * stride_words;
    const bool ci = core[i] != 0;
    int best = NONE;
    for (int64_t k = lane; k < nw; k += 32) {
      const uint32_t m = row[k] & corew[k];
      if (!m) continue;
      if (ci) {
        uint32_t um = m;
        while (um) {
          const int t = __clz(um);
          um &= ~(0x80000000u >> t);
          unite(parent, (int)i, (int)(k * 32 + t));
        }
      } else if (best == NONE) {
        best = (int)(k * 32 + __clz(m));
      }
    }
    if (!ci) {
#pragma unroll
      for (int off = 16; off; off >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, off));
      if (lane == 0 && best != NONE) bmin[i] = best;
    }
  }
}

// Runs over sorted indices s; bmin holds ORIGINAL indices of cores, cmin collects
// the lowest ORIGINAL member index of each root (borders included).
__global__ void roots_kernel(const uint8_t* __restrict__ core, const int32_t* __restrict__ parent,
                             const int32_t* __restrict__ bmin, int64_t n,
                             const int32_t* __restrict__ perm, const int32_t* __restrict__ inv,
                             int32_t* __restrict__ root, int32_t* cmin, int32_t* cid) {
  griddep_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int r = -1, o = NONE;
  if (i < n) {
    cid[i] = -1;  // cluster ids (indexed by root), written by scan_label_kernel
    if (core[i]) {
      r = find_root_ro(parent, (int)i);
    } else {
      const int b = bmin[i];
      if (b != NONE) r = find_root_ro(parent, inv ? inv[b] : b);
    }
    root[i] = r;
    o = perm ? perm[i] : (int)i;
  }
  // first appearance: one atomicMin per distinct root of the warp (spatially sorted
  // neighbours mostly share a cluster, so this removes the same-address contention)
  const unsigned grp = __match_any_sync(0xffffffffu, r);
  const int m = (int)__reduce_min_sync(grp, (unsigned)o);  // o >= 0
  if (r >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicMin(&cmin[r], m);
}

// Single-pass exclusive scan (decoupled look-back): tiles of SCAN_BLK elements are
// taken in ticket order; each tile publishes its aggregate, then warp 0 reads the
// predecessors' published {flag, value} words 32 at a time until it meets an
// inclusive prefix, and publishes its own. state[] and the ticket are zeroed before
// the launch.
constexpr unsigned long long SC_AGG = 1ull << 62, SC_PRE = 2ull << 62;

// scan input: the array itself
struct ScanInPlace {
  const int32_t* data;
  __device__ __forceinline__ int operator()(int64_t i) const { return data[i]; }
};
template <class In>
__global__ void __launch_bounds__(SCAN_T) scan_lookback_kernel(In in, int32_t* data, int64_t n,
                                                               unsigned int* ticket,
                                                               unsigned long long* state,
                                                               int32_t* total) {
  griddep_wait();
  __shared__ unsigned int tile_sh;
  __shared__ int prefix_sh;
  if (threadIdx.x == 0) tile_sh = atomicAdd(ticket, 1u);
  __syncthreads();
  const unsigned int tile = tile_sh;
  const int64_t base = (int64_t)tile * SCAN_BLK + (int64_t)threadIdx.x * SCAN_PER;
  int v[SCAN_PER];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    v[k] = base + k < n ? in(base + k) : 0;
    sum += v[k];
  }
  int agg;
  const int excl = block_exclusive_scan(sum, agg);
  if (threadIdx.x < 32) {  // warp 0: publish the aggregate, look back 32 tiles at a time
    const int lane = threadIdx.x;
    volatile unsigned long long* st = state;
    int prefix = 0;
    if (tile == 0) {
      if (lane == 0) st[0] = SC_PRE | (unsigned int)agg;
    } else {
      if (lane == 0) st[tile] = SC_AGG | (unsigned int)agg;
      int64_t hi = (int64_t)tile - 1;  // predecessors hi, hi-1, ... still to add
      for (;;) {
        const int64_t j = hi - lane;
        const unsigned long long w = j >= 0 ? st[j] : (2ull << 62);  // before tile 0: prefix 0
        const unsigned flag = (unsigned)(w >> 62);
        const unsigned pre = __ballot_sync(0xffffffffu, flag == 2u);
        const int stop = pre ? __ffs(pre) - 1 : 31;  // nearest inclusive prefix in reach
        const unsigned need = stop == 31 ? 0xffffffffu : ((2u << stop) - 1u);
        if (__ballot_sync(0xffffffffu, flag == 0u) & need) continue;  // not published yet
        int v = lane <= stop ? (int)(unsigned int)w : 0;
#pragma unroll
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        prefix += v;
        if (pre) break;
        hi -= 32;
      }
      if (lane == 0) {
        __threadfence();
        st[tile] = SC_PRE | (unsigned int)(prefix + agg);
      }
    }
    if (lane == 0) {
      prefix_sh = prefix;
      if ((int64_t)(tile + 1) * SCAN_BLK >= n) *total = prefix + agg;  // last tile
    }
  }
  __syncthreads();
  int run = prefix_sh + excl;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    if (base + k < n) data[base + k] = run;
    run += v[k];
  }
}

// Canonical labels in one pass over ORIGINAL indices o (decoupled look-back, tiles in
// ticket order): flag(o) = 1 iff o is the first appearance (lowest original member) of
// its cluster; the exclusive scan of the flags at o is that cluster's id. Each tile,
// once its prefix is known, publishes the ids of the clusters that first appear in it
// (cid[root]); then every o reads cid[root(o)]. A cluster's first appearance is never
// after any of its members (cmin <= o), so it is in this tile or an earlier one — an
// earlier tile got its ticket first and publishes its ids right after its own
// look-back, so the wait below is short and cannot deadlock. Labels are written in
// original order. Replaces scan_lookback + label_kernel. With host_scalars set, the
// last block to finish copies the scalar block there.
__global__ void __launch_bounds__(SCAN_T) scan_label_kernel(
    const int32_t* __restrict__ root, const int32_t* __restrict__ cmin,
    const int32_t* __restrict__ inv, int32_t* cid, int64_t n, unsigned int* ticket,
    unsigned long long* state, int32_t* total, int64_t* __restrict__ labels,
    unsigned long long* stamps, unsigned int* done, const unsigned long long* dev_scalars,
    unsigned long long* host_scalars, int scalar_words) {
  griddep_wait();
  __shared__ unsigned int tile_sh;
  __shared__ int prefix_sh;
  if (threadIdx.x == 0) tile_sh = atomicAdd(ticket, 1u);
  __syncthreads();
  const unsigned int tile = tile_sh;
  const int64_t base = (int64_t)tile * SCAN_BLK + (int64_t)threadIdx.x * SCAN_PER;
  int r[SCAN_PER];
  int f[SCAN_PER];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    const int64_t o = base + k;
    r[k] = o < n ? root[inv ? inv[o] : o] : -1;
    f[k] = (r[k] >= 0 && cmin[r[k]] == (int)o) ? 1 : 0;
    sum += f[k];
  }
  int agg;
  const int excl = block_exclusive_scan(sum, agg);
  if (threadIdx.x < 32) {  // warp 0: publish the aggregate, look back 32 tiles at a time
    const int lane = threadIdx.x;
    volatile unsigned long long* st = state;
    int prefix = 0;
    if (tile == 0) {
      if (lane == 0) st[0] = SC_PRE | (unsigned int)agg;
    } else {
      if (lane == 0) st[tile] = SC_AGG | (unsigned int)agg;
      int64_t hi = (int64_t)tile - 1;
      for (;;) {
        const int64_t j = hi - lane;
        const unsigned long long w = j >= 0 ? st[j] : (2ull << 62);
        const unsigned flag = (unsigned)(w >> 62);
        const unsigned pre = __ballot_sync(0xffffffffu, flag == 2u);
        const int stop = pre ? __ffs(pre) - 1 : 31;
        const unsigned need = stop == 31 ? 0xffffffffu : ((2u << stop) - 1u);
        if (__ballot_sync(0xffffffffu, flag == 0u) & need) continue;  // not published yet
        int v = lane <= stop ? (int)(unsigned int)w : 0;
#pragma unroll
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        prefix += v;
        if (pre) break;
        hi -= 32;
      }
      if (lane == 0) {
        __threadfence();
        st[tile] = SC_PRE | (unsigned int)(prefix + agg);
      }
    }
    if (lane == 0) {
      prefix_sh = prefix;
      if ((int64_t)(tile + 1) * SCAN_BLK >= n) *total = prefix + agg;  // last tile
    }
  }
  __syncthreads();
  int run = prefix_sh + excl;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    if (f[k]) cid[r[k]] = run;
    run += f[k];
  }
  __threadfence();
  __syncthreads();
  const volatile int32_t* vc = cid;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    int64_t lab = -1;
    if (r[k] >= 0) {
      int v = vc[r[k]];
      while (v < 0) v = vc[r[k]];  // published by an earlier tile (see above)
      lab = v;
    }
    if (base + k < n) labels[base + k] = lab;
  }
  if (stamps || host_scalars) {  // the last block to finish: end-of-stage-3 stamp, scalars
    __shared__ bool last_sh;
    __threadfence();  // this block's writes (ids, the cluster count) before its arrival
    __syncthreads();
    if (threadIdx.x == 0) last_sh = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last_sh) {  // block-uniform
      if (threadIdx.x == 0 && stamps) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        stamps[ST_LABELS_DONE] = t;
      }
      __syncthreads();
      // one word per thread; the kernel's completion makes them visible to the host
      if (host_scalars && (int)threadIdx.x < scalar_words) {
        const volatile unsigned long long* src = dev_scalars;
        host_scalars[threadIdx.x] = src[threadIdx.x];
      }
    }
  }
}

__global__ void counts_i64_kernel(const int32_t* __restrict__ cnt, int64_t n,
                                  const int32_t* __restrict__ perm, int64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[perm ? perm[i] : i] = cnt[i];
}

// chunks -> dense native-word rows in ORIGINAL index order, both orientations
// (the chunks only hold a <= b)
__global__ void export_bits_kernel(const uint2* __restrict__ words, unsigned long long words_cap,
                                   const uint2* __restrict__ uchunks, const uint4* __restrict__ dir,
                                   const unsigned long long* __restrict__ ndir,
                                   const int32_t* __restrict__ perm, uint32_t* bits32,
                                   int64_t stride_words) {
  __shared__ ItemWords iw;
  const unsigned long long total = *ndir;
  for (unsigned long long c = blockIdx.x; c < total; c += gridDim.x) {
    const DirInfo ci = decode_dir(dir[c]);
    load_item_words(ci, uchunks, words_cap, iw);
    if (!iw.ok) continue;
    for (int k = threadIdx.x; k < iw.total; k += blockDim.x) {
      const uint2 rec = item_word(iw, words, (uint32_t)k);
      uint32_t x = rec.x;
      const int64_t is = (int64_t)ci.a * TILE + (rec.y >> 4);
      const int64_t i = perm ? perm[is] : is;
      const int64_t jw = (int64_t)ci.b * WPR + (rec.y & 15u);
      while (x) {
        const int t = __clz(x);
        x &= ~(0x80000000u >> t);
        const int64_t js = jw * 32 + t;
        const int64_t j = perm ? perm[js] : js;
        atomicOr(&bits32[i * stride_words + (j >> 5)], 0x80000000u >> (j & 31));
        atomicOr(&bits32[j * stride_words + (i >> 5)], 0x80000000u >> (i & 31));
      }
    }
  }
}

// native word (bit 31 = first column) <-> little-endian bytes of numpy packbits rows
__global__ void bswap_kernel(uint32_t* bits32, int64_t total) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x)
    bits32[k] = __byte_perm(bits32[k], 0, 0x0123);
}

// Multi-GPU: fold the R per-shard forests into one. parents is R x n; every
// parent pointer of a shard is a connectivity fact of that shard's edges, so
// linking i with parents[r][i] for all r yields the union of all shards' edges.
__global__ void merge_forests_kernel(const int32_t* __restrict__ parents, int R, int64_t n,
                                     const uint8_t* __restrict__ core, int32_t* parent) {
  const int64_t total = (int64_t)R * n;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k % n;
    const int p = parents[k];
    if (p != (int)i && core[i]) link_root(parent, find_plain(parent, (int)i), p);
  }
}

// Multi-GPU pairwise fold: parent |= the forest `other` (link i with other[i] for every
// i it moves), then every entry is pointed at its root so the forest sent on in the
// next round of the exchange is flat.
__global__ void fold_forest_kernel(const int32_t* __restrict__ other, int64_t n, int32_t* parent) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int p = other[i];
    if (p != (int)i) link_root(parent, find_plain(parent, (int)i), p);
  }
}

__global__ void flatten_forest_kernel(int64_t n, int32_t* parent) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    parent[i] = find_root_ro(parent, (int)i);  // roots are final: read-only walk
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

cudaError_t launch_fold_forest(int32_t* parent, const int32_t* other, int64_t n, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  fold_forest_kernel<<<sms * 8, 256, 0, s>>>(other, n, parent);
  flatten_forest_kernel<<<sms * 8, 256, 0, s>>>(n, parent);
  return cudaGetLastError();
}

int64_t scan_partials_len(int64_t n) { return 2 * ((n + SCAN_BLK - 1) / SCAN_BLK + 1); }

cudaError_t launch_core_init(const MergeWs& w, int64_t min_pts, cudaStream_t s) {
  const int t = 256;
  core_init_kernel<<<blocks_for(w.n, t), t, 0, s>>>(w.cnt, w.n, min_pts, w.core, w.corew,
                                                    w.parent, w.bmin, w.cmin, w.ncore);
  return cudaGetLastError();
}

cudaError_t launch_union_chunks(const MergeWs& w, const UnitArgs& units, int lane_blocks,
                                const uint2* diag_range, const CoreInit& ci, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // round 1: one CTA per tile (wide, dense in shared memory); round 2: a warp per unit
  const size_t diag_smem = (size_t)(WPR * DIAG_RS + 512) * 4 + (size_t)3 * TILE * 4;
  // kernel attributes and occupancy are per device (idempotent if raced)
  static std::atomic<int> links_per_sm_dev[DS_MAX_DEVICES] = {};
  int links_per_sm = dev < DS_MAX_DEVICES ? links_per_sm_dev[dev].load() : 0;
  if (links_per_sm == 0) {
    cudaFuncSetAttribute(union_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)diag_smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&links_per_sm, union_links_kernel,
                                                      LINK_WARPS * 32, 0) != cudaSuccess ||
        links_per_sm < 1)
      links_per_sm = 4;
    if (dev < DS_MAX_DEVICES) links_per_sm_dev[dev].store(links_per_sm);
  }
  const int64_t ntiles = (w.n + TILE - 1) / TILE;
  const int64_t grid = ntiles < (int64_t)sms * 8 ? ntiles : (int64_t)sms * 8;
  cudaError_t e = launch_pdl(union_diag_kernel, dim3((unsigned)grid), dim3(512), diag_smem, s, units,
                             lane_blocks, diag_range, ci, (const uint32_t*)w.corew, w.parent,
                             w.bmin, w.perm, w.blk_root);
  if (e != cudaSuccess) return e;
  // one resident wave of union_links: warps take units grid-stride
  return launch_pdl(union_links_kernel, dim3(sms * links_per_sm), dim3(LINK_WARPS * 32), 0, s, units,
                    lane_blocks, (const uint32_t*)w.corew, w.parent, w.bmin, w.perm,
                    (const int32_t*)w.blk_root, w.link_tab, w.link_mask);
}

cudaError_t launch_union_dense(const MergeWs& w, const uint32_t* bits32, int64_t stride_words,
                               cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  union_dense_kernel<<<sms * 8, 256, 0, s>>>(bits32, stride_words, w.n, w.core, w.corew, w.parent,
                                             w.bmin);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const MergeWs& w, int64_t* labels, cudaStream_t s) {
  const int t = 256;
  const unsigned b = blocks_for(w.n, t);
  // canonical ids: exclusive scan of the first-appearance flags, in original order; its
  // look-back state is zeroed first so that roots -> scan -> label chain directly
  const int64_t tiles = (w.n + SCAN_BLK - 1) / SCAN_BLK;
  int32_t* state = w.scan_zeroed ? w.scan_state : w.partials;
  cudaError_t e = w.scan_zeroed ? cudaSuccess
                                : cudaMemsetAsync(state, 0, (size_t)(tiles + 1) * 8, s);
  if (e != cudaSuccess) return e;
  e = launch_pdl(roots_kernel, dim3(b), dim3(t), 0, s, (const uint8_t*)w.core,
                 (const int32_t*)w.parent, (const int32_t*)w.bmin, w.n, w.perm, w.inv, w.root, w.cmin,
                 w.flag);
  if (e != cudaSuccess) return e;
  return launch_pdl(scan_label_kernel, dim3((unsigned)tiles), dim3(SCAN_T), 0, s,
                    (const int32_t*)w.root, (const int32_t*)w.cmin, w.inv, w.flag, w.n,
                    reinterpret_cast<unsigned int*>(state),
                    reinterpret_cast<unsigned long long*>(state) + 1, w.nclusters, labels,
                    w.stamps, w.label_blocks, w.dev_scalars, w.host_scalars,
                    w.scalar_words);
}

cudaError_t launch_merge_forests(const MergeWs& w, const int32_t* parents, int R,
                                 cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  merge_forests_kernel<<<sms * 8, 256, 0, s>>>(parents, R, w.n, w.core, w.parent);
  return cudaGetLastError();
}

// counts between sorted order (device workspace) and original order (shard ABI)
__global__ void permute_i32_kernel(const int32_t* __restrict__ src, int64_t n,
                                   const int32_t* __restrict__ perm, int to_original,
                                   int32_t* __restrict__ dst) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t o = perm ? perm[s] : s;
  if (to_original) dst[o] = src[s];
  else dst[s] = src[o];
}

cudaError_t launch_permute_i32(const int32_t* src, int64_t n, const int32_t* perm, int to_original,
                               int32_t* dst, cudaStream_t s) {
  permute_i32_kernel<<<blocks_for(n, 256), 256, 0, s>>>(src, n, perm, to_original, dst);
  return cudaGetLastError();
}

// partials: scan_partials_len(n) int32 of workspace {ticket, pad, state[tiles]}
cudaError_t launch_exclusive_scan(int32_t* data, int64_t n, int32_t* partials, int32_t* total,
                                  cudaStream_t s) {
  if (n <= 0) return cudaMemsetAsync(total, 0, sizeof(int32_t), s);
  const int64_t tiles = (n + SCAN_BLK - 1) / SCAN_BLK;
  cudaError_t e = cudaMemsetAsync(partials, 0, (size_t)(tiles + 1) * 8, s);
  if (e != cudaSuccess) return e;
  scan_lookback_kernel<<<(unsigned)tiles, SCAN_T, 0, s>>>(
      ScanInPlace{data}, data, n, reinterpret_cast<unsigned int*>(partials),
      reinterpret_cast<unsigned long long*>(partials) + 1, total);
  return cudaGetLastError();
}

cudaError_t launch_scan_zeroed(int32_t* data, int64_t n, void* state, cudaStream_t s) {
  const int64_t tiles = (n + SCAN_BLK - 1) / SCAN_BLK;
  unsigned long long* st = reinterpret_cast<unsigned long long*>(state);
  return launch_pdl(scan_lookback_kernel<ScanInPlace>, dim3((unsigned)tiles), dim3(SCAN_T), 0, s,
                    ScanInPlace{data}, data, n, reinterpret_cast<unsigned int*>(st), st + 1,
                    reinterpret_cast<int32_t*>(st + 1 + tiles));
}
size_t scan_zeroed_bytes(int64_t n) { return (size_t)((n + SCAN_BLK - 1) / SCAN_BLK + 2) * 8; }

cudaError_t launch_counts_i64(const int32_t* cnt, int64_t n, const int32_t* perm, int64_t* out,
                              cudaStream_t s) {
  counts_i64_kernel<<<blocks_for(n, 256), 256, 0, s>>>(cnt, n, perm, out);
  return cudaGetLastError();
}

cudaError_t launch_export_bits(const uint2* words, unsigned long long words_cap, const uint2* uchunks,
                               const uint4* dir, const unsigned long long* ndir, const int32_t* perm,
                               uint32_t* bits32, int64_t stride_words, cudaStream_t s) {
  export_bits_kernel<<<148 * 4, 256, 0, s>>>(words, words_cap, uchunks, dir, ndir, perm, bits32,
                                             stride_words);
  return cudaGetLastError();
}

cudaError_t launch_bswap_rows(uint32_t* bits32, int64_t n, int64_t stride_words, cudaStream_t s) {
  const int64_t total = n * stride_words;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  bswap_kernel<<<(unsigned)blocks, 256, 0, s>>>(bits32, total);
  return cudaGetLastError();
}

}  // namespace ds
