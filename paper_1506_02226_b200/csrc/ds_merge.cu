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

// Read-only find for the compress pass: a path-halving write racing with the
// compress store could otherwise re-point an already compressed node at a
// non-root ancestor.
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

// ---- union over tile-pair chunks (two rounds, shared-memory local forests) ---------
// Round 1 (diagonal chunks, one per tile): the core-core words of tile a with
// itself are merged in a shared-memory union-find over the tile's 512 points;
// every core point then gets parent = its local root (the smallest index of
// its local component). Each tile is owned by exactly one CTA, so these
// writes need no atomics.
// Round 2 (off-diagonal chunks): the 1024 points of tiles a and b first look
// up their current global roots; a core-core bit whose endpoints already share
// a root costs nothing, the others are merged in shared memory, and only one
// global link per (local component, differing global root) is issued. In dense
// regions that is ~1 global CAS per tile pair instead of one per in-range pair.
// Border minima are reduced per chunk in shared memory, then once per point in
// global memory.
struct ChunkInfo {
  int a, b;
  unsigned long long base;
  int count;
};

__device__ __forceinline__ ChunkInfo decode_chunk(uint4 c) {
  ChunkInfo ci;
  ci.a = (int)c.x;
  ci.b = (int)c.y;
  ci.base = (unsigned long long)c.z | ((unsigned long long)(c.w >> 16) << 32);
  ci.count = (int)(c.w & 0xffffu);
  return ci;
}

__device__ __forceinline__ int find_local(int* lp, int v) {
  int p = lp[v];
  while (p != v) {
    const int gp = lp[p];
    if (gp != p) lp[v] = gp;  // halving (smem; benign race)
    v = p;
    p = gp;
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

template <int ROUND>
__global__ void __launch_bounds__(128) union_chunks_kernel(
    const uint4* __restrict__ chunks, const unsigned long long* __restrict__ nchunks,
    const uint2* __restrict__ words, int64_t n, const uint8_t* __restrict__ core,
    const uint32_t* __restrict__ corew, int32_t* parent, int32_t* bmin,
    const int32_t* __restrict__ perm) {
  __shared__ int lp[2 * TILE];
  __shared__ int gr[2 * TILE];
  __shared__ int lb[2 * TILE];
  __shared__ uint32_t lcw[2 * WPR];
  const int tid = threadIdx.x;
  const unsigned long long total = *nchunks;
  const int64_t nw = (n + 31) / 32;
  for (unsigned long long c = blockIdx.x; c < total; c += gridDim.x) {
    const ChunkInfo ci = decode_chunk(chunks[c]);
    const bool diag = ci.a == ci.b;
    if ((ROUND == 1) != diag) continue;  // uniform per CTA
    const int nloc = diag ? TILE : 2 * TILE;
    for (int v = tid; v < nloc; v += blockDim.x) {
      const int64_t g = (int64_t)(v < TILE ? ci.a : ci.b) * TILE + (v & (TILE - 1));
      lp[v] = v;
      lb[v] = NONE;
      int r = (int)g;
      if (ROUND == 2 && g < n && core[g]) r = find_plain(parent, (int)g);
      gr[v] = r;
    }
    if (tid < (diag ? WPR : 2 * WPR)) {
      const int64_t gw = (int64_t)(tid < WPR ? ci.a : ci.b) * WPR + (tid & (WPR - 1));
      lcw[tid] = gw < nw ? corew[gw] : 0u;
    }
    __syncthreads();
    const int jb = diag ? 0 : TILE;  // local index of column 0 of tile b
    for (int k = tid; k < ci.count; k += blockDim.x) {
      const uint2 rec = words[ci.base + k];
      const uint32_t x = rec.x;
      const int u = (int)(rec.y >> 4);
      const int w = (int)(rec.y & 15u);
      const uint32_t cw = lcw[(diag ? 0 : WPR) + w];
      const bool cu = (lcw[u >> 5] >> (31 - (u & 31))) & 1u;
      const int vb = jb + w * 32;
      if (cu) {
        uint32_t um = x & cw;  // core-core (merge.py:149-159)
        while (um) {
          const int t = __clz(um);
          um &= ~(0x80000000u >> t);
          const int v = vb + t;
          if (ROUND == 1 || gr[u] != gr[v]) unite_local(lp, u, v);
        }
        uint32_t bm = x & ~cw;  // core u in range of non-core v (merge.py:116-130)
        const int gu = perm ? perm[ci.a * TILE + u] : ci.a * TILE + u;  // original index
        while (bm) {
          const int t = __clz(bm);
          bm &= ~(0x80000000u >> t);
          atomicMin(&lb[vb + t], gu);
        }
      } else {
        const uint32_t cm = x & cw;  // non-core u: its lowest in-range core
        if (cm) {
          const int jb0 = (diag ? ci.a : ci.b) * TILE + w * 32;
          if (perm) {  // lowest ORIGINAL index among the in-range cores of the word
            int best = NONE;
            uint32_t mm = cm;
            while (mm) {
              const int t = __clz(mm);
              mm &= ~(0x80000000u >> t);
              best = min(best, perm[jb0 + t]);
            }
            atomicMin(&lb[u], best);
          } else {
            atomicMin(&lb[u], jb0 + __clz(cm));
          }
        }
      }
    }
    __syncthreads();
    for (int v = tid; v < nloc; v += blockDim.x) {
      const int64_t g = (int64_t)(v < TILE ? ci.a : ci.b) * TILE + (v & (TILE - 1));
      if (g >= n) continue;
      const int r = find_local(lp, v);
      if (ROUND == 1) {
        if (r != v) parent[g] = (int)((int64_t)ci.a * TILE + r);  // r < v: parent[x] <= x holds
      } else if (r != v && gr[v] != gr[r]) {
        link_root(parent, find_plain(parent, gr[v]), gr[r]);
      }
      if (lb[v] != NONE) atomicMin(&bmin[g], lb[v]);
    }
    __syncthreads();
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

__global__ void compress_kernel(const uint8_t* __restrict__ core, int64_t n, int32_t* parent) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && core[i]) parent[i] = find_root_ro(parent, (int)i);
}

// Runs over sorted indices s; bmin holds ORIGINAL indices of cores, cmin collects
// the lowest ORIGINAL member index of each root (borders included).
__global__ void roots_kernel(const uint8_t* __restrict__ core, const int32_t* __restrict__ parent,
                             const int32_t* __restrict__ bmin, int64_t n,
                             const int32_t* __restrict__ perm, const int32_t* __restrict__ inv,
                             int32_t* __restrict__ root, int32_t* cmin) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int r = -1;
  if (core[i]) {
    r = parent[i];
  } else {
    const int b = bmin[i];
    if (b != NONE) r = parent[inv ? inv[b] : b];
  }
  root[i] = r;
  if (r >= 0) atomicMin(&cmin[r], perm ? perm[i] : (int)i);  // first appearance
}

// flag[o] = 1 iff original index o is the first appearance of its cluster
__global__ void flags_kernel(const int32_t* __restrict__ root, const int32_t* __restrict__ cmin,
                             int64_t n, const int32_t* __restrict__ perm, int32_t* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int r = root[i];
  const int o = perm ? perm[i] : (int)i;
  flag[o] = (r >= 0 && cmin[r] == o) ? 1 : 0;
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

__global__ void scan_partials_kernel(const int32_t* __restrict__ flag, int64_t n,
                                     int32_t* __restrict__ partials) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_BLK + (int64_t)threadIdx.x * SCAN_PER;
  int s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k)
    if (base + k < n) s += flag[base + k];
  int total;
  block_exclusive_scan(s, total);
  if (threadIdx.x == 0) partials[blockIdx.x] = total;
}

__global__ void scan_top_kernel(int32_t* partials, int64_t np, int32_t* total_out) {
  int carry = 0;
  for (int64_t c0 = 0; c0 < np; c0 += SCAN_T) {
    const int64_t idx = c0 + threadIdx.x;
    const int v = idx < np ? partials[idx] : 0;
    int total;
    const int excl = block_exclusive_scan(v, total);
    if (idx < np) partials[idx] = carry + excl;
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total_out = carry;
}

__global__ void scan_apply_kernel(int32_t* flag, int64_t n, const int32_t* __restrict__ partials) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_BLK + (int64_t)threadIdx.x * SCAN_PER;
  int v[SCAN_PER];
  int s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    v[k] = base + k < n ? flag[base + k] : 0;
    s += v[k];
  }
  int total;
  int run = block_exclusive_scan(s, total) + partials[blockIdx.x];
#pragma unroll
  for (int k = 0; k < SCAN_PER; ++k) {
    if (base + k < n) flag[base + k] = run;
    run += v[k];
  }
}

__global__ void label_kernel(const int32_t* __restrict__ root, const int32_t* __restrict__ cmin,
                             const int32_t* __restrict__ id, int64_t n,
                             const int32_t* __restrict__ perm, int64_t* __restrict__ labels) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int r = root[i];
  labels[perm ? perm[i] : i] = r >= 0 ? (int64_t)id[cmin[r]] : (int64_t)-1;
}

__global__ void counts_i64_kernel(const int32_t* __restrict__ cnt, int64_t n,
                                  const int32_t* __restrict__ perm, int64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[perm ? perm[i] : i] = cnt[i];
}

// chunks -> dense native-word rows in ORIGINAL index order, both orientations
// (the chunks only hold a <= b)
__global__ void export_bits_kernel(const uint2* __restrict__ words, const uint4* __restrict__ chunks,
                                   const unsigned long long* __restrict__ nchunks,
                                   const int32_t* __restrict__ perm, uint32_t* bits32,
                                   int64_t stride_words) {
  const unsigned long long total = *nchunks;
  for (unsigned long long c = blockIdx.x; c < total; c += gridDim.x) {
    const ChunkInfo ci = decode_chunk(chunks[c]);
    for (int k = threadIdx.x; k < ci.count; k += blockDim.x) {
      const uint2 rec = words[ci.base + k];
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

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

int64_t scan_partials_len(int64_t n) { return (n + SCAN_BLK - 1) / SCAN_BLK; }

cudaError_t launch_core_init(const MergeWs& w, int64_t min_pts, cudaStream_t s) {
  const int t = 256;
  core_init_kernel<<<blocks_for(w.n, t), t, 0, s>>>(w.cnt, w.n, min_pts, w.core, w.corew,
                                                    w.parent, w.bmin, w.cmin, w.ncore);
  return cudaGetLastError();
}

cudaError_t launch_union_chunks(const MergeWs& w, const uint2* words, const uint4* chunks,
                                const unsigned long long* nchunks, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  union_chunks_kernel<1><<<sms * 16, 128, 0, s>>>(chunks, nchunks, words, w.n, w.core, w.corew,
                                                 w.parent, w.bmin, w.perm);
  union_chunks_kernel<2><<<sms * 16, 128, 0, s>>>(chunks, nchunks, words, w.n, w.core, w.corew,
                                                 w.parent, w.bmin, w.perm);
  return cudaGetLastError();
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
  compress_kernel<<<b, t, 0, s>>>(w.core, w.n, w.parent);
  roots_kernel<<<b, t, 0, s>>>(w.core, w.parent, w.bmin, w.n, w.perm, w.inv, w.root, w.cmin);
  flags_kernel<<<b, t, 0, s>>>(w.root, w.cmin, w.n, w.perm, w.flag);
  const int64_t np = scan_partials_len(w.n);
  scan_partials_kernel<<<(unsigned)np, SCAN_T, 0, s>>>(w.flag, w.n, w.partials);
  scan_top_kernel<<<1, SCAN_T, 0, s>>>(w.partials, np, w.nclusters);
  scan_apply_kernel<<<(unsigned)np, SCAN_T, 0, s>>>(w.flag, w.n, w.partials);
  label_kernel<<<b, t, 0, s>>>(w.root, w.cmin, w.flag, w.n, w.perm, labels);
  return cudaGetLastError();
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

cudaError_t launch_exclusive_scan(int32_t* data, int64_t n, int32_t* partials, int32_t* total,
                                  cudaStream_t s) {
  const int64_t np = scan_partials_len(n);
  scan_partials_kernel<<<(unsigned)np, SCAN_T, 0, s>>>(data, n, partials);
  scan_top_kernel<<<1, SCAN_T, 0, s>>>(partials, np, total);
  scan_apply_kernel<<<(unsigned)np, SCAN_T, 0, s>>>(data, n, partials);
  return cudaGetLastError();
}

cudaError_t launch_counts_i64(const int32_t* cnt, int64_t n, const int32_t* perm, int64_t* out,
                              cudaStream_t s) {
  counts_i64_kernel<<<blocks_for(n, 256), 256, 0, s>>>(cnt, n, perm, out);
  return cudaGetLastError();
}

cudaError_t launch_export_bits(const uint2* words, const uint4* chunks,
                               const unsigned long long* nchunks, const int32_t* perm,
                               uint32_t* bits32, int64_t stride_words, cudaStream_t s) {
  export_bits_kernel<<<148 * 4, 256, 0, s>>>(words, chunks, nchunks, perm, bits32, stride_words);
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
