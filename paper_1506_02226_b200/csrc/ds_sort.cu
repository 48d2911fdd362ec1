// Spatial ordering of the points before tiling.
//
// The eps-tile kernel evaluates 512 x 512 tile pairs, and bounding-box culling
// (ds_tile.cu, keep_item) skips the pairs of tiles that are provably apart. Both
// work best when a tile is a compact region: the points are therefore visited in
// Morton (Z-curve) order of their quantised coordinates. Sorting only changes
// which pairs share a tile, never a pair's arithmetic, so bits and counts are
// unchanged; every index-dependent rule (the lowest-indexed-core border rule,
// merge.py:116-130, and first-appearance numbering, core.py:116-132) is applied
// to ORIGINAL indices through perm / inv (ds_merge.cu).
//
// Keys: up to 4 leading dimensions quantised to a 2^(b/k)-per-dimension grid over
// the global bounding box (reduced by the prep kernel), b = 16 bits (two radix passes)
// for 1-2-D inputs up to 2^18 points and 24 bits otherwise — far finer than a
// 512-point tile. The sort is a hand-written stable LSD radix sort over 8-bit digits
// on (key, original index) — ties keep index order — so the permutation is
// deterministic and identical on every rank:
//   morton_kernel   keys of one chunk of points per CTA + the chunk's digit
//                   histogram of pass 0 (shared-memory atomics, written per chunk);
//   digit_scan      one CTA per digit: exclusive scan over the chunks of that digit's
//                   per-chunk counts, and the digit's total;
//   radix_scatter   one CTA per chunk of the pass's input order: digit bases (scan of
//                   the 256 totals), stable rank of each
//                   item among equal digits (warp match_any + per-warp counts in
//                   shared memory, rounds of 256 items in index order), written to
//                   base + rank; it also counts the next pass's digits per output
//                   chunk (global atomics) and, on the last pass, writes perm / inv.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ds_internal.cuh"

namespace ds {
namespace {

// total key bits: 16 (two radix passes, a 256 x 256 grid) for 1-2-D inputs up to
// 2^18 points, 24 (three passes) otherwise
// Measured on B200 (key-bit sweep, round 1): about one point per grid cell keeps the
// 32-point block boxes tight — 12-bit keys nearly double the pairs evaluated at C2,
// 16 bits are best up to ~2^18 points (two radix passes), 24 above (C3 -3 %, C5 -12 %
// pairs vs 16/20 bits).
inline int key_bits(int64_t n, int kd) { return (kd <= 2 && n <= (1 << 18)) ? 16 : 24; }

__device__ __forceinline__ float unord(unsigned int u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

constexpr int RS_T = 256;               // threads per radix CTA
constexpr int RS_MAXP = 3;              // passes (24-bit keys)
// items per thread (chunk = RS_T * items per CTA): 2 up to 2^18 points (more, shorter
// CTAs: C2 best), 4 above (C5: fewer per-chunk counts and CTA waves, -17 us)
inline int rs_items(int64_t n) { return n <= (1 << 18) ? 2 : 4; }
__host__ __device__ inline int64_t rs_chunks(int64_t n, int items) {
  return (n + RS_T * items - 1) / (RS_T * items);
}

// Keys of chunk c (items c*CHUNK + r*256 + t) and the chunk's pass-0 digit counts
// (counts0[d * nch + c]).
template <int RS_ITEMS>
__global__ void __launch_bounds__(RS_T) morton_kernel(
    const float* __restrict__ rec, int64_t n, int S, int kd, int total_bits, int npass,
    const unsigned int* __restrict__ lo_bits, const unsigned int* __restrict__ hi_bits,
    uint32_t* __restrict__ keys, int32_t* __restrict__ counts) {
  griddep_wait();
  __shared__ int hist[1][256];
  const int t = threadIdx.x;
  constexpr int RS_CHUNK = RS_T * RS_ITEMS;
  const int64_t nch = rs_chunks(n, RS_ITEMS);
  const int64_t c = blockIdx.x;
  hist[0][t] = 0;
  __syncthreads();
  const int bits = total_bits / kd;
  const float levels = (float)((1u << bits) - 1);
  // quantisation in float (any deterministic, monotone map is fine: the order only
  // schedules work); the scale is computed once per CTA instead of a division per item
  float lo[4], scale[4];
  for (int k = 0; k < kd; ++k) {
    lo[k] = unord(~lo_bits[k]);  // lo is stored inverted
    const float span = unord(hi_bits[k]) - lo[k];
    scale[k] = span > 0.f ? levels / span : 0.f;
  }
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    const int64_t i = c * RS_CHUNK + r * RS_T + t;
    if (i >= n) break;
    uint32_t q[4] = {0, 0, 0, 0};
    for (int k = 0; k < kd; ++k) {
      float v = (rec[i * S + k] - lo[k]) * scale[k];
      v = v < 0.f ? 0.f : (v > levels ? levels : v);
      q[k] = (v == v) ? (uint32_t)v : 0u;  // NaN -> 0
    }
    uint32_t key = 0;  // <= 24 bits
    for (int b = bits - 1; b >= 0; --b)
      for (int k = 0; k < kd; ++k) key = (key << 1) | ((q[k] >> b) & 1u);
    keys[i] = key;
    atomicAdd(&hist[0][key & 255u], 1);
  }
  __syncthreads();
  counts[(int64_t)t * nch + c] = hist[0][t];  // the next passes' rows: zeroed by digit_scan
}

// One CTA per digit d: exclusive scan over the chunks of the digit's counts (in
// place) and the digit's total (totals[d]); the scatter adds the digit bases.
// next (nullable): the next pass's counts, whose row d this CTA zeroes (coalesced; that
// pass's radix_scatter of this pass adds to them once this kernel has completed).
__global__ void __launch_bounds__(RS_T) digit_scan_kernel(int32_t* __restrict__ counts,
                                                          int32_t* __restrict__ totals,
                                                          int64_t nch, int32_t* __restrict__ next) {
  griddep_wait();
  if (next)
    for (int64_t c = threadIdx.x; c < nch; c += RS_T) next[(int64_t)blockIdx.x * nch + c] = 0;
  __shared__ int warp_sum[RS_T / 32];
  const int d = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int carry = 0;
  int32_t* row = counts + (int64_t)d * nch;
  for (int64_t base = 0; base < nch; base += RS_T) {
    const int64_t c = base + t;
    const int x = c < nch ? row[c] : 0;
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) warp_sum[warp] = inc;
    __syncthreads();
    int wpre = 0, all = 0;
#pragma unroll
    for (int w = 0; w < RS_T / 32; ++w) {
      const int ws = warp_sum[w];
      if (w < warp) wpre += ws;
      all += ws;
    }
    if (c < nch) row[c] = carry + wpre + inc - x;
    carry += all;
    __syncthreads();  // warp_sum is rewritten by the next round
  }
  if (t == 0) totals[d] = carry;
}

// Stable scatter of one pass: chunk c of the input order (keys_in / vals_in, vals
// implicit = index on pass 0). Items are ranked in index order; on the last pass the
// permutation goes to perm / inv, otherwise keys / values to the output arrays and the
// next pass's digit is counted for the output chunk.
template <int RS_ITEMS>
__global__ void __launch_bounds__(RS_T) radix_scatter_kernel(
    int64_t n, int shift, const uint32_t* __restrict__ keys_in, const int32_t* __restrict__ vals_in,
    const int32_t* __restrict__ offs, uint32_t* __restrict__ keys_out, int32_t* __restrict__ vals_out,
    int32_t* __restrict__ next_counts, int32_t* __restrict__ perm, int32_t* __restrict__ inv,
    const int32_t* __restrict__ totals) {
  griddep_wait();
  __shared__ int base[256];
  __shared__ int wsum[RS_T / 32];
  __shared__ int wcnt[2][RS_T / 32][256];  // double-buffered over the rounds
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  constexpr int RS_CHUNK = RS_T * RS_ITEMS;
  const int64_t nch = rs_chunks(n, RS_ITEMS);
  const int64_t c = blockIdx.x;
  {  // digit base = exclusive scan of the digit totals, plus this chunk's offset
    const int x = totals[t];
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int wpre = 0;
#pragma unroll
    for (int w = 0; w < RS_T / 32; ++w)
      if (w < warp) wpre += wsum[w];
    base[t] = wpre + inc - x + offs[(int64_t)t * nch + c];
  }
  const uint32_t lt = (1u << lane) - 1u;
  for (int r = 0; r < RS_ITEMS; ++r) {
    const int64_t i = c * RS_CHUNK + r * RS_T + t;
    const bool valid = i < n;
    uint32_t key = 0;
    int32_t val = 0;
    if (valid) {
      key = keys_in[i];
      val = vals_in ? vals_in[i] : (int32_t)i;
    }
    const int dig = valid ? (int)((key >> shift) & 255u) : 256;
    // buffer r & 1 was last read two rounds ago: the barriers of round r - 1 separate
    // those reads from this zeroing
    int(*wc)[256] = wcnt[r & 1];
#pragma unroll
    for (int w = 0; w < RS_T / 32; ++w) wc[w][t] = 0;
    __syncthreads();  // also orders base[] (round 0)
    const uint32_t peers = __match_any_sync(0xffffffffu, dig);
    const int lrank = __popc(peers & lt);
    if (valid && lrank == 0) wc[warp][dig] = __popc(peers);
    __syncthreads();
    {  // per digit: exclusive prefix over the warps, then advance the digit's base
      int run = base[t];
#pragma unroll
      for (int w = 0; w < RS_T / 32; ++w) {
        const int x = wc[w][t];
        wc[w][t] = run;
        run += x;
      }
      base[t] = run;
    }
    __syncthreads();
    if (valid) {
      const int64_t pos = (int64_t)wc[warp][dig] + lrank;
      if (perm) {
        perm[pos] = val;
        inv[val] = (int32_t)pos;
      } else {
        keys_out[pos] = key;
        vals_out[pos] = val;
        if (next_counts)
          atomicAdd(&next_counts[(int64_t)((key >> (shift + 8)) & 255u) * nch + pos / RS_CHUNK], 1);
      }
    }
  }
}

// ---- counting sort on 16-bit keys (one GPU): the order within a key is arbitrary ----
// The key grid cell (~1 point per cell at n <= 2^18) is the unit of locality; the order
// of the points inside a cell does not matter for the tiles' compactness, and labels do
// not depend on the order at all. Three kernels instead of the radix
// sort's five: keys + a global histogram over the 65536 cells, a look-back exclusive
// scan of it (16 CTAs), and a scatter with one atomic per (warp, cell) group. bins is
// followed by the scan's look-back state; both zeroed per call.
constexpr int CS_BINS = 1 << 16;

__global__ void __launch_bounds__(RS_T) morton_count_kernel(
    const float* __restrict__ rec, int64_t n, int S, int kd, int total_bits,
    const unsigned int* __restrict__ lo_bits, const unsigned int* __restrict__ hi_bits,
    uint32_t* __restrict__ keys, unsigned int* __restrict__ bins) {
  griddep_wait();
  const int bits = total_bits / kd;
  const float levels = (float)((1u << bits) - 1);
  float lo[4], scale[4];
  for (int k = 0; k < kd; ++k) {
    lo[k] = unord(~lo_bits[k]);  // lo is stored inverted
    const float span = unord(hi_bits[k]) - lo[k];
    scale[k] = span > 0.f ? levels / span : 0.f;
  }
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    uint32_t key = 0xffffffffu;
    if (i < n) {
      uint32_t q[4] = {0, 0, 0, 0};
      for (int k = 0; k < kd; ++k) {
        float v = (rec[i * S + k] - lo[k]) * scale[k];
        v = v < 0.f ? 0.f : (v > levels ? levels : v);
        q[k] = (v == v) ? (uint32_t)v : 0u;  // NaN -> 0
      }
      key = 0;
      for (int b = bits - 1; b >= 0; --b)
        for (int k = 0; k < kd; ++k) key = (key << 1) | ((q[k] >> b) & 1u);
      keys[i] = key;
    }
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    if (i < n && lane == __ffs(grp) - 1) atomicAdd(&bins[key], (unsigned int)__popc(grp));
  }
}

// positions: one atomic per (warp, cell) group on the cell's running start
__global__ void __launch_bounds__(RS_T) count_scatter_kernel(int64_t n, const uint32_t* __restrict__ keys,
                                                             unsigned int* __restrict__ bins,
                                                             int32_t* __restrict__ perm,
                                                             int32_t* __restrict__ inv) {
  griddep_wait();
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const uint32_t key = i < n ? keys[i] : 0xffffffffu;
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(grp) - 1;
    unsigned int base = 0;
    if (i < n && lane == leader) base = atomicAdd(&bins[key], (unsigned int)__popc(grp));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (i < n) {
      const int64_t pos = (int64_t)base + __popc(grp & ((1u << lane) - 1u));
      perm[pos] = (int32_t)i;
      inv[i] = (int32_t)pos;
    }
  }
}

__global__ void permute_kernel(const float* __restrict__ rec, int64_t n, int S,
                               const int32_t* __restrict__ perm, float* __restrict__ out) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t o = perm[s];
  const float4* src = reinterpret_cast<const float4*>(rec + o * S);
  float4* dst = reinterpret_cast<float4*>(out + s * S);
  for (int v = 0; v < S / 4; ++v) dst[v] = src[v];
}

// permute_kernel fused with the culling bounds (stage 1+2 with culling on): one CTA of
// PB_T threads per 512-point tile (TILE / PB_T points per thread, their loads in
// flight together; 128 threads at C5's 3,907 tiles: two resident waves instead of
// seven of 512-thread CTAs) copies its records into sorted order, then reduces per 32-point block (one
// warp and round) the box and max squared norm (blk, the layout of block_bounds_kernel
// in ds_tile.cu; nullptr: skip) and per tile the box and max norm (lo / hi / maxnorm,
// the layout of tile_bounds_kernel), and adds the tile box to its super tile's.
template <int PB_T>
__global__ void __launch_bounds__(PB_T) permute_bounds_kernel(
    const float* __restrict__ rec, int64_t n, int S, int dpad, const int32_t* __restrict__ perm,
    float* __restrict__ out, float* __restrict__ lo,
    float* __restrict__ hi, float* __restrict__ maxnorm, float* __restrict__ blk,
    unsigned int* __restrict__ super) {
  constexpr int PB_P = TILE / PB_T;
  griddep_wait();
  // per column (dpad <= 64, + the norm) and 32-point block: the block's min / max; the
  // tile's box is reduced from them after one barrier, one column per thread
  __shared__ float smn[65][TILE / 32], smx[65][TILE / 32];
  const int64_t tile = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int64_t o[PB_P];
#pragma unroll
  for (int j = 0; j < PB_P; ++j) {
    const int64_t sj = tile * TILE + j * PB_T + t;
    o[j] = sj < n ? perm[sj] : -1;
  }
#pragma unroll
  for (int j = 0; j < PB_P; ++j) {
    if (o[j] < 0) continue;
    const int64_t sj = tile * TILE + j * PB_T + t;
    const float4* src = reinterpret_cast<const float4*>(rec + o[j] * S);
    float4* dst = reinterpret_cast<float4*>(out + sj * S);
    for (int v = 0; v < S / 4; ++v) dst[v] = src[v];
  }
  const int BS = 2 * dpad + 1;
  for (int k = 0; k <= dpad; ++k) {  // k == dpad: the norm column
#pragma unroll
    for (int j = 0; j < PB_P; ++j) {  // block j * (PB_T / 32) + warp of the tile
      const int64_t sj = tile * TILE + j * PB_T + t;
      const bool valid = o[j] >= 0;
      const float v = valid ? out[sj * S + k] : 0.f;
      float mn = valid ? v : INFINITY, mx = valid ? v : -INFINITY;
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      }
      const int bw = j * (PB_T / 32) + warp;
      const int64_t wb = tile * (TILE / 32) + bw;  // global 32-point block
      if (lane == 0) {
        if (blk && wb * 32 < n) {
          if (k < dpad) {
            blk[wb * BS + k] = mn;
            blk[wb * BS + dpad + k] = mx;
          } else {
            blk[wb * BS + 2 * dpad] = mx;
          }
        }
        smn[k][bw] = mn;
        smx[k][bw] = mx;
      }
    }
  }
  __syncthreads();
  for (int k = t; k <= dpad; k += PB_T) {  // k == dpad: the norm column
    float mn = smn[k][0], mx = smx[k][0];
    for (int w = 1; w < TILE / 32; ++w) {
      mn = fminf(mn, smn[k][w]);
      mx = fmaxf(mx, smx[k][w]);
    }
    if (k < dpad) {
      lo[tile * dpad + k] = mn;
      hi[tile * dpad + k] = mx;
    } else {
      maxnorm[tile] = mx;
    }
    if (super) super_box_add(super, tile, dpad, k, mn, mx);
  }
}

}  // namespace

size_t sort_temp_bytes(int64_t n) {
  return ((size_t)RS_MAXP * 256 * rs_chunks(n, rs_items(n)) + RS_MAXP * 256) * 4;  // counts + totals
}

cudaError_t launch_spatial_sort(const float* rec, int64_t n, int d, float* rec_sorted,
                                int32_t* perm, int32_t* inv, unsigned long long* keys,
                                unsigned long long* keys_alt, int32_t* idx, void* temp,
                                size_t temp_bytes, unsigned int* bbox, const SortBounds& bnd,
                                unsigned int* bins, cudaStream_t s) {
  const int dp = padded_dim(d);
  const int S = rec_stride(d);
  const int kd = d < 4 ? d : 4;
  // the bounding box was reduced by the prep kernel (launch_prep with a bbox buffer)
  const int kb = key_bits(n, kd);
  const int end_bit = (kb / kd) * kd;
  const int npass = (end_bit + 7) / 8;
  const int items = rs_items(n);
  const int64_t nch = rs_chunks(n, items);
  if (temp_bytes < sort_temp_bytes(n)) return cudaErrorInvalidValue;
  int32_t* counts = reinterpret_cast<int32_t*>(temp);
  int32_t* totals = counts + (int64_t)RS_MAXP * 256 * nch;  // per pass, written by the scans
  // ping-pong: keys A / B in the two halves of `keys`, values in idx / keys_alt
  uint32_t* kA = reinterpret_cast<uint32_t*>(keys);
  uint32_t* kB = kA + n;
  int32_t* vA = idx;
  int32_t* vB = reinterpret_cast<int32_t*>(keys_alt);
  cudaError_t e = cudaSuccess;
  if (bins && kb == 16) {  // counting sort (zeroed bins): keys + histogram, scan, scatter
    const unsigned g = (unsigned)std::min<int64_t>((n + RS_T - 1) / RS_T, 148 * 8);
    e = launch_pdl(morton_count_kernel, dim3(g), dim3(RS_T), 0, s, rec, n, S, kd, kb,
                   (const unsigned int*)bbox, (const unsigned int*)(bbox + 4), kA, bins);
    if (e != cudaSuccess) return e;
    e = launch_scan_zeroed(reinterpret_cast<int32_t*>(bins), CS_BINS, bins + CS_BINS, s);
    if (e != cudaSuccess) return e;
    e = launch_pdl(count_scatter_kernel, dim3(g), dim3(RS_T), 0, s, n, (const uint32_t*)kA, bins, perm,
                   inv);
    if (e != cudaSuccess) return e;
  } else {  // stable LSD radix sort (deterministic order: every rank the same)
    e = launch_pdl(items == 2 ? morton_kernel<2> : morton_kernel<4>, dim3((unsigned)nch),
                               dim3(RS_T), 0, s, rec, n, S, kd, kb,
                               npass, (const unsigned int*)bbox, (const unsigned int*)(bbox + 4), kA,
                               counts);
    if (e != cudaSuccess) return e;
    const uint32_t* kin = kA;
    const int32_t* vin = nullptr;
    for (int p = 0; p < npass; ++p) {
      int32_t* cp = counts + (int64_t)p * 256 * nch;
      e = launch_pdl(digit_scan_kernel, dim3(256), dim3(RS_T), 0, s, cp, totals + p * 256, nch,
                     p + 1 < npass ? counts + (int64_t)(p + 1) * 256 * nch : (int32_t*)nullptr);
      if (e != cudaSuccess) return e;
      const bool last = p == npass - 1;
      uint32_t* kout = (p & 1) ? kA : kB;
      int32_t* vout = (p & 1) ? vA : vB;
      e = launch_pdl(items == 2 ? radix_scatter_kernel<2> : radix_scatter_kernel<4>, dim3((unsigned)nch),
                     dim3(RS_T), 0, s, n, 8 * p, kin, vin,
                     (const int32_t*)cp, last ? (uint32_t*)nullptr : kout,
                     last ? (int32_t*)nullptr : vout,
                     last ? (int32_t*)nullptr : counts + (int64_t)(p + 1) * 256 * nch,
                     last ? perm : (int32_t*)nullptr, last ? inv : (int32_t*)nullptr,
                     (const int32_t*)(totals + p * 256));
      if (e != cudaSuccess) return e;
      kin = kout;
      vin = vout;
    }
  }
  if (bnd.lo) {
    // one 512-thread CTA per tile while the tiles fit one resident wave (C2: faster),
    // 128-thread CTAs with four points per thread beyond (C5: fewer waves)
    const bool wide = n_tiles(n) <= 148 * 4;
    e = launch_pdl(wide ? permute_bounds_kernel<TILE> : permute_bounds_kernel<128>,
                   dim3((unsigned)n_tiles(n)), dim3(wide ? TILE : 128), 0, s, rec, n, S, dp,
                   (const int32_t*)perm, rec_sorted, bnd.lo, bnd.hi, bnd.maxnorm, bnd.blk,
                   dp <= 4 ? bnd.super : (unsigned int*)nullptr);
    if (e != cudaSuccess) return e;
  } else {
    const unsigned blocks = (unsigned)((n + 255) / 256);
    permute_kernel<<<blocks, 256, 0, s>>>(rec, n, S, perm, rec_sorted);
  }
  return cudaGetLastError();
}

}  // namespace ds
