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
// 512-point tile. The sort is CUB's stable LSD radix sort on (32-bit key, original
// index), so the permutation is deterministic and identical on every rank.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/cub.cuh>

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

__global__ void morton_kernel(const float* __restrict__ rec, int64_t n, int S, int kd, int total_bits,
                              const unsigned int* __restrict__ lo_bits,
                              const unsigned int* __restrict__ hi_bits,
                              uint32_t* __restrict__ keys, int32_t* __restrict__ idx) {
  griddep_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int bits = total_bits / kd;
  const double levels = (double)((1ull << bits) - 1);
  uint32_t q[4] = {0, 0, 0, 0};
  for (int k = 0; k < kd; ++k) {
    const double lo = unord(~lo_bits[k]), hi = unord(hi_bits[k]);  // lo is stored inverted
    const double span = hi - lo;
    double t = span > 0 ? ((double)rec[i * S + k] - lo) / span * levels : 0.0;
    t = t < 0 ? 0 : (t > levels ? levels : t);  // NaN -> 0 via the comparisons below
    q[k] = (t == t) ? (uint32_t)t : 0u;
  }
  uint32_t key = 0;  // <= 24 bits
  for (int b = bits - 1; b >= 0; --b)
    for (int k = 0; k < kd; ++k) key = (key << 1) | ((q[k] >> b) & 1u);
  keys[i] = key;
  idx[i] = (int32_t)i;
}

__global__ void permute_kernel(const float* __restrict__ rec, int64_t n, int S,
                               const int32_t* __restrict__ perm, float* __restrict__ out,
                               int32_t* __restrict__ inv) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t o = perm[s];
  const float4* src = reinterpret_cast<const float4*>(rec + o * S);
  float4* dst = reinterpret_cast<float4*>(out + s * S);
  for (int v = 0; v < S / 4; ++v) dst[v] = src[v];
  inv[o] = (int32_t)s;
}

// permute_kernel fused with the culling bounds (stage 1+2 with culling on): one CTA
// per 512-point tile copies its records into sorted order, then reduces per
// 32-point block (one warp) the box and max squared norm (blk, the layout of
// block_bounds_kernel in ds_tile.cu; nullptr: skip) and per tile the box and max
// norm (lo / hi / maxnorm, the layout of tile_bounds_kernel).
__global__ void __launch_bounds__(TILE) permute_bounds_kernel(
    const float* __restrict__ rec, int64_t n, int S, int dpad, const int32_t* __restrict__ perm,
    float* __restrict__ out, int32_t* __restrict__ inv, float* __restrict__ lo,
    float* __restrict__ hi, float* __restrict__ maxnorm, float* __restrict__ blk) {
  griddep_wait();
  __shared__ float smn[TILE / 32], smx[TILE / 32];
  const int64_t tile = blockIdx.x;
  const int64_t s = tile * TILE + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool valid = s < n;
  if (valid) {
    const int64_t o = perm[s];
    const float4* src = reinterpret_cast<const float4*>(rec + o * S);
    float4* dst = reinterpret_cast<float4*>(out + s * S);
    for (int v = 0; v < S / 4; ++v) dst[v] = src[v];
    inv[o] = (int32_t)s;
  }
  const int64_t wb = tile * (TILE / 32) + warp;  // global 32-point block
  const bool wvalid = wb * 32 < n;
  const int BS = 2 * dpad + 1;
  for (int k = 0; k <= dpad; ++k) {  // k == dpad: the norm column
    const float v = valid ? out[s * S + k] : 0.f;
    float mn = valid ? v : INFINITY, mx = valid ? v : -INFINITY;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    }
    if (lane == 0) {
      if (blk && wvalid) {
        if (k < dpad) {
          blk[wb * BS + k] = mn;
          blk[wb * BS + dpad + k] = mx;
        } else {
          blk[wb * BS + 2 * dpad] = mx;
        }
      }
      smn[warp] = mn;
      smx[warp] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < TILE / 32; ++w) {
        mn = fminf(mn, smn[w]);
        mx = fmaxf(mx, smx[w]);
      }
      if (k < dpad) {
        lo[tile * dpad + k] = mn;
        hi[tile * dpad + k] = mx;
      } else {
        maxnorm[tile] = mx;
      }
    }
    __syncthreads();
  }
}

}  // namespace

size_t sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return bytes;
}

cudaError_t launch_spatial_sort(const float* rec, int64_t n, int d, float* rec_sorted,
                                int32_t* perm, int32_t* inv, unsigned long long* keys,
                                unsigned long long* keys_alt, int32_t* idx, void* temp,
                                size_t temp_bytes, unsigned int* bbox, const SortBounds& bnd,
                                cudaStream_t s) {
  const int dp = padded_dim(d);
  const int S = rec_stride(d);
  const int kd = d < 4 ? d : 4;
  // the bounding box was reduced by the prep kernel (launch_prep with a bbox buffer)
  const unsigned blocks = (unsigned)((n + 255) / 256);
  const int kb = key_bits(n, kd);
  uint32_t* k32 = reinterpret_cast<uint32_t*>(keys);
  uint32_t* k32_alt = reinterpret_cast<uint32_t*>(keys_alt);
  cudaError_t e = launch_pdl(morton_kernel, dim3(blocks), dim3(256), 0, s, rec, n, S, kd, kb,
                             (const unsigned int*)bbox, (const unsigned int*)(bbox + 4), k32, idx);
  if (e != cudaSuccess) return e;
  e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k32, k32_alt, idx, perm,
                                                  (int)n, 0, (kb / kd) * kd, s);
  if (e != cudaSuccess) return e;
  if (bnd.lo) {
    e = launch_pdl(permute_bounds_kernel, dim3((unsigned)n_tiles(n)), dim3(TILE), 0, s, rec, n, S, dp,
                   (const int32_t*)perm, rec_sorted, inv, bnd.lo, bnd.hi, bnd.maxnorm, bnd.blk);
    if (e != cudaSuccess) return e;
  } else {
    permute_kernel<<<blocks, 256, 0, s>>>(rec, n, S, perm, rec_sorted, inv);
  }
  return cudaGetLastError();
}

}  // namespace ds
