// The Warshall backend's building blocks on the device:
//   build_core_adjacency  (reference merge.py:179-188): the neighbourhood matrix
//                         restricted to core rows and columns, m x ceil(m/8) packbits;
//   warshall_closure      (merge.py:191-215): its transitive closure.
//
// Bit matrices are held as rows of 32-bit words, bit 31 - t <-> column 32 w + t (the
// byte-swapped packbits layout, ds_merge.cu bswap_kernel), padded to `stride` words.
//
// The closure is the blocked form of the Warshall recurrence with 32-column blocks:
// for block K (pivots k0 .. k0+31), after the phase every entry (i, j) holds "j is
// reachable from i through intermediates in blocks <= K" — exactly what the
// reference's pivot loop holds after pivot k0+31, so after the last phase the
// matrices are identical (the transitive closure R+ of the input relation is unique;
// no symmetry or reflexivity is assumed). One phase:
//   A  (one CTA)  D+ = closure of the 32 x 32 diagonal block (sequential pivots, one
//                 warp); row panel R[r][J] = C[r][J] | OR_{t in D+[r]} C[k0+t][J] for the
//                 32 rows r of block K (their paths leave K through a direct edge).
//   W  (grid)     column word of every row i: W[i] = C[i][K] | OR_{t in C[i][K]} D+[t].
//   B  (grid)     every other row: C[i][J] |= OR_{t in W[i]} R[k0+t][J], C[i][K] = W[i].
// Work is O(m^3 / 32) word operations; rows with an empty column word skip the phase.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ds_internal.cuh"

namespace ds {
namespace {

constexpr int PANEL_T = 1024;

__device__ __forceinline__ uint32_t col_bit(int t) { return 0x80000000u >> t; }

// flags[i] = valid[i] (int32, for the exclusive scan that numbers the cores)
__global__ void valid_flags_kernel(const uint8_t* __restrict__ valid, int64_t n,
                                   int32_t* __restrict__ flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = valid[i] ? 1 : 0;
}

// core_indices[rank] = i for every core point i (ascending: rank = exclusive scan)
__global__ void core_scatter_kernel(const uint8_t* __restrict__ valid,
                                    const int32_t* __restrict__ rank, int64_t n,
                                    int32_t* __restrict__ ci32, int64_t* __restrict__ ci64) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (valid[i]) {
      ci32[rank[i]] = (int32_t)i;
      ci64[rank[i]] = i;
    }
}

// One warp per output row r: lane t of output word w reads the bit of column
// core_indices[32 w + t] in row core_indices[r]; the ballot is the output word.
__global__ void core_gather_kernel(const uint32_t* __restrict__ bits, int64_t stride_n,
                                   const int32_t* __restrict__ ci, int64_t m,
                                   uint32_t* __restrict__ adj, int64_t stride_m) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < m;
       r += warps) {
    const uint32_t* row = bits + (int64_t)ci[r] * stride_n;
    uint32_t* out = adj + r * stride_m;
    for (int64_t w = 0; w < stride_m; ++w) {
      const int64_t c = w * 32 + lane;
      bool bit = false;
      if (c < m) {
        const int32_t j = ci[c];
        bit = (row[j >> 5] & col_bit(j & 31)) != 0;
      }
      const uint32_t word = __brev(__ballot_sync(0xffffffffu, bit));  // lane t -> bit 31-t
      if (lane == 0) out[w] = word;
    }
  }
}

// Phase part A: diagonal closure D+ (-> dplus[32]) and the row panel of block K.
__global__ void __launch_bounds__(PANEL_T) closure_panel_kernel(uint32_t* __restrict__ C,
                                                                int64_t m, int64_t stride,
                                                                int64_t K,
                                                                uint32_t* __restrict__ dplus) {
  __shared__ uint32_t sd[32];
  const int64_t k0 = K * 32;
  const int rows = (int)((m - k0) < 32 ? (m - k0) : 32);
  if (threadIdx.x < 32) {
    const int t = threadIdx.x;
    uint32_t w = t < rows ? C[(k0 + t) * stride + K] : 0u;
    // Warshall over the block's pivots, in order: row t absorbs row p if t -> p
    for (int p = 0; p < rows; ++p) {
      const uint32_t wp = __shfl_sync(0xffffffffu, w, p);
      if (w & col_bit(p)) w |= wp;
    }
    sd[t] = w;
    if (t < rows) dplus[t] = w;
  }
  __syncthreads();
  for (int64_t J = threadIdx.x; J < stride; J += blockDim.x) {
    if (J == K) {
      for (int r = 0; r < rows; ++r) C[(k0 + r) * stride + J] = sd[r];
      continue;
    }
    uint32_t v[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) v[t] = t < rows ? C[(k0 + t) * stride + J] : 0u;
    for (int r = 0; r < rows; ++r) {
      uint32_t acc = v[r];
      const uint32_t dr = sd[r];
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (dr & col_bit(t)) acc |= v[t];
      C[(k0 + r) * stride + J] = acc;
    }
  }
}

// Phase part W: the updated column-block word of every row outside block K.
__global__ void closure_colword_kernel(const uint32_t* __restrict__ C, int64_t m, int64_t stride,
                                       int64_t K, const uint32_t* __restrict__ dplus,
                                       uint32_t* __restrict__ W) {
  __shared__ uint32_t sd[32];
  const int64_t k0 = K * 32;
  const int rows = (int)((m - k0) < 32 ? (m - k0) : 32);
  if (threadIdx.x < 32) sd[threadIdx.x] = threadIdx.x < rows ? dplus[threadIdx.x] : 0u;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i >= k0 && i < k0 + rows) continue;
    const uint32_t c = C[i * stride + K];
    uint32_t w = c;
    for (uint32_t rest = c; rest;) {
      const int t = __clz(rest);  // highest set bit <-> lowest column index t
      w |= sd[t];
      rest &= ~col_bit(t);
    }
    W[i] = w;
  }
}

// Phase part B: one warp per row outside block K; lanes stride over the words.
__global__ void closure_update_kernel(uint32_t* __restrict__ C, int64_t m, int64_t stride,
                                     int64_t K, const uint32_t* __restrict__ W) {
  const int lane = threadIdx.x & 31;
  const int64_t k0 = K * 32;
  const int64_t rows_end = k0 + 32 < m ? k0 + 32 : m;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < m;
       i += warps) {
    if (i >= k0 && i < rows_end) continue;
    const uint32_t w = W[i];
    if (w == 0) continue;
    uint32_t* row = C + i * stride;
    for (int64_t J = lane; J < stride; J += 32) {
      if (J == K) {
        row[J] = w;
        continue;
      }
      uint32_t acc = row[J];
      for (uint32_t rest = w; rest;) {
        const int t = __clz(rest);
        acc |= C[(k0 + t) * stride + J];
        rest &= ~col_bit(t);
      }
      row[J] = acc;
    }
  }
}

}  // namespace
}  // namespace ds

namespace ds {

static unsigned grid_for(int64_t work, int per_block) {
  int64_t b = (work + per_block - 1) / per_block;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t launch_core_index(const uint8_t* valid, int64_t n, int32_t* flags, int32_t* partials,
                              int32_t* total, int32_t* ci32, int64_t* ci64, cudaStream_t s) {
  valid_flags_kernel<<<grid_for(n, 256), 256, 0, s>>>(valid, n, flags);
  cudaError_t e = launch_exclusive_scan(flags, n, partials, total, s);
  if (e != cudaSuccess) return e;
  core_scatter_kernel<<<grid_for(n, 256), 256, 0, s>>>(valid, flags, n, ci32, ci64);
  return cudaGetLastError();
}

cudaError_t launch_core_gather(const uint32_t* bits, int64_t stride_n, const int32_t* ci, int64_t m,
                               uint32_t* adj, int64_t stride_m, cudaStream_t s) {
  if (m < 1) return cudaSuccess;
  core_gather_kernel<<<grid_for(m, 8), 256, 0, s>>>(bits, stride_n, ci, m, adj, stride_m);
  return cudaGetLastError();
}

cudaError_t launch_closure(uint32_t* C, int64_t m, int64_t stride, uint32_t* dplus, uint32_t* W,
                           cudaStream_t s) {
  const int64_t blocks = (m + 31) / 32;
  for (int64_t K = 0; K < blocks; ++K) {
    closure_panel_kernel<<<1, PANEL_T, 0, s>>>(C, m, stride, K, dplus);
    closure_colword_kernel<<<grid_for(m, 256), 256, 0, s>>>(C, m, stride, K, dplus, W);
    closure_update_kernel<<<grid_for(m, 8), 256, 0, s>>>(C, m, stride, K, W);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ds
