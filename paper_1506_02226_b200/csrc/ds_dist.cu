// The reference's materialising ladder on sm_100a.
//
// Replaces dist_baseline / dist_soa / dist_tiled (pkg/src/densescan/kernels.py:153-281,
// all four rungs compute the same direct-formula values, kernels.py:21-25 and
// _direct_block 197-210) and build_clusters_from_dist (kernels.py:284-308).
//
//   dist_kernel       out[i][j] = ((x_j - x_i)^2 + (y_j - y_i)^2) + (z_j - z_i)^2 ...
//                     in float32, every op separately rounded (no FMA), the d-dim form
//                     extended left to right. HBM-write bound: 4 bytes per pair; each
//                     thread owns 4 consecutive columns (one float4 store per row; one
//                     column above 16-D) and walks DIST_ROWS rows, so the column
//                     records are read once per DIST_ROWS rows.
//   threshold_kernel  bits (numpy packbits layout: MSB-first bytes, ceil(n/8) per row)
//                     of d <= eps32 (NaN -> 0, like numpy) and int64 row counts.
//                     HBM-read bound: 4 bytes per pair.
// The matrix rows on the device use a pitch of roundup4(n) floats.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ds_internal.cuh"

namespace ds {
namespace {

constexpr int DIST_THREADS = 256;
constexpr int DIST_ROWS = 16;

// CPT columns per thread: 4 (one float4 store per row) up to 16-D; wider records keep
// one column per thread so the column records stay in registers
template <int D>
struct DistGeo {
  static constexpr int CPT = D <= 16 ? 4 : 1;
};

template <int D>
__global__ void __launch_bounds__(DIST_THREADS) dist_kernel(const float* __restrict__ rec, int S,
                                                            int64_t n, int64_t row0, int64_t rows,
                                                            int64_t pitch, float* __restrict__ out) {
  constexpr int CPT = DistGeo<D>::CPT;
  const int64_t j0 = ((int64_t)blockIdx.x * DIST_THREADS + threadIdx.x) * CPT;
  if (j0 >= n) return;
  float cj[CPT][D];
#pragma unroll
  for (int t = 0; t < CPT; ++t) {
    const int64_t j = j0 + t < n ? j0 + t : n - 1;
#pragma unroll
    for (int q = 0; q < D; ++q) cj[t][q] = __ldg(rec + j * S + q);
  }
  const int64_t r_begin = (int64_t)blockIdx.y * DIST_ROWS;
  for (int r = 0; r < DIST_ROWS; ++r) {
    const int64_t il = r_begin + r;  // row within this launch's block
    if (il >= rows) break;
    const int64_t i = row0 + il;
    float ci[D];
#pragma unroll
    for (int q = 0; q < D; ++q) ci[q] = __ldg(rec + i * S + q);
    float v[CPT];
#pragma unroll
    for (int t = 0; t < CPT; ++t) {
      float dx = __fsub_rn(cj[t][0], ci[0]);  // column minus row (kernels.py:205)
      float acc = __fmul_rn(dx, dx);
#pragma unroll
      for (int q = 1; q < D; ++q) {
        dx = __fsub_rn(cj[t][q], ci[q]);
        acc = __fadd_rn(acc, __fmul_rn(dx, dx));
      }
      v[t] = acc;
    }
    float* dst = out + il * pitch + j0;
    if constexpr (CPT == 4) {
      *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);  // j0 + 3 < pitch
    } else {
      dst[0] = v[0];
    }
  }
}

// One CTA per row (grid-stride over rows): byte k of the row holds columns 8k..8k+7,
// column 8k+t at bit 7-t (np.packbits order).
__global__ void __launch_bounds__(256) threshold_kernel(const float* __restrict__ dist, int64_t n,
                                                        int64_t rows, int64_t pitch, float eps32,
                                                        uint8_t* __restrict__ bits,
                                                        int64_t* __restrict__ counts) {
  const int64_t rb = (n + 7) / 8;
  __shared__ int warp_cnt[8];
  for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
    const float* row = dist + i * pitch;
    int cnt = 0;
    for (int64_t k = threadIdx.x; k < rb; k += blockDim.x) {
      const int64_t c0 = k * 8;
      uint32_t byte = 0;
      if (c0 + 8 <= n) {
        const float4 a = *reinterpret_cast<const float4*>(row + c0);
        const float4 b = *reinterpret_cast<const float4*>(row + c0 + 4);
        const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int t = 0; t < 8; ++t) byte |= (x[t] <= eps32 ? 1u : 0u) << (7 - t);
      } else {
        for (int t = 0; c0 + t < n; ++t) byte |= (row[c0 + t] <= eps32 ? 1u : 0u) << (7 - t);
      }
      bits[i * rb + k] = (uint8_t)byte;
      cnt += __popc(byte);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if ((threadIdx.x & 31) == 0) warp_cnt[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t tot = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += warp_cnt[w];
      counts[i] = tot;
    }
    __syncthreads();
  }
}

template <int D>
cudaError_t launch_dist_d(const float* rec, int S, int64_t n, int64_t row0, int64_t rows,
                          int64_t pitch, float* out, cudaStream_t s) {
  constexpr int CPT = DistGeo<D>::CPT;
  const dim3 grid((unsigned)((n + CPT * DIST_THREADS - 1) / (CPT * DIST_THREADS)),
                  (unsigned)((rows + DIST_ROWS - 1) / DIST_ROWS));
  dist_kernel<D><<<grid, DIST_THREADS, 0, s>>>(rec, S, n, row0, rows, pitch, out);
  return cudaGetLastError();
}

}  // namespace

int64_t dist_pitch(int64_t n) { return (n + 3) / 4 * 4; }

cudaError_t launch_dist(const float* rec, int64_t n, int d, int64_t row0, int64_t rows,
                        float* out, cudaStream_t s) {
  const int S = rec_stride(d);
  const int64_t pitch = dist_pitch(n);
  switch (padded_dim(d)) {
    case 1: return launch_dist_d<1>(rec, S, n, row0, rows, pitch, out, s);
    case 2: return launch_dist_d<2>(rec, S, n, row0, rows, pitch, out, s);
    case 3: return launch_dist_d<3>(rec, S, n, row0, rows, pitch, out, s);
    case 4: return launch_dist_d<4>(rec, S, n, row0, rows, pitch, out, s);
    case 8: return launch_dist_d<8>(rec, S, n, row0, rows, pitch, out, s);
    case 16: return launch_dist_d<16>(rec, S, n, row0, rows, pitch, out, s);
    case 32: return launch_dist_d<32>(rec, S, n, row0, rows, pitch, out, s);
    default: return launch_dist_d<64>(rec, S, n, row0, rows, pitch, out, s);
  }
}

cudaError_t launch_threshold(const float* dist, int64_t n, int64_t rows, float eps32, uint8_t* bits,
                             int64_t* counts, cudaStream_t s) {
  int64_t grid = rows < 148 * 16 ? rows : 148 * 16;
  if (grid < 1) grid = 1;
  threshold_kernel<<<(unsigned)grid, 256, 0, s>>>(dist, n, rows, dist_pitch(n), eps32, bits, counts);
  return cudaGetLastError();
}

}  // namespace ds
