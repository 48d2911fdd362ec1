// The reference's float64 semantic oracle `serial_dbscan` (pkg/src/densescan/oracle.py:48-111)
// on the device, for the CLI's `--variant serial` and the `bench` equivalence gate
// (cli.py:94-122, 152-234).
//
// Stage 1+2 in one kernel: each thread owns one 32-column word of one row and
// evaluates the reference's float64 row formula in its order,
//   dx = x_col - x_row;  d2 = dx*dx;  d2 += dy*dy;  d2 += dz*dz;   (oracle.py:58-69)
// (left to right over further dimensions), every operation one IEEE round-to-nearest
// double op (__dsub_rn/__dmul_rn/__dadd_rn, no FMA), then in_range = d2 <= eps_sq in
// float64 (oracle.py:71-79). Words are stored MSB-first (bit 31 - t <-> column 32 w + t,
// the byte-swapped packbits layout) and counted into the row's neighbour count.
// Stage 3 reuses the dense union-find (ds_merge.cu union_dense_kernel): BFS over
// core-core pairs = connected components of the symmetric relation, borders to their
// lowest-indexed in-range core (oracle.py:98-101), canonical ids.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ds_internal.cuh"

namespace ds {
namespace {

constexpr int SER_T = 256;

// coords: float64 n x d, point-major (the PointSet layout); soa: d x n copy
__global__ void to_soa_kernel(const double* __restrict__ coords, int64_t n, int d,
                              double* __restrict__ soa) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n * d;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / d;
    const int j = (int)(k - i * d);
    soa[(int64_t)j * n + i] = coords[k];
  }
}

__global__ void __launch_bounds__(SER_T) serial_words_kernel(const double* __restrict__ soa,
                                                             int64_t n, int d, double eps_sq,
                                                             uint32_t* __restrict__ bits,
                                                             int64_t stride,
                                                             int32_t* __restrict__ cnt) {
  const int64_t total = n * stride;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / stride;
    const int64_t w = k - i * stride;
    uint32_t word = 0;
    for (int t = 0; t < 32; ++t) {
      const int64_t j = w * 32 + t;
      if (j >= n) break;
      double acc = 0.0;
      for (int c = 0; c < d; ++c) {
        const double* x = soa + (int64_t)c * n;
        const double dx = __dsub_rn(x[j], x[i]);
        const double sq = __dmul_rn(dx, dx);
        acc = c == 0 ? sq : __dadd_rn(acc, sq);
      }
      if (acc <= eps_sq) word |= 0x80000000u >> t;
    }
    bits[k] = word;
    if (word) atomicAdd(&cnt[i], __popc(word));
  }
}

}  // namespace

cudaError_t launch_serial_words(const double* coords, int64_t n, int d, double eps_sq,
                                double* soa, uint32_t* bits, int64_t stride, int32_t* cnt,
                                cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)n * 4, s);
  if (e != cudaSuccess) return e;
  to_soa_kernel<<<sms * 4, 256, 0, s>>>(coords, n, d, soa);
  serial_words_kernel<<<sms * 16, SER_T, 0, s>>>(soa, n, d, eps_sq, bits, stride, cnt);
  return cudaGetLastError();
}

}  // namespace ds
