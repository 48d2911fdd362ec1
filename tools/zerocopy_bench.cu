// Host<->device transfer paths at the C2 sizes (3.2 MB float64 points in, 1.6 MB
// int64 labels out): copy engine (cudaMemcpyAsync from/to page-locked memory) vs
// SM loads/stores straight to mapped page-locked host memory (zero copy).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/zc tools/zerocopy_bench.cu && /tmp/zc
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CK(x)                                                                \
  do {                                                                       \
    cudaError_t e_ = (x);                                                    \
    if (e_ != cudaSuccess) {                                                 \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
      exit(1);                                                               \
    }                                                                        \
  } while (0)

__global__ void read_host(const double2* __restrict__ src, size_t n2, float2* __restrict__ dst) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    const double2 v = src[i];
    dst[i] = make_float2((float)v.x, (float)v.y);
  }
}
// unrolled: 4 independent loads in flight per thread
__global__ void read_host4(const double2* __restrict__ src, size_t n2, float2* __restrict__ dst) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += 4 * stride) {
    double2 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = i + k * stride < n2 ? src[i + k * stride] : make_double2(0, 0);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < n2) dst[i + k * stride] = make_float2((float)v[k].x, (float)v[k].y);
  }
}
__global__ void write_host(const int* __restrict__ src, size_t n, long long* __restrict__ dst) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void write_host2(const int* __restrict__ src, size_t n, longlong2* __restrict__ dst) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; 2 * i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = make_longlong2(src[2 * i], src[2 * i + 1]);
}

int main(int argc, char** argv) {
  size_t npts = argc > 1 ? (size_t)atol(argv[1]) : 200000;
  const size_t in_bytes = npts * 2 * 8, out_bytes = npts * 8;
  double* h_in;
  long long* h_out;
  // page-locked the way the product does it: cudaHostRegister of a malloc'd buffer (PointSet)
  h_in = (double*)aligned_alloc(4096, (in_bytes + 4095) / 4096 * 4096);
  memset(h_in, 0, in_bytes);
  CK(cudaHostRegister(h_in, in_bytes, cudaHostRegisterDefault));
  CK(cudaMallocHost((void**)&h_out, out_bytes));
  void *d_in, *d_f, *d_i, *d_out;
  CK(cudaMalloc(&d_in, in_bytes));
  CK(cudaMalloc(&d_f, npts * 8));
  CK(cudaMalloc(&d_i, npts * 4));
  CK(cudaMemset(d_i, 0, npts * 4));
  CK(cudaMalloc(&d_out, out_bytes));
  double2* m_in;
  long long* m_out;
  CK(cudaHostGetDevicePointer((void**)&m_in, h_in, 0));
  CK(cudaHostGetDevicePointer((void**)&m_out, h_out, 0));
  printf("mapped pointers equal host pointers: in %d out %d\n", (void*)m_in == (void*)h_in,
         (void*)m_out == (void*)h_out);
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto timeit = [&](const char* what, size_t bytes, auto&& f) {
    for (int w = 0; w < 5; ++w) f();
    float best = 1e9, sum = 0;
    const int R = 50;
    for (int r = 0; r < R; ++r) {
      CK(cudaEventRecord(e0, s));
      f();
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
      sum += ms;
    }
    printf("%-44s %8.1f us best %8.1f us mean  %6.1f GB/s\n", what, best * 1e3, sum / R * 1e3,
           bytes / (best * 1e-3) / 1e9);
  };
  timeit("H2D memcpy (registered)", in_bytes,
         [&] { CK(cudaMemcpyAsync(d_in, h_in, in_bytes, cudaMemcpyHostToDevice, s)); });
  for (int mult : {1, 2, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof nm, "zero-copy read, grid %dx%d", mult, sms);
    timeit(nm, in_bytes, [&] { read_host<<<sms * mult, 256, 0, s>>>(m_in, npts, (float2*)d_f); });
    snprintf(nm, sizeof nm, "zero-copy read x4, grid %dx%d", mult, sms);
    timeit(nm, in_bytes, [&] { read_host4<<<sms * mult, 256, 0, s>>>(m_in, npts, (float2*)d_f); });
  }
  timeit("D2H memcpy (cudaMallocHost)", out_bytes,
         [&] { CK(cudaMemcpyAsync(h_out, d_out, out_bytes, cudaMemcpyDeviceToHost, s)); });
  for (int mult : {1, 2, 4}) {
    char nm[64];
    snprintf(nm, sizeof nm, "zero-copy write i64, grid %dx%d", mult, sms);
    timeit(nm, out_bytes, [&] { write_host<<<sms * mult, 256, 0, s>>>((int*)d_i, npts, m_out); });
    snprintf(nm, sizeof nm, "zero-copy write 2xi64, grid %dx%d", mult, sms);
    timeit(nm, out_bytes,
           [&] { write_host2<<<sms * mult, 256, 0, s>>>((int*)d_i, npts, (longlong2*)m_out); });
  }
  timeit("device write i64 (no host)", out_bytes,
         [&] { write_host<<<sms * 2, 256, 0, s>>>((int*)d_i, npts, (long long*)d_out); });
  return 0;
}
