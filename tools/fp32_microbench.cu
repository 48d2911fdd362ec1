// Inner-loop formulations of the 2-D algebraic eps test, timed on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o fp32_microbench fp32_microbench.cu
// Every variant must produce the same neighbour counts as V0 (checked); the
// output is pairs/s and FP32 lane-op efficiency against 128 lanes/SM/clk.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

constexpr int TILE = 512, NT = 128, KP = 4;

__device__ __forceinline__ uint32_t push_sign(uint32_t acc, float e) {
  return __funnelshift_l(__float_as_uint(e), acc, 1);
}

// V0: scalar ops, e = eps - d, sign bit via funnel shift
// V1: scalar ops, FSETP compare
// V2: dimension-packed FMUL2 + scalar cross add + FADD2 over two lane points
// V3: V2 arithmetic with FSETP compare
template <int V>
__global__ void __launch_bounds__(NT, 4) kern(const float4* __restrict__ rec, int n, float eps,
                                              int* __restrict__ cnt, int reps) {
  __shared__ float4 sp[TILE];
  const int tid = threadIdx.x;
  const int a = blockIdx.x % (n / TILE);
  float X[KP], Y[KP], T[KP], NT_[KP];
  for (int k = 0; k < KP; ++k) {
    const float4 r = rec[a * TILE + tid + NT * k];
    X[k] = __fadd_rn(r.x, r.x);
    Y[k] = __fadd_rn(r.y, r.y);
    T[k] = r.z;
    NT_[k] = -r.z;
  }
  float2 XY[KP], NT2[KP / 2];
  for (int k = 0; k < KP; ++k) XY[k] = make_float2(X[k], Y[k]);
  for (int k = 0; k < KP; k += 2) NT2[k / 2] = make_float2(NT_[k], NT_[k + 1]);
  int c[KP] = {0, 0, 0, 0};
  for (int rep = 0; rep < reps; ++rep) {
    for (int b = 0; b < n / TILE; ++b) {
      __syncthreads();
      for (int k = 0; k < KP; ++k) {
        float4 r = rec[b * TILE + tid + NT * k];
        if (V == 4) r.w = -r.z;
        sp[tid + NT * k] = r;
      }
      __syncthreads();
      for (int jw = 0; jw < TILE / 32; ++jw) {
        uint32_t acc[KP] = {0, 0, 0, 0};
#pragma unroll 4
        for (int jj = 0; jj < 32; ++jj) {
          const float4 p = sp[jw * 32 + jj];
          if (V == 0 || V == 1) {
#pragma unroll
            for (int k = 0; k < KP; ++k) {
              const float cr = __fadd_rn(__fmul_rn(X[k], p.x), __fmul_rn(Y[k], p.y));
              const float d = __fsub_rn(__fadd_rn(T[k], p.z), cr);
              if (V == 0) acc[k] = push_sign(acc[k], __fsub_rn(eps, d));
              else acc[k] = (acc[k] << 1) | (d <= eps ? 0u : 1u);
            }
          } else if (V == 4) {
            // V2 with pre-packed operands: smem record (x, y, -P, -P), lane pairs {2x, 2y}
            const float2 xy = make_float2(p.x, p.y);
            const float2 nP = make_float2(p.w, p.w);
            const float2 ep = make_float2(eps, eps);
#pragma unroll
            for (int k = 0; k < KP; k += 2) {
              const float2 m0 = __fmul2_rn(XY[k], xy);
              const float2 m1 = __fmul2_rn(XY[k + 1], xy);
              const float2 cc = make_float2(__fadd_rn(m0.x, m0.y), __fadd_rn(m1.x, m1.y));
              const float2 ntp = __fadd2_rn(NT2[k / 2], nP);
              const float2 nd = __fadd2_rn(cc, ntp);
              const float2 e = __fadd2_rn(ep, nd);
              acc[k] = push_sign(acc[k], e.x);
              acc[k + 1] = push_sign(acc[k + 1], e.y);
            }
          } else {
            const float2 xy = make_float2(p.x, p.y);
            const float2 nP = make_float2(-p.z, -p.z);
            const float2 ep = make_float2(eps, eps);
#pragma unroll
            for (int k = 0; k < KP; k += 2) {
              const float2 m0 = __fmul2_rn(make_float2(X[k], Y[k]), xy);
              const float2 m1 = __fmul2_rn(make_float2(X[k + 1], Y[k + 1]), xy);
              const float2 cc = make_float2(__fadd_rn(m0.x, m0.y), __fadd_rn(m1.x, m1.y));
              const float2 ntp = __fadd2_rn(make_float2(NT_[k], NT_[k + 1]), nP);  // -(T+P)
              const float2 nd = __fadd2_rn(cc, ntp);                                 // -(tp - c)
              if (V == 2) {
                const float2 e = __fadd2_rn(ep, nd);                                 // eps - d
                acc[k] = push_sign(acc[k], e.x);
                acc[k + 1] = push_sign(acc[k + 1], e.y);
              } else {
                acc[k] = (acc[k] << 1) | (-nd.x <= eps ? 0u : 1u);
                acc[k + 1] = (acc[k + 1] << 1) | (-nd.y <= eps ? 0u : 1u);
              }
            }
          }
        }
        for (int k = 0; k < KP; ++k) c[k] += __popc(~acc[k]);
      }
    }
  }
  for (int k = 0; k < KP; ++k) atomicAdd(&cnt[a * TILE + tid + NT * k], c[k]);
}

template <int V>
double run(const float4* d_rec, int n, float eps, int* d_cnt, std::vector<int>& out, int reps,
           int blocks_per_tile) {
  cudaMemset(d_cnt, 0, n * 4);
  const int grid = (n / TILE) * blocks_per_tile;
  kern<V><<<grid, NT>>>(d_rec, n, eps, d_cnt, 1);  // warm
  cudaDeviceSynchronize();
  cudaMemset(d_cnt, 0, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<V><<<grid, NT>>>(d_rec, n, eps, d_cnt, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  out.resize(n);
  cudaMemcpy(out.data(), d_cnt, n * 4, cudaMemcpyDeviceToHost);
  return ms;
}

int main() {
  const int n = 16384;
  std::vector<float4> h(n);
  srand(7);
  for (int i = 0; i < n; ++i) {
    const float x = (float)rand() / RAND_MAX * 40.f, y = (float)rand() / RAND_MAX * 40.f;
    volatile float xx = x * x, yy = y * y;  // separately rounded norm
    h[i] = make_float4(x, y, xx + yy, 0.f);
  }
  float4* d_rec;
  int* d_cnt;
  cudaMalloc(&d_rec, n * 16);
  cudaMalloc(&d_cnt, n * 4);
  cudaMemcpy(d_rec, h.data(), n * 16, cudaMemcpyHostToDevice);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const float eps = 0.5f;
  const int reps = 8;
  // each block handles one row tile against all columns; replicate blocks for occupancy
  const int bpt = 4 * sms / (n / TILE) + 1;
  std::vector<int> ref, got;
  const double pairs = (double)n * n * reps * bpt;
  double ms0 = run<0>(d_rec, n, eps, d_cnt, ref, reps, bpt);
  printf("sms=%d clock_khz=%d bpt=%d\n", sms, clk, bpt);
  auto report = [&](const char* name, double ms, bool same) {
    const double pps = pairs / (ms * 1e-3);
    const double lanes = (double)sms * 128 * clk * 1e3;
    printf("%-34s %8.3f ms  %7.3f Tpair/s  5-op eff %5.1f%%  %s\n", name, ms, pps / 1e12,
           100.0 * pps * 5 / lanes, same ? "counts==V0" : "COUNTS DIFFER");
  };
  report("V0 scalar, sign-bit SHF", ms0, true);
  double ms;
  ms = run<1>(d_rec, n, eps, d_cnt, got, reps, bpt);
  report("V1 scalar, FSETP", ms, got == ref);
  ms = run<2>(d_rec, n, eps, d_cnt, got, reps, bpt);
  report("V2 packed f32x2, sign-bit SHF", ms, got == ref);
  ms = run<3>(d_rec, n, eps, d_cnt, got, reps, bpt);
  report("V3 packed f32x2, FSETP", ms, got == ref);
  ms = run<4>(d_rec, n, eps, d_cnt, got, reps, bpt);
  report("V4 packed f32x2, pre-packed operands", ms, got == ref);
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
