// Issue/pipe throughput of the instruction classes the eps-tile inner loop uses, on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_mb tools/pipe_microbench.cu
// Each warp runs 8 independent chains of one instruction mix; the result is warp-
// instructions per cycle per SM sub-partition (scheduler) and FP32 lane-ops per
// cycle per SM, for 4 and 8 warps per scheduler.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define ITERS 2048

template <int M>
__global__ void mix(float* out, long long* cyc, float a0) {
  float r[8];
  float2 p[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) {
    r[i] = a0 + threadIdx.x * 1e-3f + i;
    u[i] = threadIdx.x * 7 + i;
    p[i] = make_float2(r[i], r[i] + 0.5f);
  }
  const float2 e2 = make_float2(0.25f, 0.125f);
  const float e = 0.25f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (M == 0) {  // FADD
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(r[i]) : "f"(e));
      } else if (M == 1) {  // FADD2 (f32x2)
        p[i] = __fadd2_rn(p[i], e2);
      } else if (M == 2) {  // FMUL2
        p[i] = __fmul2_rn(p[i], e2);
      } else if (M == 3) {  // FFMA
        asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(r[i]) : "f"(e));
      } else if (M == 4) {  // FSETP + SELP (compare -> bit)
        asm volatile("{.reg .pred p; setp.le.f32 p, %1, %2; selp.b32 %0, 1, 0, p;}"
                     : "=r"(u[i]) : "f"(r[i]), "f"(e));
        r[i] = __uint_as_float(u[i]);
      } else if (M == 5) {  // SHF funnel
        asm volatile("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(u[i]) : "r"(u[(i + 3) & 7]));
      } else if (M == 6) {  // FADD2 + SHF interleaved
        p[i] = __fadd2_rn(p[i], e2);
        asm volatile("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(u[i]) : "r"(u[(i + 3) & 7]));
      } else if (M == 7) {  // FADD + SHF interleaved
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(r[i]) : "f"(e));
        asm volatile("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(u[i]) : "r"(u[(i + 3) & 7]));
      } else if (M == 8) {  // FADD + FADD2 interleaved
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(r[i]) : "f"(e));
        p[i] = __fadd2_rn(p[i], e2);
      } else if (M == 9) {  // FSETP only (predicate result consumed by a predicated op rarely)
        asm volatile("{.reg .pred p; setp.le.f32 p, %1, %2; @p add.u32 %0, %0, 1;}"
                     : "+r"(u[i]) : "f"(r[i]), "f"(e));
      } else if (M == 10) {  // LOP3
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]), "r"(u[(i + 2) & 7]));
      } else if (M == 11) {  // IADD3-like integer add
        asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
      }
    }
  }
  const long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += r[i] + (float)u[i] + p[i].x + p[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0;
}

// instrs per inner step per warp, FP32 lane-ops per lane per step
static const char* NAMES[] = {"FADD", "FADD2", "FMUL2", "FFMA", "FSETP+SEL", "SHF", "FADD2+SHF",
                              "FADD+SHF", "FADD+FADD2", "FSETP+@IADD", "LOP3", "IADD"};
static const int INSTR[] = {1, 1, 1, 1, 2, 1, 2, 2, 2, 2, 1, 1};
static const int FPOPS[] = {1, 2, 2, 1, 0, 0, 2, 1, 3, 0, 0, 0};

template <int M>
void run(int sms, int warps_per_sched) {
  const int threads = 32 * 4 * warps_per_sched;
  float* out;
  long long* cyc;
  cudaMalloc(&out, sms * threads * 4);
  cudaMalloc(&cyc, sms * threads / 32 * 8);
  mix<M><<<sms, threads>>>(out, cyc, 1.0f);
  mix<M><<<sms, threads>>>(out, cyc, 1.0f);
  cudaDeviceSynchronize();
  long long h[8192];
  const int nw = sms * threads / 32;
  cudaMemcpy(h, cyc, nw * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < nw; ++i) mx = h[i] > mx ? h[i] : mx;
  // per scheduler: warps_per_sched warps x ITERS x 8 steps x INSTR
  const double instr = (double)warps_per_sched * ITERS * 8 * INSTR[M];
  const double lane_ops = 4.0 * warps_per_sched * ITERS * 8 * 32 * FPOPS[M];
  printf("%-12s warps/sched=%d  issue %.3f warp-instr/clk/sched   FP32 %.1f lane-ops/clk/SM\n",
         NAMES[M], warps_per_sched, instr / mx, lane_ops / mx);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8}) {
    run<0>(sms, w); run<1>(sms, w); run<2>(sms, w); run<3>(sms, w);
    run<4>(sms, w); run<5>(sms, w); run<6>(sms, w); run<7>(sms, w);
    run<8>(sms, w); run<9>(sms, w); run<10>(sms, w); run<11>(sms, w);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
