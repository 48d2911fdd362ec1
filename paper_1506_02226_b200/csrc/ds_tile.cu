// Stage 1+2 of the densescan hot path on sm_100a: the fused eps-tile kernel.
//
// Replaces the reference's fused_build / fused_build_algebraic
// (pkg/src/densescan/kernels.py:311-442): every pair (i, j) is tested
// against eps^2 in float32 with the reference's operation order and
// rounding, the distance matrix is never stored, and the result leaves the
// kernel as bit-packed 32-bit adjacency words plus neighbour counts.
//
// Work decomposition. Points are cut into tiles of TILE=512. The relation is
// exactly symmetric (both formulas are bitwise symmetric in (i, j), see
// DESIGN.md §2), so only tile pairs (a, b) with a <= b are evaluated: one
// "item" = one tile pair = 262,144 pair evaluations. A persistent grid pulls
// items from an atomic counter. Per item:
//   * tile b (the broadcast side) is staged into shared memory with a TMA
//     bulk copy (cp.async.bulk, mbarrier completion), double-buffered so the
//     next item's copy overlaps this item's arithmetic;
//   * tile a (the lane side) lives in registers: each thread owns KPT points
//     and keeps 2*c (algebraic) or c (direct) plus the norm T;
//   * every thread walks the 512 staged points; for each pair it computes
//     d2 in exact reference order: every operation a separately rounded
//     f32 op (never contracted into an FMA; tests/test_sass_gate.py checks
//     the SASS). The FP32 pipe is the bound, so the arithmetic is issued as
//     packed f32x2 where the reference order allows it — products of two
//     dimensions in one FMUL2, T + P and the final subtraction of two lane
//     points in one FADD2 — which executes exactly the 2d+1 (algebraic) or
//     3d-1 (direct) FP32 lane-ops per pair and nothing else on that pipe;
//   * the compare is split between an FSETP on the ALU pipe and the sign bit
//     of fl(eps32 - d2) (see pack_bits) to balance the two pipes; 32 results
//     pack into one 32-bit word per lane point;
//   * words go to shared memory; the lane-side counts are popcounts of the
//     words, the broadcast-side counts a bit-sliced (carry-save) vertical
//     popcount of the same words; the non-zero words are appended to HBM for
//     stage 3 after a block-wide prefix scan, as one contiguous "chunk" per
//     tile pair: 8-byte records {word, row << 4 | column word} plus a chunk
//     entry {a, b, base, count}.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ds_internal.cuh"

namespace ds {
namespace {

// ---- PTX helpers: mbarrier + TMA bulk copy -------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "DS_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra DS_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- item <-> tile pair --------------------------------------------------------
__device__ __forceinline__ int64_t row_offset(int64_t a, int64_t T) {
  return a * T - a * (a - 1) / 2;
}
__device__ __forceinline__ void decode_item(int64_t q, int64_t T, int& a, int& b) {
  const double tt = 2.0 * (double)T + 1.0;
  int64_t r = (int64_t)floor((tt - sqrt(tt * tt - 8.0 * (double)q)) * 0.5);
  if (r < 0) r = 0;
  if (r > T - 1) r = T - 1;
  while (r + 1 <= T - 1 && row_offset(r + 1, T) <= q) ++r;
  while (r > 0 && row_offset(r, T) > q) --r;
  a = (int)r;
  b = (int)(r + (q - row_offset(r, T)));
}

// Diagonal tile: keep columns t >= rel (j >= i incl. the self pair; the self bit
// is needed by the reference-layout export and is a no-op for the merge).
__device__ __forceinline__ uint32_t diag_keep(int rel) {
  return rel <= 0 ? 0xffffffffu : (rel > 31 ? 0u : ((1u << (32 - rel)) - 1u));
}

// Item q -> tile pair: through the culled item list when one is given, else the
// dense upper-triangle enumeration.
__device__ __forceinline__ void item_tiles(const TileArgs& args, int64_t q, int64_t T, int& a,
                                           int& b) {
  if (args.item_list) {
    const uint32_t ab = args.item_list[q];
    a = (int)(ab >> 16);
    b = (int)(ab & 0xffffu);
  } else {
    decode_item(q, T, a, b);
  }
}

__device__ __forceinline__ uint32_t valid_mask(int m) {
  // bit (31 - t) <-> column t of the word; the first m columns are valid
  return m >= 32 ? 0xffffffffu : (m <= 0 ? 0u : (0xffffffffu << (32 - m)));
}

// ---- exact reference arithmetic ------------------------------------------------
// Algebraic (kernels.py:403-417): cross = ((X0*x0 + X1*x1) + ...), d2 = (T + P) - cross
// with X = 2c of the lane point; by symmetry the lane point may be the row or
// the column of the reference's matrix.
template <int D>
__device__ __forceinline__ float d2_algebraic(const float (&lv)[D], float lt, const float* xj,
                                              float pj) {
  float cross = __fmul_rn(lv[0], xj[0]);
#pragma unroll
  for (int c = 1; c < D; ++c) cross = __fadd_rn(cross, __fmul_rn(lv[c], xj[c]));
  return __fsub_rn(__fadd_rn(lt, pj), cross);
}
// Direct (kernels.py:197-210): d2 = ((dx0^2 + dx1^2) + ...), dx = col - row.
template <int D>
__device__ __forceinline__ float d2_direct(const float (&lv)[D], const float* xj) {
  float dx = __fsub_rn(xj[0], lv[0]);
  float acc = __fmul_rn(dx, dx);
#pragma unroll
  for (int c = 1; c < D; ++c) {
    dx = __fsub_rn(xj[c], lv[c]);
    acc = __fadd_rn(acc, __fmul_rn(dx, dx));
  }
  return acc;
}

// ---- lane points in packed form ------------------------------------------------
// ALG: v2[k][p] = {2c_{2p}, 2c_{2p+1}} (X = 2c is exact), t[k] = T = P_i.
// DIR: v2[k][p] = {-c_{2p}, -c_{2p+1}} so that x_j + (-x_i) == fl(x_j - x_i).
template <int D, int KP>
struct Lanes {
  static constexpr int DP = D / 2;
  static constexpr bool ODD = (D & 1) != 0;
  float2 v2[KP][DP > 0 ? DP : 1];
  float v1[KP];
  float t[KP];
};

// Squared distances of the KP lane points to staged point j (xj: its record,
// pj = P_j), in the reference's order with one rounding per operation.
template <int D, int F, int KP>
__device__ __forceinline__ void eval_d2(const Lanes<D, KP>& L, const float* xj, float pj,
                                        float (&d2)[KP]) {
  constexpr int DP = Lanes<D, KP>::DP;
  constexpr bool ODD = Lanes<D, KP>::ODD;
  if constexpr (F == DS_FORMULA_ALGEBRAIC) {
    // cross = ((X0*x0 + X1*x1) + X2*x2) + ...            (kernels.py:409-414)
    float c[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      float acc;
      if constexpr (DP > 0) {
        float2 m = __fmul2_rn(L.v2[k][0], make_float2(xj[0], xj[1]));
        acc = __fadd_rn(m.x, m.y);
#pragma unroll
        for (int q = 1; q < DP; ++q) {
          m = __fmul2_rn(L.v2[k][q], make_float2(xj[2 * q], xj[2 * q + 1]));
          acc = __fadd_rn(acc, m.x);
          acc = __fadd_rn(acc, m.y);
        }
        if constexpr (ODD) acc = __fadd_rn(acc, __fmul_rn(L.v1[k], xj[D - 1]));
      } else {
        acc = __fmul_rn(L.v1[k], xj[0]);
      }
      c[k] = acc;
    }
    // d2 = (T + P) - cross, two lane points per FADD2       (kernels.py:415-417)
    if constexpr (KP % 2 == 0) {
#pragma unroll
      for (int k = 0; k < KP; k += 2) {
        const float2 tp = __fadd2_rn(make_float2(L.t[k], L.t[k + 1]), make_float2(pj, pj));
        const float2 d = __fadd2_rn(tp, make_float2(-c[k], -c[k + 1]));
        d2[k] = d.x;
        d2[k + 1] = d.y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < KP; ++k) d2[k] = __fsub_rn(__fadd_rn(L.t[k], pj), c[k]);
    }
  } else {
    // d2 = ((dx0^2 + dx1^2) + dx2^2) + ..., dx = x_col - x_row  (kernels.py:197-210)
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      float acc;
      if constexpr (DP > 0) {
        float2 dx = __fadd2_rn(make_float2(xj[0], xj[1]), L.v2[k][0]);
        float2 sq = __fmul2_rn(dx, dx);
        acc = __fadd_rn(sq.x, sq.y);
#pragma unroll
        for (int q = 1; q < DP; ++q) {
          dx = __fadd2_rn(make_float2(xj[2 * q], xj[2 * q + 1]), L.v2[k][q]);
          sq = __fmul2_rn(dx, dx);
          acc = __fadd_rn(acc, sq.x);
          acc = __fadd_rn(acc, sq.y);
        }
        if constexpr (ODD) {
          const float e = __fadd_rn(xj[D - 1], L.v1[k]);
          acc = __fadd_rn(acc, __fmul_rn(e, e));
        }
      } else {
        const float e = __fadd_rn(xj[0], L.v1[k]);
        acc = __fmul_rn(e, e);
      }
      d2[k] = acc;
    }
  }
}

// How the KP predicates of one staged point become bits. The first KC lane points
// use an FSETP compare (ALU pipe, NaN-exact); the rest push the sign bit of
// fl(eps32 - d2) with a funnel shift (one more FP lane-op, one ALU op). With all
// operands finite, fl(eps32 - d2) < 0 <=> d2 > eps32 (round-to-nearest keeps the
// sign and x - x = +0), so the sign bit is exactly the out-of-range bit. Mixing
// the two balances the FP32 and ALU pipes; SAFE=false (inputs whose squares can
// overflow) compares every lane point.
template <int KP, bool SAFE>
struct Pack {
  static constexpr int KC = SAFE ? KP / 2 : KP;
};

template <int KP, bool SAFE>
__device__ __forceinline__ void pack_bits(const float (&d2)[KP], float eps32, int jj,
                                          uint32_t (&acc)[KP]) {
  constexpr int KC = Pack<KP, SAFE>::KC;
#pragma unroll
  for (int k = 0; k < KC; ++k) acc[k] |= (d2[k] <= eps32 ? 1u : 0u) << (31 - jj);
  if constexpr (KC < KP) {
    if constexpr ((KP - KC) % 2 == 0) {
#pragma unroll
      for (int k = KC; k < KP; k += 2) {
        const float2 e = __fadd2_rn(make_float2(eps32, eps32), make_float2(-d2[k], -d2[k + 1]));
        acc[k] = __funnelshift_l(__float_as_uint(e.x), acc[k], 1);
        acc[k + 1] = __funnelshift_l(__float_as_uint(e.y), acc[k + 1], 1);
      }
    } else {
#pragma unroll
      for (int k = KC; k < KP; ++k)
        acc[k] = __funnelshift_l(__float_as_uint(__fsub_rn(eps32, d2[k])), acc[k], 1);
    }
  }
}

template <int D>
struct Geo {
  static constexpr int KP = D <= 8 ? 4 : (D <= 32 ? 2 : 1);  // lane points per thread
  static constexpr int THREADS = TILE / KP;
  static constexpr int S = ((D + 1) + 3) / 4 * 4;           // floats per record
  static constexpr int NBUF = (2 * TILE * S * 4 <= 96 * 1024) ? 2 : 1;
  static constexpr int CHUNKS = THREADS / WPR;               // row chunks per word column
  static constexpr int ROWS = TILE / CHUNKS;                 // rows per chunk
  static constexpr int SL0 = ROWS == 64 ? 7 : (ROWS == 32 ? 6 : 5);  // slices per chunk
  static constexpr size_t SMEM = (size_t)NBUF * TILE * S * 4 + (size_t)WPR * BSTRIDE * 4;
};

// Bit-sliced add of a partner counter (10 slices) into ours.
__device__ __forceinline__ void sliced_add(uint32_t (&s)[10], const uint32_t (&o)[10]) {
  uint32_t carry = 0;
#pragma unroll
  for (int l = 0; l < 10; ++l) {
    const uint32_t a = s[l], b = o[l];
    s[l] = a ^ b ^ carry;
    carry = (a & b) | (carry & (a ^ b));
  }
}

template <int D, int F, bool SAFE>
__global__ void __launch_bounds__(Geo<D>::THREADS, (D <= 8 ? 4 : (D <= 32 ? 2 : 1)))
eps_tile_kernel(const TileArgs args) {
  using G = Geo<D>;
  constexpr int KP = G::KP;
  constexpr int NTH = G::THREADS;
  constexpr int S = G::S;
  constexpr int KC = Pack<KP, SAFE>::KC;

  if ((*args.unsafe_flag != 0) == SAFE) return;  // the other instantiation owns this input

  extern __shared__ __align__(128) unsigned char smem[];
  float* bc = reinterpret_cast<float*>(smem);
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem + (size_t)G::NBUF * TILE * S * 4);
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ long long item_sh[2];
  __shared__ unsigned int scan_sh[NTH / 32 + 1];
  __shared__ unsigned long long base_sh;
  __shared__ uint8_t unit_active[(NTH / 32) * WPR];
  __shared__ uint16_t unit_list[(NTH / 32) * WPR];
  __shared__ int unit_count;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int64_t n = args.n;
  const int64_t T = args.T;
  const float eps32 = args.eps32;

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();

  auto issue = [&](long long q, int buf) {  // thread 0 only
    int a, b;
    item_tiles(args, q, T, a, b);
    const int64_t nb = min((int64_t)TILE, n - (int64_t)b * TILE);
    const uint32_t bytes = (uint32_t)(nb * S * 4);
    mbar_expect_tx(&mbar[buf], bytes);
    bulk_g2s(bc + (size_t)buf * TILE * S, args.rec + (size_t)b * TILE * S, bytes, &mbar[buf]);
  };

  __shared__ long long range_sh[2];
  if (tid == 0) {
    long long lo = args.item_lo, hi = args.item_hi;
    if (args.item_list) {  // culled list: this shard's slice of the device-side count
      const long long total = (long long)*args.item_count;
      lo = total * args.shard_rank / args.shard_world;
      hi = total * (args.shard_rank + 1) / args.shard_world;
    }
    range_sh[0] = lo;
    range_sh[1] = hi;
  }
  __syncthreads();
  const long long item_lo = range_sh[0], item_hi = range_sh[1];
  if (tid == 0) {
    const long long q0 = item_lo + (long long)atomicAdd(args.work_ctr, 1ull);
    item_sh[0] = q0;
    if (q0 < item_hi) issue(q0, 0);
  }
  __syncthreads();

  long long q = item_sh[0];
  uint32_t phase = 0;  // bit b = parity of buffer b's next completion
  int it = 0;
  while (q < item_hi) {
    const int cur = (G::NBUF == 2) ? (it & 1) : 0;
    if (tid == 0) {
      const long long qn = item_lo + (long long)atomicAdd(args.work_ctr, 1ull);
      item_sh[(it + 1) & 1] = qn;
      if (G::NBUF == 2 && qn < item_hi) issue(qn, cur ^ 1);
    }
    int a, b;
    item_tiles(args, q, T, a, b);
    const int na = (int)min((int64_t)TILE, n - (int64_t)a * TILE);
    const int nb = (int)min((int64_t)TILE, n - (int64_t)b * TILE);

    // ---- work units: (lane block of 32*KP points) x (32-column group) ------------
    // LB = NTH/32 lane blocks x WPR column groups. A unit is inactive when its
    // columns are past the ragged end or (SAFE, d <= 4, culling on) the union box
    // of the lane block and the 32-point column block are provably out of range
    // (the bound of keep_item, evaluated in float with a 1e-5 relative and a 4x
    // rounding-error margin). Active units are split evenly across the warps, so
    // a warp whose own points are far from tile b still does its share.
    constexpr int LB = NTH / 32;
    constexpr int NU = LB * WPR;
    constexpr bool kBlockSkip = SAFE && D <= 4;
    const bool block_skip = kBlockSkip && args.blk != nullptr;
    mbar_wait(&mbar[cur], (phase >> cur) & 1u);
    phase ^= (1u << cur);
    const float* bcb = bc + (size_t)cur * TILE * S;
    for (int u = tid; u < NU; u += NTH) {
      const int lb = u / WPR, jw = u % WPR;
      bool active = jw * 32 < nb && lb * 32 * KP < na;
      if (kBlockSkip && block_skip && active) {
        constexpr int BS = 2 * D + 1;
        const float* cb = args.blk + (size_t)(b * (TILE / 32) + jw) * BS;
        const float* lbb = args.blk + (size_t)(a * (TILE / 32) + lb * KP) * BS;
        float L = 0.f, wn = 0.f;
#pragma unroll
        for (int q = 0; q < D; ++q) {
          float lo = INFINITY, hi = -INFINITY;
#pragma unroll
          for (int k = 0; k < KP; ++k) {
            lo = fminf(lo, __ldg(lbb + k * BS + q));
            hi = fmaxf(hi, __ldg(lbb + k * BS + D + q));
          }
          const float g = fmaxf(0.f, fmaxf(__ldg(cb + q) - hi, lo - __ldg(cb + D + q)));
          L += g * g;
        }
#pragma unroll
        for (int k = 0; k < KP; ++k) wn = fmaxf(wn, __ldg(lbb + k * BS + 2 * D));
        float bound = L * (1.0f - 1e-5f);
        if (F == DS_FORMULA_ALGEBRAIC)
          bound -= 4.0f * (2.0f * D + 3.0f) * 5.97e-8f * (wn + __ldg(cb + 2 * D)) * 1.01f;
        active = !(bound > eps32);  // NaN keeps the unit
      }
      unit_active[u] = active ? 1 : 0;
    }
    __syncthreads();
    if (tid < 32 && NU > 0) {
      // compact the active units in (lane block, column group) order
      int cnt_total = 0;
      for (int u0 = 0; u0 < NU; u0 += 32) {
        const bool act = (u0 + tid < NU) && unit_active[u0 + tid];
        const uint32_t bal = __ballot_sync(0xffffffffu, act);
        if (act) unit_list[cnt_total + __popc(bal & ((1u << tid) - 1u))] = (uint16_t)(u0 + tid);
        cnt_total += __popc(bal);
      }
      if (tid == 0) unit_count = cnt_total;
    }
    __syncthreads();
    const int nact = unit_count;
    const int warp = tid >> 5;
    // zero the rows of inactive units (their words are 0)
    for (int u = warp; u < NU; u += LB) {
      if (unit_active[u]) continue;
      const int lb = u / WPR, jw = u % WPR;
#pragma unroll
      for (int k = 0; k < KP; ++k) bits[jw * BSTRIDE + k * NTH + lb * 32 + lane] = 0u;
    }

    uint32_t any = 0;
    uint32_t groups = 0;
    int cur_lb = -1;
    Lanes<D, KP> L;
    bool lvalid[KP];
    const int u_lo = nact * warp / LB, u_hi = nact * (warp + 1) / LB;
    for (int ui = u_lo; ui < u_hi; ++ui) {
      const int u = unit_list[ui];
      const int lb = u / WPR, jw = u % WPR;
      if (lb != cur_lb) {  // (re)load the lane block's points into registers
        cur_lb = lb;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const int il = (lb * 32 + lane) * KP + k;  // 32*KP consecutive points per block
          lvalid[k] = il < na;
          const int64_t i = (int64_t)a * TILE + (lvalid[k] ? il : 0);
          const float4* r4 = reinterpret_cast<const float4*>(args.rec + (size_t)i * S);
          float tmp[S];
#pragma unroll
          for (int v = 0; v < S / 4; ++v) {
            const float4 x = __ldg(r4 + v);
            tmp[4 * v + 0] = x.x;
            tmp[4 * v + 1] = x.y;
            tmp[4 * v + 2] = x.z;
            tmp[4 * v + 3] = x.w;
          }
          float c[D];
#pragma unroll
          for (int q = 0; q < D; ++q)
            c[q] = (F == DS_FORMULA_ALGEBRAIC) ? __fadd_rn(tmp[q], tmp[q]) : -tmp[q];
#pragma unroll
          for (int q = 0; q < Lanes<D, KP>::DP; ++q) L.v2[k][q] = make_float2(c[2 * q], c[2 * q + 1]);
          L.v1[k] = c[D - 1];
          L.t[k] = tmp[D];
        }
      }
      ++groups;
      uint32_t acc[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) acc[k] = 0;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const float4* p4 = reinterpret_cast<const float4*>(bcb + (size_t)(jw * 32 + jj) * S);
        float xj[S];
#pragma unroll
        for (int v = 0; v < S / 4; ++v) {
          const float4 x = p4[v];
          xj[4 * v + 0] = x.x;
          xj[4 * v + 1] = x.y;
          xj[4 * v + 2] = x.z;
          xj[4 * v + 3] = x.w;
        }
        float d2[KP];
        eval_d2<D, F, KP>(L, xj, xj[D], d2);
        pack_bits<KP, SAFE>(d2, eps32, jj, acc);
      }
      const uint32_t vm = valid_mask(nb - jw * 32);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const uint32_t w = lvalid[k] ? ((k < KC ? acc[k] : ~acc[k]) & vm) : 0u;
        bits[jw * BSTRIDE + k * NTH + lb * 32 + lane] = w;
        any |= w;
      }
    }

    // ---- epilogue --------------------------------------------------------------
    if (lane == 0 && groups)  // pairs actually evaluated: groups x 32 columns x 32*KP lane points
      atomicAdd(args.pairs_done, (unsigned long long)groups * 32ull * 32ull * KP);
    const int any_all = __syncthreads_or(any != 0);
    if (any_all) {  // lane-side counts: popcount of each row's active words (slot k*NTH + tid)
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        uint32_t cnt_k = 0;
#pragma unroll
        for (int jw = 0; jw < WPR; ++jw)
          if (unit_active[warp * WPR + jw]) cnt_k += __popc(bits[jw * BSTRIDE + k * NTH + tid]);
        if (cnt_k) atomicAdd(&args.cnt[(int64_t)a * TILE + tid * KP + k], (int)cnt_k);
      }
    }

    if (any_all) {
      const int w = tid / G::CHUNKS;   // word column handled by this thread
      const int c = tid % G::CHUNKS;   // row chunk: slots c, c + CHUNKS, ...
      const uint32_t* col = bits + w * BSTRIDE + c;
      // slots c + CHUNKS*r for r in [r0, r0 + SEG) all belong to one lane block, so
      // an inactive (lane block, w) unit skips SEG rows at once
      constexpr int SEG = 32 / G::CHUNKS;

      // pass 1: staged-side counts (vertical popcount of word column w) and the
      // number of words to append (upper triangle only on the diagonal tile)
      uint32_t s[10];
#pragma unroll
      for (int l = 0; l < 10; ++l) s[l] = 0;
      uint32_t nz = 0;
      for (int r0 = 0; r0 < G::ROWS; r0 += SEG) {
        const int lb0 = ((c + r0 * G::CHUNKS) % NTH) / 32;
        if (!unit_active[lb0 * WPR + w]) continue;
#pragma unroll
        for (int r = r0; r < r0 + SEG; ++r) {
          uint32_t x = col[r * G::CHUNKS];
          if (!x) continue;
          if (a != b) {
            uint32_t carry = x;
#pragma unroll
            for (int l = 0; l < G::SL0; ++l) {
              const uint32_t t2 = s[l] & carry;
              s[l] ^= carry;
              carry = t2;
            }
          } else {
            const int p = c + r * G::CHUNKS;  // smem slot -> point (slot k*NTH + t holds t*KP + k)
            const int il = (p % NTH) * KP + p / NTH;
            x &= diag_keep(il - w * 32);      // keep columns t >= row
          }
          nz += (x != 0);
        }
      }
      if (a != b) {
#pragma unroll
        for (int off = 1; off < G::CHUNKS; off <<= 1) {
          uint32_t o[10];
#pragma unroll
          for (int l = 0; l < 10; ++l) o[l] = __shfl_xor_sync(0xffffffffu, s[l], off);
          sliced_add(s, o);
        }
        constexpr int PER = 32 / G::CHUNKS;
#pragma unroll
        for (int qq = 0; qq < PER; ++qq) {
          const int p = c * PER + qq;  // bit position
          uint32_t v = 0;
#pragma unroll
          for (int l = 0; l < 10; ++l) v |= ((s[l] >> p) & 1u) << l;
          if (v) atomicAdd(&args.cnt[(int64_t)b * TILE + w * 32 + (31 - p)], (int)v);
        }
      }

      uint32_t incl = nz;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      if (lane == 31) scan_sh[tid >> 5] = incl;
      __syncthreads();
      if (tid == 0) {
        unsigned int run = 0;
        for (int wi = 0; wi < NTH / 32; ++wi) {
          const unsigned int t2 = scan_sh[wi];
          scan_sh[wi] = run;
          run += t2;
        }
        base_sh = run ? atomicAdd(args.words_count, (unsigned long long)run) : 0ull;
        if (run) {
          // one chunk per non-empty tile pair: its words are contiguous
          const unsigned long long ci = atomicAdd(args.nonempty_count, 1ull);
          if (ci < args.chunks_cap)
            args.chunks[ci] = make_uint4((uint32_t)a, (uint32_t)b, (uint32_t)base_sh,
                                         run | ((uint32_t)(base_sh >> 32) << 16));
        }
      }
      __syncthreads();
      // pass 2: append the words
      unsigned long long pos = base_sh + scan_sh[tid >> 5] + (incl - nz);
      if (nz) {
        for (int r0 = 0; r0 < G::ROWS; r0 += SEG) {
          const int lb0 = ((c + r0 * G::CHUNKS) % NTH) / 32;
          if (!unit_active[lb0 * WPR + w]) continue;
#pragma unroll
          for (int r = r0; r < r0 + SEG; ++r) {
            uint32_t x = col[r * G::CHUNKS];
            if (!x) continue;
            const int p = c + r * G::CHUNKS;
            const int il = (p % NTH) * KP + p / NTH;
            if (a == b) x &= diag_keep(il - w * 32);
            if (x) {
              if (pos < args.words_cap) args.words[pos] = make_uint2(x, (uint32_t)(il << 4 | w));
              ++pos;
            }
          }
        }
      }
    }
    __syncthreads();
    const long long qn = item_sh[(it + 1) & 1];
    if (G::NBUF == 1 && tid == 0 && qn < item_hi) issue(qn, 0);
    q = qn;
    ++it;
  }
}

// ---- prep: narrow to float32 (RN), squared norms, padded records ------------------
__global__ void prep_kernel(const double* __restrict__ coords, int64_t n, int d, int dpad, int S,
                            float* __restrict__ rec, uint32_t* unsafe_flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* src = coords + i * d;
  float* dst = rec + i * S;
  float p = 0.f;
  bool bad = false;
  for (int c = 0; c < dpad; ++c) {
    const float v = c < d ? __double2float_rn(src[c]) : 0.f;  // kernels.py:148-150
    dst[c] = v;
    const float sq = __fmul_rn(v, v);
    p = (c == 0) ? sq : __fadd_rn(p, sq);  // kernels.py:388-391, left to right
    bad |= !(fabsf(v) <= SAFE_ABS);
  }
  dst[dpad] = p;
  for (int c = dpad + 1; c < S; ++c) dst[c] = 0.f;
  if (bad) atomicOr(unsafe_flag, 1u);
}

// ---- tile culling ------------------------------------------------------------------
// Per tile: coordinate bounding box (float32, exact) and max squared norm.
__global__ void tile_bounds_kernel(const float* __restrict__ rec, int64_t n, int dpad, int S,
                                   float* __restrict__ lo, float* __restrict__ hi,
                                   float* __restrict__ maxnorm) {
  const int tile = blockIdx.x;
  const int64_t base = (int64_t)tile * TILE;
  const int cnt = (int)min((int64_t)TILE, n - base);
  __shared__ float red[32];
  for (int k = 0; k <= dpad; ++k) {  // k == dpad: the norm column
    float mn = INFINITY, mx = -INFINITY;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const float v = rec[(base + i) * S + k];
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
    }
    for (int off = 16; off; off >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (lane == 0) red[warp] = mn;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < nw; ++w) mn = fminf(mn, red[w]);
      red[0] = mn;
    }
    __syncthreads();
    mn = red[0];
    __syncthreads();
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < nw; ++w) mx = fmaxf(mx, red[w]);
      if (k < dpad) {
        lo[(int64_t)tile * dpad + k] = mn;
        hi[(int64_t)tile * dpad + k] = mx;
      } else {
        maxnorm[tile] = mx;
      }
    }
    __syncthreads();
  }
}

// Per 32-point block (one warp each): box and max squared norm, in the layout
// blk[block][lo 0..dpad-1, hi 0..dpad-1, maxnorm] the tile kernel reads.
__global__ void block_bounds_kernel(const float* __restrict__ rec, int64_t n, int dpad, int S,
                                   float* __restrict__ blk) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nblk = (n + 31) / 32;
  if (warp >= nblk) return;
  const int64_t i = warp * 32 + lane;
  const bool valid = i < n;
  float* out = blk + warp * (2 * dpad + 1);
  for (int k = 0; k <= dpad; ++k) {
    const float v = valid ? rec[i * S + k] : 0.f;
    float mn = valid ? v : INFINITY, mx = valid ? v : -INFINITY;
    for (int off = 16; off; off >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    }
    if (lane == 0) {
      if (k < dpad) {
        out[k] = mn;
        out[dpad + k] = mx;
      } else {
        out[2 * dpad] = mx;
      }
    }
  }
}

// Keep tile pair (a, b), a <= b, unless every pair in it is provably out of range
// in the formula's float32 arithmetic. L = squared gap between the boxes (exact
// reals, evaluated in double). DIRECT: every op is monotone in |dx| and the terms
// are >= 0, so d2_computed >= L (1 - u)^(3d); ALGEBRAIC: |d2_computed - D| <=
// (2d+3) u (T + P) (1 + O(u)) by the standard summation bound, D >= L. Both
// slacks are taken 4x larger; a tile pair is culled only if even the slackened
// lower bound exceeds eps32. Inputs that need the overflow-safe compare are never
// culled (the flag is checked here, on the device).
__device__ __forceinline__ bool keep_item(const float* __restrict__ lo, const float* __restrict__ hi,
                                          const float* __restrict__ maxnorm, int dpad, int a, int b,
                                          float eps32, int formula, bool unsafe) {
  if (unsafe || a == b) return true;
  const double u = 1.0 / 16777216.0;
  double L = 0.0;
  for (int k = 0; k < dpad; ++k) {
    const double g1 = (double)lo[(int64_t)b * dpad + k] - (double)hi[(int64_t)a * dpad + k];
    const double g2 = (double)lo[(int64_t)a * dpad + k] - (double)hi[(int64_t)b * dpad + k];
    const double g = fmax(0.0, fmax(g1, g2));
    L += g * g;
  }
  double bound = L * (1.0 - 4.0 * 3.0 * dpad * u) * (1.0 - 1e-12);
  if (formula == DS_FORMULA_ALGEBRAIC)
    bound -= 4.0 * (2.0 * dpad + 3.0) * u * ((double)maxnorm[a] + (double)maxnorm[b]) * 1.001;
  return !(bound > (double)eps32);  // NaN bounds keep the pair
}

// pass 1: keep flag per item (int32, scanned in place afterwards)
__global__ void cull_flags_kernel(const float* __restrict__ lo, const float* __restrict__ hi,
                                  const float* __restrict__ maxnorm, int dpad, int64_t T,
                                  float eps32, int formula, const uint32_t* __restrict__ unsafe_flag,
                                  int32_t* __restrict__ flags) {
  const int64_t total = T * (T + 1) / 2;
  const bool unsafe = *unsafe_flag != 0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    int a, b;
    decode_item(q, T, a, b);
    flags[q] = keep_item(lo, hi, maxnorm, dpad, a, b, eps32, formula, unsafe) ? 1 : 0;
  }
}

// pass 3: stable scatter by the exclusive scan, so the kept list is in item order
// and identical on every rank (ranks slice it by position)
__global__ void cull_scatter_kernel(const float* __restrict__ lo, const float* __restrict__ hi,
                                    const float* __restrict__ maxnorm, int dpad, int64_t T,
                                    float eps32, int formula,
                                    const uint32_t* __restrict__ unsafe_flag,
                                    const int32_t* __restrict__ pos, const int32_t* __restrict__ total_kept,
                                    uint32_t* __restrict__ list, unsigned long long* count) {
  const int64_t total = T * (T + 1) / 2;
  const bool unsafe = *unsafe_flag != 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = (unsigned long long)*total_kept;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    int a, b;
    decode_item(q, T, a, b);
    if (keep_item(lo, hi, maxnorm, dpad, a, b, eps32, formula, unsafe))
      list[pos[q]] = ((uint32_t)a << 16) | (uint32_t)b;
  }
}

int pad_dim(int d) {
  if (d <= 4) return d;
  if (d <= 8) return 8;
  if (d <= 16) return 16;
  if (d <= 32) return 32;
  return 64;
}

template <int D, int F, bool SAFE>
cudaError_t launch_one(const TileArgs& a, int sm_count, cudaStream_t s) {
  using G = Geo<D>;
  auto kern = eps_tile_kernel<D, F, SAFE>;
  static bool configured = false;
  static int per_sm = 1;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::THREADS, G::SMEM);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    configured = true;
  }
  const int64_t items = a.item_list ? (int64_t)1 << 40 : a.item_hi - a.item_lo;
  int64_t grid = (int64_t)sm_count * per_sm;
  if (grid > items) grid = items;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, G::THREADS, G::SMEM, s>>>(a);
  return cudaGetLastError();
}

// Both instantiations are launched back to back; each reads the device flag set by
// the prep kernel and the one that does not own the input exits immediately, so
// the host never waits for the range check.
template <int D, int F>
cudaError_t launch_df(const TileArgs& a, int sm_count, cudaStream_t s) {
  cudaError_t e = launch_one<D, F, true>(a, sm_count, s);
  if (e != cudaSuccess) return e;
  return launch_one<D, F, false>(a, sm_count, s);
}

template <int D>
cudaError_t launch_d(const TileArgs& a, int formula, int sm_count, cudaStream_t s) {
  return formula == DS_FORMULA_ALGEBRAIC ? launch_df<D, DS_FORMULA_ALGEBRAIC>(a, sm_count, s)
                                         : launch_df<D, DS_FORMULA_DIRECT>(a, sm_count, s);
}

}  // namespace

int padded_dim(int d) { return pad_dim(d); }

size_t tile_smem_bytes(int d) {
  switch (pad_dim(d)) {
    case 1: return Geo<1>::SMEM;
    case 2: return Geo<2>::SMEM;
    case 3: return Geo<3>::SMEM;
    case 4: return Geo<4>::SMEM;
    case 8: return Geo<8>::SMEM;
    case 16: return Geo<16>::SMEM;
    case 32: return Geo<32>::SMEM;
    default: return Geo<64>::SMEM;
  }
}

cudaError_t launch_prep(const double* coords, int64_t n, int d, float* rec, uint32_t* unsafe_flag,
                        cudaStream_t s) {
  const int dp = pad_dim(d);
  const int S = ((dp + 1) + 3) / 4 * 4;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  prep_kernel<<<(unsigned)blocks, threads, 0, s>>>(coords, n, d, dp, S, rec, unsafe_flag);
  return cudaGetLastError();
}

cudaError_t launch_cull(const float* rec, int64_t n, int d, float eps32, int formula,
                        const uint32_t* unsafe_flag, float* lo, float* hi, float* maxnorm,
                        int32_t* flags, int32_t* partials, int32_t* total_kept, uint32_t* list,
                        unsigned long long* count, cudaStream_t s) {
  const int dp = pad_dim(d);
  const int S = ((dp + 1) + 3) / 4 * 4;
  const int64_t T = (n + TILE - 1) / TILE;
  tile_bounds_kernel<<<(unsigned)T, 256, 0, s>>>(rec, n, dp, S, lo, hi, maxnorm);
  const int64_t total = T * (T + 1) / 2;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  cull_flags_kernel<<<(unsigned)blocks, 256, 0, s>>>(lo, hi, maxnorm, dp, T, eps32, formula,
                                                     unsafe_flag, flags);
  cudaError_t e = launch_exclusive_scan(flags, total, partials, total_kept, s);
  if (e != cudaSuccess) return e;
  cull_scatter_kernel<<<(unsigned)blocks, 256, 0, s>>>(lo, hi, maxnorm, dp, T, eps32, formula,
                                                       unsafe_flag, flags, total_kept, list, count);
  return cudaGetLastError();
}

cudaError_t launch_block_bounds(const float* rec, int64_t n, int d, float* blk, cudaStream_t s) {
  const int dp = pad_dim(d);
  const int S = ((dp + 1) + 3) / 4 * 4;
  const int64_t warps = (n + 31) / 32;
  block_bounds_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(rec, n, dp, S, blk);
  return cudaGetLastError();
}

cudaError_t launch_tile(const TileArgs& a, int formula, int sm_count, cudaStream_t s) {
  switch (pad_dim(a.d)) {
    case 1: return launch_d<1>(a, formula, sm_count, s);
    case 2: return launch_d<2>(a, formula, sm_count, s);
    case 3: return launch_d<3>(a, formula, sm_count, s);
    case 4: return launch_d<4>(a, formula, sm_count, s);
    case 8: return launch_d<8>(a, formula, sm_count, s);
    case 16: return launch_d<16>(a, formula, sm_count, s);
    case 32: return launch_d<32>(a, formula, sm_count, s);
    default: return launch_d<64>(a, formula, sm_count, s);
  }
}

}  // namespace ds
