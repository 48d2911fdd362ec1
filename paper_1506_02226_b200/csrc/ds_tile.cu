// Stage 1+2 of the densescan hot path on sm_100a: the fused eps-tile kernel.
//
// Replaces the reference's fused_build / fused_build_algebraic
// (pkg/src/densescan/kernels.py:311-442): every pair (i, j) is tested
// against eps^2 in float32 with the reference's operation order and
// rounding, the distance matrix is never stored, and the result leaves the
// kernel as bit-packed 32-bit adjacency words plus neighbour counts.
//
// Work decomposition. Points (in spatial order, ds_sort.cu) are cut into tiles of
// TILE=512. The relation is exactly symmetric (both formulas are bitwise symmetric
// in (i, j)), so only tile pairs (a, b) with a <= b are evaluated.
// Inside a tile pair the work unit of one warp is (a lane block of 32*KP points of
// tile a, held in registers) x (up to 4-16 column blocks of 32 points of tile b,
// streamed through a per-warp double buffer with cp.async). Warps run independently:
// no block-level barrier, dynamic batches of units (see eps_unit_kernel). Per staged
// point every lane computes d2 for its KP points in the exact reference order, every
// operation a separately rounded f32 op (never contracted into an FMA;
// tests/test_abi.py checks the SASS) — the FP32 pipe is the bound, so products of two
// dimensions go through one FMUL2 and T + P / the final subtraction of two lane
// points through one FADD2, which executes exactly the 2d+1 (algebraic) or 3d-1
// (direct) FP32 lane-ops per pair. Predicates become 32-bit words (FSETP or the sign
// bit of fl(eps32 - d2), see pack_bits); lane-side counts are popcounts of the words,
// column-side counts a bit-sliced vertical popcount; the non-zero words are appended
// to HBM for stage 3 with their local row and column block, one chunk entry per
// (unit, column block).
#include <cuda_runtime.h>

#include <atomic>
#include <stdint.h>

#include <algorithm>

#include "ds_internal.cuh"

namespace ds {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}


// Diagonal tile: keep columns t >= rel (j >= i incl. the self pair; the self bit
// is needed by the reference-layout export and is a no-op for the merge).
__device__ __forceinline__ uint32_t diag_keep(int rel) {
  return rel <= 0 ? 0xffffffffu : (rel > 31 ? 0u : ((1u << (32 - rel)) - 1u));
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
// KP even and d >= DS_PAIR_MIN_D (PAIRED): lane points 2h and 2h+1 share every packed register instead —
// c2[h][q] = {c_q of 2h, c_q of 2h+1} (the ALG / DIR value above), t2[h] = {T_2h, T_2h+1}
// — so every FP op of the pair loop is a two-lane-point FFMA2 / FADD2 with the staged
// coordinate broadcast (`R.F32` operand): an FP32-pipe slot does two lane-ops for every
// term, where the per-lane-point packing spent scalar FADDs on the cross sum.
// Measured on B200 (A/B, round 2): the paired packing cuts the C4 (16-D) eps kernel
// 20.2 -> 18.5 ms; at d = 2 (C2 / C3 / C5) it is neutral to +2 % — the culled 2-D
// schedule is bound by the per-step epilogue, not the FP32 pipe — so d <= 4 keeps the
// per-lane-point packing.
#ifndef DS_PAIR_MIN_D
#define DS_PAIR_MIN_D 5
#endif
template <int D, int KP>
struct Lanes {
  static constexpr int DP = D / 2;
  static constexpr bool ODD = (D & 1) != 0;
  static constexpr bool PAIRED = KP % 2 == 0 && D >= DS_PAIR_MIN_D;
  static constexpr int H = PAIRED ? KP / 2 : 1;
  float2 c2[H][PAIRED ? D : 1];
  float2 t2[H];
  float2 v2[PAIRED ? 1 : KP][DP > 0 && !PAIRED ? DP : 1];
  float v1[KP];
  float t[KP];
};

// fl(a * b) for two lanes as FFMA2(a, b, z) with z = {-0, -0} held in a register: the
// exact product plus -0 rounds once to the product's own rounding (+0 + -0 = +0 in RN),
// so it is bitwise the FMUL2 — but unlike FMUL2 it cannot be contracted with the FADD2
// that consumes it (ptxas turns FMUL2 -> FADD2 into FFMA2 even at --fmad=false, which
// would drop a rounding; tests/test_abi.py checks every FFMA2 of the pair loop adds z).
__device__ __forceinline__ float2 mul2_exact(float2 a, float2 b, float2 z) { return __ffma2_rn(a, b, z); }

// Squared distances of lane points K0 .. K1-1 to staged point j (xj: its record,
// pj = P_j), in the reference's order with one rounding per operation.
template <int D, int F, int KP, int K0 = 0, int K1 = KP>
__device__ __forceinline__ void eval_d2(const Lanes<D, KP>& L, const float* xj, float pj, float2 z,
                                        float (&d2)[KP]) {
  constexpr int DP = Lanes<D, KP>::DP;
  constexpr bool ODD = Lanes<D, KP>::ODD;
  if constexpr (Lanes<D, KP>::PAIRED) {
    static_assert(K0 % 2 == 0 && K1 % 2 == 0, "lane points are evaluated in pairs");
#pragma unroll
    for (int h = K0 / 2; h < K1 / 2; ++h) {
      float2 acc;
      if constexpr (F == DS_FORMULA_ALGEBRAIC) {
        // cross = ((X0*x0 + X1*x1) + X2*x2) + ...          (kernels.py:409-414)
        acc = mul2_exact(L.c2[h][0], make_float2(xj[0], xj[0]), z);
#pragma unroll
        for (int q = 1; q < D; ++q)
          acc = __fadd2_rn(acc, mul2_exact(L.c2[h][q], make_float2(xj[q], xj[q]), z));
        // d2 = (T + P) - cross                              (kernels.py:415-417)
        const float2 tp = __fadd2_rn(L.t2[h], make_float2(pj, pj));
        acc = __fadd2_rn(tp, make_float2(-acc.x, -acc.y));
      } else {
        // d2 = ((dx0^2 + dx1^2) + dx2^2) + ..., dx = x_col - x_row  (kernels.py:197-210)
        float2 dx = __fadd2_rn(make_float2(xj[0], xj[0]), L.c2[h][0]);
        acc = mul2_exact(dx, dx, z);
#pragma unroll
        for (int q = 1; q < D; ++q) {
          dx = __fadd2_rn(make_float2(xj[q], xj[q]), L.c2[h][q]);
          acc = __fadd2_rn(acc, mul2_exact(dx, dx, z));
        }
      }
      d2[2 * h] = acc.x;
      d2[2 * h + 1] = acc.y;
    }
  } else if constexpr (F == DS_FORMULA_ALGEBRAIC) {
    // cross = ((X0*x0 + X1*x1) + X2*x2) + ...            (kernels.py:409-414)
    float c[KP];
#pragma unroll
    for (int k = K0; k < K1; ++k) {
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
      for (int k = K0; k < K1; k += 2) {
        const float2 tp = __fadd2_rn(make_float2(L.t[k], L.t[k + 1]), make_float2(pj, pj));
        const float2 d = __fadd2_rn(tp, make_float2(-c[k], -c[k + 1]));
        d2[k] = d.x;
        d2[k + 1] = d.y;
      }
    } else {
#pragma unroll
      for (int k = K0; k < K1; ++k) d2[k] = __fsub_rn(__fadd_rn(L.t[k], pj), c[k]);
    }
  } else {
    // d2 = ((dx0^2 + dx1^2) + dx2^2) + ..., dx = x_col - x_row  (kernels.py:197-210)
#pragma unroll
    for (int k = K0; k < K1; ++k) {
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
// Measured on B200 (tools/tile_bench.py): d <= 4 runs best with 3 of 4 lane points
// compared (the FP32 pipe is the tighter one there), wider records with all lane
// points on the sign-bit path (the cross-product chain leaves the ALU idle). A
// compare costs FSETP + SEL + half an IADD3 (ptxas lowers set.* and predicated
// lop3 to the same), the sign bit one FP op + one funnel shift.
template <int KP, bool SAFE, int D>
struct Pack {
#ifndef DS_KC_SMALL
#define DS_KC_SMALL 3
#endif
  static constexpr int KC = !SAFE ? KP : (D <= 4 ? (DS_KC_SMALL * KP) / 4 : 0);
};

template <int KP, bool SAFE, int D, int K0 = 0, int K1 = KP>
__device__ __forceinline__ void pack_bits(const float (&d2)[KP], float eps32, int jj,
                                          uint32_t (&acc)[KP]) {
  constexpr int KC = Pack<KP, SAFE, D>::KC;
  constexpr int KS = KC > K0 ? KC : K0;  // first sign-bit lane point of the range
#pragma unroll
  for (int k = K0; k < (KC < K1 ? KC : K1); ++k) acc[k] |= (d2[k] <= eps32 ? 1u : 0u) << (31 - jj);
  if constexpr (KS < K1) {
    if constexpr ((K1 - KS) % 2 == 0) {
#pragma unroll
      for (int k = KS; k < K1; k += 2) {
        const float2 e = __fadd2_rn(make_float2(eps32, eps32), make_float2(-d2[k], -d2[k + 1]));
        acc[k] = __funnelshift_l(__float_as_uint(e.x), acc[k], 1);
        acc[k + 1] = __funnelshift_l(__float_as_uint(e.y), acc[k + 1], 1);
      }
    } else {
#pragma unroll
      for (int k = KS; k < K1; ++k)
        acc[k] = __funnelshift_l(__float_as_uint(__fsub_rn(eps32, d2[k])), acc[k], 1);
    }
  }
}

template <int D>
struct Geo {
  static constexpr int KP = D <= 16 ? 4 : (D <= 32 ? 2 : 1);  // lane points per lane
  static constexpr int S = ((D + 1) + 3) / 4 * 4;           // floats per record
  static constexpr int WARPS = 4;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int STAGE = 32 * S;                       // floats per staged block
  static constexpr size_t SMEM = (size_t)WARPS * 2 * STAGE * 4;
#ifndef DS_UNROLL_WIDE
#define DS_UNROLL_WIDE 8
#endif
#ifndef DS_MINB16
#define DS_MINB16 3
#endif
#ifndef DS_UNROLL_SMALL
#define DS_UNROLL_SMALL 32
#endif
  static constexpr int UNROLL = D <= 4 ? DS_UNROLL_SMALL : DS_UNROLL_WIDE;
  // resident CTAs (x 4 warps) per SM: 16-D holds 4 lane points x 17 floats per lane
#ifndef DS_MINB_SMALL
#define DS_MINB_SMALL 4
#endif
  static constexpr int MINB = D <= 4 ? DS_MINB_SMALL
                                     : ((D <= 8 || D == 32) ? 4 : (D == 16 ? DS_MINB16 : 3));
};

// Column-side counts of one unit: the number of set bits of every column over the
// warp's 32*KP words. Per lane the KP words are added bit-sliced (carry-save), then
// five butterfly rounds add the lanes' slice vectors; lane j extracts column j.
template <int KP>
__device__ __forceinline__ uint32_t column_counts(const uint32_t (&w)[KP], int lane) {
  constexpr int W0 = KP == 4 ? 3 : (KP == 2 ? 2 : 1);
  uint32_t s[W0 + 5];
#pragma unroll
  for (int l = 0; l < W0 + 5; ++l) s[l] = 0u;
  if constexpr (KP == 4) {
    const uint32_t x = w[0] ^ w[1] ^ w[2];
    const uint32_t c1 = (w[0] & w[1]) | (w[2] & (w[0] ^ w[1]));
    s[0] = x ^ w[3];
    const uint32_t c2 = x & w[3];
    s[1] = c1 ^ c2;
    s[2] = c1 & c2;
  } else if constexpr (KP == 2) {
    s[0] = w[0] ^ w[1];
    s[1] = w[0] & w[1];
  } else {
    s[0] = w[0];
  }
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int width = W0 + r;
    uint32_t carry = 0u;
#pragma unroll
    for (int l = 0; l < W0 + 4; ++l) {
      if (l < width) {
        const uint32_t t = s[l];
        const uint32_t o = __shfl_xor_sync(0xffffffffu, t, 16 >> r);
        s[l] = t ^ o ^ carry;
        carry = (t & o) | (carry & (t ^ o));
      }
    }
#pragma unroll
    for (int l = 0; l < W0 + 5; ++l)
      if (l == width) s[l] = carry;
  }
  const int p = 31 - lane;  // bit (31 - j) <-> column j
  uint32_t v = 0u;
#pragma unroll
  for (int l = 0; l < W0 + 5; ++l) v |= ((s[l] >> p) & 1u) << l;
  return v;
}

// ---- row units ---------------------------------------------------------------------
// A row unit is (tile pair (a, b), lane block lb) plus a 16-bit mask of the column
// blocks jw (32 points of tile b each) it evaluates. The warp holds the lane block
// (32*KP consecutive points of tile a) in registers for the whole unit and streams
// the masked column blocks through shared memory. Column block jw of unit u owns
// chunk entry u * WPR + jw (its words), so a tile pair's words are the chunk entries
// of its units. LB = TILE / (32*KP) lane blocks per tile.
//
// Structural mask: column blocks inside tile b (ragged tail) and, on a diagonal tile
// (a == b), not entirely below the lane block — pairs below the diagonal are covered
// by the mirrored unit. `self` column blocks (a == b, jw < (lb+1)*KP) overlap the
// lane block and keep only j >= i.
__device__ __forceinline__ uint32_t struct_mask(int n, int KP, int a, int b, int lb) {
  const int na = min(TILE, n - a * TILE);
  const int nb = min(TILE, n - b * TILE);
  if (lb * 32 * KP >= na) return 0u;
  const int nblk = (nb + 31) / 32;
  uint32_t m = (1u << nblk) - 1u;  // nblk <= 16
  if (a == b) m &= ~((1u << (lb * KP)) - 1u);
  return m;
}

// One column-block step of a row unit.
struct Step {
  long long u;
  int a, b, lb, jw;
  int pm;  // row-block pairs to evaluate: bit 0 lane points 0-1, bit 1 lane points 2-3
};

// One column-block step's pair loop over lane points K0 .. K1-1 (KP = 4: one or both
// pairs of lane points; the row-pair mask of the unit list, see box_pairs).
template <int D, int F, bool SAFE, int K0, int K1>
__device__ __forceinline__ void pair_loop(const Lanes<D, Geo<D>::KP>& L, const float* st, float eps32,
                                          float2 z, uint32_t (&acc)[Geo<D>::KP]) {
  using G = Geo<D>;
  constexpr int S = G::S;
  constexpr int KP = G::KP;
  // full unroll for d <= 4; wider records unroll by 8 to keep the independent
  // warps' code inside the instruction cache
#pragma unroll(G::UNROLL)
  for (int jj = 0; jj < 32; ++jj) {
    const float4* p4 = reinterpret_cast<const float4*>(st + jj * S);
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
    eval_d2<D, F, KP, K0, K1>(L, xj, xj[D], z, d2);
    pack_bits<KP, SAFE, D, K0, K1>(d2, eps32, jj, acc);
  }
}

// cp.async staging of one column block (16 bytes per instruction, zero-filled past n)
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The eps-tile kernel. Warps work independently (no block-level synchronisation):
//   * units come in batches of B consecutive units (about 32 batches per warp, 128 for
//     records wider than 4 dimensions): the
//     first two batches of a warp are static, later ones come from a global atomic
//     counter; each batch's index and its list entries (one per lane, coalesced) are
//     fetched one batch ahead, so neither the atomic nor the list load is on the
//     critical path;
//   * the unit's lane block is held in registers; the masked column blocks are copied
//     into the warp's double buffer with cp.async (one 16-byte copy per lane and
//     record quarter), issued one column block ahead, across unit boundaries;
//   * per staged point every lane evaluates its KP points in the reference's exact
//     operation order (eval_d2) and packs the predicates (pack_bits);
//   * lane-side counts are popcounts accumulated in registers across the units of a
//     lane block; column-side counts (off-diagonal column blocks only: each unordered
//     pair is evaluated once) come from column_counts, one atomic per column;
//   * non-zero words go to a run of word slots the warp reserved earlier (one global
//     atomic per WORD_RUN slots) and the chunk entry records where they went. Column
//     blocks without a single bit (most of a dense schedule) skip both.
template <int D, int F, bool SAFE>
__device__ __forceinline__ void eps_unit_body(const UnitArgs& A) {
  using G = Geo<D>;
  constexpr int KP = G::KP;
  constexpr int S = G::S;
  constexpr int KC = Pack<KP, SAFE, D>::KC;
  constexpr int LB = TILE / (32 * KP);

  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  float* stage = reinterpret_cast<float*>(smem) + (size_t)warp * 2 * G::STAGE;

  const int n = (int)A.n;
  const int T = A.T;
  const float eps32 = A.eps32;
  const float2 z2 = make_float2(A.negz, A.negz);  // {-0, -0}, see mul2_exact
  const uint2* list = A.unit_list;
  // tile-local row of lane point k of `lane` in lane block lb: with row-pair culling (d <=
  // 4) lane point k is row block k of the lane block (rows lb*128 + 32k + lane), else the
  // lane holds KP consecutive rows
  constexpr bool STRIDED = KP == 4 && D <= 4;
  auto lrow = [](int lb, int ln, int k) -> int {
    return STRIDED ? lb * 32 * KP + k * 32 + ln : (lb * 32 + ln) * KP + k;
  };
  long long r_lo, r_hi;
  unit_range(A, r_lo, r_hi);
  if (r_lo >= r_hi) return;

  // ---- batches of row units: [lo, hi) + list entries (lane i: entry lo + i) ----
  // about 32 (d <= 4) or 128 (wider) batches per warp; indices from a 32-bit atomic counter
  const long long nw = (long long)gridDim.x * G::WARPS;
#ifndef DS_BATCH_MIN
#define DS_BATCH_MIN 1
#endif
  // wide records: a unit is tens of us (C4: ~33 us per warp), so the last batches set the
  // end of the launch — smaller batches (~128 per warp) keep that tail short
#ifndef DS_BATCHES_WIDE
#define DS_BATCHES_WIDE 128
#endif
// d <= 4: ~32 batches per warp (A/B, round 2: 16 -> 32 cut the C5 eps kernel's tail,
// 1.351 -> 1.324 ms, C3 0.622 -> 0.613 ms; 64 about the same, 128+ slower — the batches
// reach one unit and the counter traffic grows)
#ifndef DS_BATCHES_SMALL
#define DS_BATCHES_SMALL 32
#endif
  constexpr long long BATCHES = D > 4 ? DS_BATCHES_WIDE : DS_BATCHES_SMALL;
  long long B = (r_hi - r_lo) / (nw * BATCHES);
  B = B < DS_BATCH_MIN ? DS_BATCH_MIN : (B > 32 ? 32 : B);
  unsigned int* const ctr = reinterpret_cast<unsigned int*>(A.work_ctr);
  auto load_entries = [&](long long lo) -> uint2 {
    return (list && lo + lane < r_hi && lane < B) ? __ldg(list + lo + lane) : make_uint2(0u, 0u);
  };
  auto batch_lo = [&](unsigned int x) -> long long {
    const long long lo = r_lo + (long long)x * B;
    return lo < r_hi ? lo : r_hi;
  };
  // the first two batches of warp gw are gw and nw + gw; later ones come from the counter
  // (offset by 2 nw), its first fetch issued here and consumed two batches later
  const unsigned int gw = blockIdx.x * G::WARPS + warp;
  unsigned int pend = 0;
  if (lane == 0) pend = atomicAdd(ctr, 1u) + 2u * (unsigned int)nw;
  long long gpos = batch_lo(gw);  // next unit of the batch
  long long cb_lo = gpos;
  long long cb_hi = gpos + B < r_hi ? gpos + B : r_hi;
  uint2 cent = load_entries(cb_lo);
  long long nb_lo = batch_lo(gw + (unsigned int)nw);
  uint2 nent = load_entries(nb_lo);

  // ---- step generator: (unit, column block) in order ----
  uint32_t grem = 0u;  // column blocks of unit gu not yet handed out
  long long gu = 0;
  uint32_t gab = 0u;  // a << 16 | b
  int glb = 0;
  uint32_t gsub = 0xffffffffu;  // row-pair masks of unit gu's column blocks, 2 bits each
  auto next_step = [&](Step& st) -> bool {
    while (grem == 0u) {
      if (gpos >= cb_hi) {  // switch to the prefetched batch, prefetch the one after
        if (nb_lo >= r_hi) return false;
        cb_lo = gpos = nb_lo;
        cb_hi = nb_lo + B < r_hi ? nb_lo + B : r_hi;
        cent = nent;
        nb_lo = batch_lo(__shfl_sync(0xffffffffu, pend, 0));
        nent = load_entries(nb_lo);
        if (lane == 0) pend = atomicAdd(ctr, 1u) + 2u * (unsigned int)nw;
      }
      const long long u = gpos++;
      uint32_t m;
      if (list) {
        const int src = (int)(u - cb_lo);
        gab = __shfl_sync(0xffffffffu, cent.x, src);
        const uint32_t ey = __shfl_sync(0xffffffffu, cent.y, src);
        glb = (int)((ey >> 16) & 0xfu);
        m = ey & 0xffffu;
        gsub = KP == 4 ? ey >> 20 : 0xffffffffu;
      } else {
        int a, b;
        decode_item(u / LB, T, a, b);
        glb = (int)(u % LB);
        gab = ((uint32_t)a << 16) | (uint32_t)b;
        m = struct_mask(n, KP, a, b, glb);
        gsub = 0xffffffffu;  // up to 16 column blocks, all rows
      }
      gu = u;
      if (lane < WPR && !((m >> lane) & 1u)) A.uchunks[u * WPR + lane] = make_uint2(0u, 0u);
      grem = m;
    }
    st.u = gu;
    st.a = (int)(gab >> 16);
    st.b = (int)(gab & 0xffffu);
    st.lb = glb;
    st.jw = __ffs(grem) - 1;
    grem &= grem - 1u;
    st.pm = STRIDED ? (int)(gsub & 3u) : 3;
    gsub >>= 2;
    return true;
  };
  auto issue = [&](const Step& st, int buf) {  // all lanes: record `lane` of the block
    const int j = st.b * TILE + st.jw * 32 + lane;
    const bool v = j < n;
    const float* src = A.rec + (size_t)(v ? j : 0) * S;
    float* dst = stage + (size_t)buf * G::STAGE + lane * S;
#pragma unroll
    for (int q = 0; q < S / 4; ++q) cp_async16(dst + 4 * q, src + 4 * q, v ? 16u : 0u);
    cp_async_commit();
  };

  Step cur, nxt;
  bool have = next_step(cur);
  if (have) issue(cur, 0);
  int it = 0;
  int la = -1, llb = -1;  // lane block held in registers
  Lanes<D, KP> L;
  bool lvalid[KP];
  uint32_t lcnt[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    lvalid[k] = false;
    lcnt[k] = 0u;
  }
  unsigned long long steps_done = 0;
  unsigned long long wpos = 0, wend = 0;  // the warp's reserved run of word slots

  auto flush = [&]() {
    if (la < 0) return;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (lcnt[k]) atomicAdd(&A.cnt[la * TILE + lrow(llb, lane, k)], (int)lcnt[k]);
      lcnt[k] = 0u;
    }
  };

  while (have) {
    const int buf = it & 1;
    __syncwarp();  // every lane is done reading the other buffer
    const bool hn = next_step(nxt);
    if (hn) issue(nxt, buf ^ 1);

    if (cur.a != la || cur.lb != llb) {  // (re)load the lane block into registers
      flush();
      la = cur.a;
      llb = cur.lb;
      const int na = min(TILE, n - la * TILE);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int il = lrow(llb, lane, k);
        lvalid[k] = il < na;
        const int i = la * TILE + (lvalid[k] ? il : 0);
        const float4* r4 = reinterpret_cast<const float4*>(A.rec + (size_t)i * S);
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
        if constexpr (Lanes<D, KP>::PAIRED) {
#pragma unroll
          for (int q = 0; q < D; ++q) {
            if (k & 1) L.c2[k >> 1][q].y = c[q];
            else L.c2[k >> 1][q].x = c[q];
          }
          if (k & 1) L.t2[k >> 1].y = tmp[D];
          else L.t2[k >> 1].x = tmp[D];
        } else {
#pragma unroll
          for (int q = 0; q < Lanes<D, KP>::DP; ++q) L.v2[k][q] = make_float2(c[2 * q], c[2 * q + 1]);
          L.v1[k] = c[D - 1];
          L.t[k] = tmp[D];
        }
      }
    }

    if (hn) cp_async_wait<1>();  // this step's group is complete
    else cp_async_wait<0>();
    __syncwarp();
    const float* st = stage + (size_t)buf * G::STAGE;
    uint32_t acc[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) acc[k] = 0u;
    if constexpr (STRIDED) {  // warp-uniform: the step's row-pair mask
#ifndef DS_HALF_SWAP
#define DS_HALF_SWAP 1
#endif
      if (cur.pm == 3) {
        pair_loop<D, F, SAFE, 0, 4>(L, st, eps32, z2, acc);
      } else if (!DS_HALF_SWAP) {
        if (cur.pm == 1) pair_loop<D, F, SAFE, 0, 2>(L, st, eps32, z2, acc);
        else pair_loop<D, F, SAFE, 2, 4>(L, st, eps32, z2, acc);
      } else {
        // one half-step loop body for both halves (less hot code: the 2-D kernel's warps
        // stall on instruction fetch): lane points 2-3 are swapped into 0-1 and back
        auto swap_halves = [&]() {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
#pragma unroll
            for (int q = 0; q < Lanes<D, KP>::DP; ++q) {
              const float2 t = L.v2[k][q];
              L.v2[k][q] = L.v2[k + 2][q];
              L.v2[k + 2][q] = t;
            }
            const float t1 = L.v1[k];
            L.v1[k] = L.v1[k + 2];
            L.v1[k + 2] = t1;
            const float tt = L.t[k];
            L.t[k] = L.t[k + 2];
            L.t[k + 2] = tt;
          }
        };
        if (cur.pm == 2) swap_halves();
        pair_loop<D, F, SAFE, 0, 2>(L, st, eps32, z2, acc);
        if (cur.pm == 2) {
          swap_halves();
          // lane points 0-1 are compared (bit = in range); the epilogue inverts lane
          // points k >= KC (sign-bit words: bit = out of range), so those are stored inverted
          acc[2] = 2 < KC ? acc[0] : ~acc[0];
          acc[3] = 3 < KC ? acc[1] : ~acc[1];
          acc[0] = 0u;
          acc[1] = 0u;
        }
      }
    } else {
      pair_loop<D, F, SAFE, 0, KP>(L, st, eps32, z2, acc);
    }
    steps_done += (STRIDED && cur.pm != 3) ? 2 : KP;  // lane points evaluated

    const int nb = min(TILE, n - cur.b * TILE);
    const uint32_t vm = valid_mask(nb - cur.jw * 32);
    const bool self = cur.a == cur.b && cur.jw < (cur.lb + 1) * KP;
    uint32_t w[KP];
    uint32_t any = 0u;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const bool ev = !STRIDED || ((cur.pm >> (k >> 1)) & 1);  // lane point k evaluated
      w[k] = (lvalid[k] && ev) ? ((k < KC ? acc[k] : ~acc[k]) & vm) : 0u;
      lcnt[k] += __popc(w[k]);
      any |= w[k];
    }
    unsigned long long base = 0;
    int total = 0;
    if (__any_sync(0xffffffffu, any != 0u)) {
      if (!self) {
        const uint32_t v = column_counts<KP>(w, lane);
        if (v) atomicAdd(&A.cnt[cur.b * TILE + cur.jw * 32 + lane], (int)v);
      } else {
#pragma unroll
        for (int k = 0; k < KP; ++k)  // keep columns j >= row (incl. the self pair)
          w[k] &= diag_keep(lrow(llb, lane, k) - cur.jw * 32);
      }
      // append the non-zero words into the warp's reserved run
      // word order: lane-major, then k; offsets from one ballot per k (no shuffle chain)
      const uint32_t lt = (1u << lane) - 1u;
      int excl = 0;
      total = 0;
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const uint32_t m = __ballot_sync(0xffffffffu, w[k] != 0u);
        excl += __popc(m & lt);
        total += __popc(m);
      }
      if (wpos + (unsigned long long)total > wend) {  // reserve WORD_RUN more slots
        unsigned long long r = 0;
        if (lane == 0) r = atomicAdd(A.words_count, (unsigned long long)WORD_RUN);
        wpos = __shfl_sync(0xffffffffu, r, 0);
        wend = wpos + WORD_RUN;
      }
      base = wpos;
      wpos += (unsigned long long)total;
      if (base + (unsigned long long)total <= A.words_cap) {  // else dropped: the host re-runs
        uint2* dst = A.words + base + excl;
        const uint32_t tag = ((uint32_t)lrow(llb, lane, 0) << 4) | (uint32_t)cur.jw;
        int o = 0;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          if (w[k]) dst[o] = make_uint2(w[k], tag + ((uint32_t)(lrow(0, 0, k)) << 4));
          o += w[k] ? 1 : 0;
        }
      }
    }
    if (lane == 0)
      A.uchunks[cur.u * WPR + cur.jw] =
          make_uint2((uint32_t)base, (uint32_t)total | ((uint32_t)(base >> 32) << 16));

    cur = nxt;
    have = hn;
    ++it;
  }
  flush();
  if (lane == 0 && steps_done)
    atomicAdd(A.pairs_done, steps_done * 32ull * 32ull);
}

// One launch serves both number ranges: the prep kernel's device flag selects the
// body (no host round trip); SAFE=false compares every predicate (inputs whose
// squares could overflow).
template <int D, int F>
__global__ void __launch_bounds__(Geo<D>::THREADS, Geo<D>::MINB) eps_unit_kernel(const UnitArgs A) {
  griddep_wait();
  stamp(A.stamps, ST_TILE);
  if (*A.unsafe_flag != 0) eps_unit_body<D, F, false>(A);
  else eps_unit_body<D, F, true>(A);
}

// ---- culled schedule: row-unit list ----------------------------------------------------
// Column block jw of lane block lb in kept tile pair (a, b) is evaluated unless it is
// structurally empty (struct_mask) or, for d <= 4, every 32-point row block of the lane
// block is provably out of range of it: the bound of keep_item, in double, on the row
// block box and the column block box (block_bounds_kernel). The row blocks that are not
// also give the step's row-pair mask: lane point k of every lane is row block k of the
// lane block, so a pair of row blocks (0-1, 2-3) without a possible pair is skipped by
// the eps kernel (C2: 28 % of the pairs of the kept column blocks).
// Row-pair mask of (lane block lb of tile a) x (column block jw of tile b), d <= 4 (KP =
// 4): bit 0 if row block 0 or 1 may hold an in-range pair, bit 1 for row blocks 2-3.
// rb: the lane block's 4 row-block boxes (BS floats each), nrb of them valid; cb: the
// column block's box (both staged in shared memory by pair_masks).
template <int DP>
__device__ __forceinline__ uint32_t box_pairs(const float* rb, int nrb, const float* cb, float eps32,
                                              int formula) {
  // keep_item's bound in float with directed rounding: every operation rounds toward a
  // smaller bound (gaps, squares and sums down, the subtracted rounding slack up), so
  // the float bound is below the exact one and culling stays exact; the constants carry
  // an extra 1e-6 / 0.1 % margin for their own rounding
  constexpr int BS = 2 * DP + 1;
  constexpr float u = 1.0f / 16777216.0f;
  constexpr float C1 = 1.0f - 12.0f * DP * u - 1e-6f;                   // (1 - 12 DP u)(1 - 1e-12)
  constexpr float C2 = 8.0f * (2.0f * DP + 3.0f) * u * 1.001f * 1.001f;  // 4 (2DP+3) u 2 w 1.001
  float c[BS];
#pragma unroll
  for (int q = 0; q < BS; ++q) c[q] = cb[q];
  uint32_t pm = 0u;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k >= nrb) break;
    const float* r = rb + k * BS;
    float L = 0.f;
#pragma unroll
    for (int q = 0; q < DP; ++q) {
      const float g = fmaxf(0.f, fmaxf(__fsub_rd(c[q], r[DP + q]), __fsub_rd(r[q], c[DP + q])));
      L = __fadd_rd(L, __fmul_rd(g, g));
    }
    float bound = __fmul_rd(L, C1);
    if (formula == DS_FORMULA_ALGEBRAIC) bound = __fsub_rd(bound, __fmul_ru(fmaxf(r[2 * DP], c[2 * DP]), C2));
    if (!(bound > eps32)) pm |= 1u << (k >> 1);  // NaN bounds keep the block
  }
  return pm;
}

// 0: not evaluated; else the row-pair mask (3 where no box test applies)
__device__ __forceinline__ uint32_t unit_pairs(const float* __restrict__ blk, const float* rb, int nrb,
                                               const float* cb, int dpad, int64_t n, int KP, int a,
                                               int b, int lb, int jw, float eps32, int formula,
                                               bool unsafe) {
  const int64_t na = min((int64_t)TILE, n - (int64_t)a * TILE);
  const int64_t nb = min((int64_t)TILE, n - (int64_t)b * TILE);
  if (jw * 32 >= nb || lb * 32 * KP >= na) return 0u;
  if (a == b && jw < lb * KP) return 0u;
  if (unsafe || !blk || KP != 4 || (a == b && jw < (lb + 1) * KP)) return 3u;
  switch (dpad) {
    case 1: return box_pairs<1>(rb, nrb, cb, eps32, formula);
    case 2: return box_pairs<2>(rb, nrb, cb, eps32, formula);
    case 3: return box_pairs<3>(rb, nrb, cb, eps32, formula);
    case 4: return box_pairs<4>(rb, nrb, cb, eps32, formula);
    default: return 3u;
  }
}

// Column masks of two lane blocks (2p, 2p + 1) of item (a, b): lanes 0-15 test the 16
// column blocks of the first, lanes 16-31 those of the second. keep: evaluated column
// blocks; pair0 / pair1: those whose row-pair mask has bit 0 / bit 1. rb / cbs: the
// item's 16 row-block boxes and 16 column-block boxes, staged by stage_boxes.
struct PairMasks {
  uint32_t keep, pair0, pair1;
};
__device__ __forceinline__ void stage_boxes(const float* __restrict__ blk, float* rb, float* cbs,
                                            int dpad, int64_t n, int KP, int a, int b, int lane) {
  if (!(blk && KP == 4 && dpad <= 4)) return;
  const int BS = 2 * dpad + 1;
  const int64_t nblk = (n + 31) / 32;
  const int64_t r0 = (int64_t)a * WPR, c0 = (int64_t)b * WPR;  // first row / column block
  __syncwarp();  // the previous item's readers are done
  for (int i = lane; i < WPR * BS; i += 32) {  // all loads issued together: one round trip
    rb[i] = r0 + i / BS < nblk ? blk[r0 * BS + i] : 0.f;
    cbs[i] = c0 + i / BS < nblk ? blk[c0 * BS + i] : 0.f;
  }
  __syncwarp();
}
__device__ __forceinline__ PairMasks pair_masks(const float* __restrict__ blk, const float* rb,
                                                const float* cbs, int dpad, int64_t n, int KP, int a,
                                                int b, int p, float eps32, int formula, bool unsafe,
                                                int lane) {
  const int BS = 2 * dpad + 1;
  const int64_t nblk = (n + 31) / 32;
  const int64_t r0 = (int64_t)a * WPR + (int64_t)(2 * p) * 4;  // first row block (KP = 4)
  rb += (2 * p) * 4 * BS;
  const int h = lane >> 4;
  const int lb = 2 * p + h;
  const int nrb = (int)min((int64_t)4, nblk - (r0 + 4 * h));
  const uint32_t pm = unit_pairs(blk, rb + 4 * BS * h, nrb, cbs + (lane & 15) * BS, dpad, n, KP, a,
                                 b, lb, lane & 15, eps32, formula, unsafe);
  return {__ballot_sync(0xffffffffu, pm != 0u), __ballot_sync(0xffffffffu, (pm & 1u) != 0u),
          __ballot_sync(0xffffffffu, (pm & 2u) != 0u)};
}

// For KP = 4 (d <= 8) a (lane block, tile pair) with many kept column blocks is
// listed as several row units of at most 2 (n <= UNIT_SMALL_N) or 4 column blocks each
// (finer work balance at the tail); a tile pair then has at most 32 units x WPR = 512
// chunk entries, the bound the union kernels hold in shared memory (MAX_UPT); KP <= 2
// units are unsplit (16 per tile pair). Measured (A/B): pieces of 2 cut C1's eps launch
// 11.2 -> 9.3 us and C2's by 1.2 us, but cost C3 / C5 15-60 us in union_links
// (per-unit overhead), hence the size switch.
__device__ __forceinline__ int unit_cols(int KP, int64_t n) {
  return KP == 4 ? (n <= UNIT_SMALL_N ? 2 : 4) : 16;
}

// The row-unit list of this launch's shard, one kernel: warp per kept item (items are
// dealt to the shards cyclically, q = rank + k * world, which spreads the dense and
// the sparse regions evenly), masks by pair_masks, split into pieces, one atomic per
// item reserves its list run. The order of the runs is arbitrary; item_units[q]
// records {first unit, units} for the directory.
__global__ void __launch_bounds__(256, 4) unit_list_kernel(
    const float* __restrict__ blk, int dpad, int64_t n, int KP, float eps32, int formula,
    const uint32_t* __restrict__ unsafe_flag, const uint32_t* __restrict__ items,
    const unsigned long long* __restrict__ kept, int rank, int world, uint2* __restrict__ list,
    unsigned long long cap, unsigned long long* __restrict__ unit_count,
    uint2* __restrict__ item_units, uint2* __restrict__ diag_range) {
  griddep_wait();
  constexpr int W = 8;  // warps per CTA; one list reservation per CTA and round
  __shared__ int wcnt[W];
  __shared__ unsigned long long wpos[W];
  __shared__ uint32_t msk[W][3][8];  // per warp and lane-block pair: keep, pair0, pair1
  __shared__ float rbs[W][WPR * 9];  // per warp: the row-block boxes of tile a
  __shared__ float cbs[W][WPR * 9];  // per warp: the column-block boxes of tile b
  const int64_t K = (int64_t)*kept;
  const bool unsafe = *unsafe_flag != 0;
  const int LB = TILE / (32 * KP);
  const int uc = unit_cols(KP, n);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t mine = K > rank ? (K - rank + world - 1) / world : 0;
  for (int64_t t0 = (int64_t)blockIdx.x * W; t0 < mine; t0 += (int64_t)gridDim.x * W) {
    const int64_t t = t0 + warp;
    const int64_t q = rank + t * world;
    uint32_t ab = 0u;
    int c = 0;
    if (t < mine) {  // warp-uniform
      ab = items[q];
      const int a = (int)(ab >> 16), b = (int)(ab & 0xffffu);
      stage_boxes(blk, rbs[warp], cbs[warp], dpad, n, KP, a, b, lane);
      for (int p = 0; p < LB / 2; ++p) {
        const PairMasks pmk = pair_masks(blk, rbs[warp], cbs[warp], dpad, n, KP, a, b, p, eps32,
                                         formula, unsafe, lane);
        if (lane == 0) {
          msk[warp][0][p] = pmk.keep;
          msk[warp][1][p] = pmk.pair0;
          msk[warp][2][p] = pmk.pair1;
        }
        c += (__popc(pmk.keep & 0xffffu) + uc - 1) / uc + (__popc(pmk.keep >> 16) + uc - 1) / uc;
      }
    }
    if (lane == 0) wcnt[warp] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < W; ++w) tot += wcnt[w];
      unsigned long long base = tot ? atomicAdd(unit_count, (unsigned long long)tot) : 0ull;
      for (int w = 0; w < W; ++w) {
        wpos[w] = base;
        base += (unsigned long long)wcnt[w];
      }
    }
    __syncthreads();
    if (t < mine) {  // warp-uniform; lane j of half h writes the unit starting at column j
      unsigned long long pos = wpos[warp];
      if (lane == 0) {
        const uint2 iu = make_uint2((uint32_t)pos, (uint32_t)c | ((uint32_t)(pos >> 32) << 16));
        item_units[q] = iu;
        if ((ab >> 16) == (ab & 0xffffu)) diag_range[ab >> 16] = iu;  // for union_diag
      }
      const int h = lane >> 4, j = lane & 15;
      for (int p = 0; p < LB / 2; ++p) {
        const uint32_t keep = msk[warp][0][p];
        const uint32_t m = h ? keep >> 16 : keep & 0xffffu;
        const int np0 = (__popc(keep & 0xffffu) + uc - 1) / uc;  // units of lane block 2p
        const int np1 = (__popc(keep >> 16) + uc - 1) / uc;
        const int r = __popc(m & ((1u << j) - 1u));  // rank of column j among kept ones
        if (((m >> j) & 1u) && r % uc == 0) {  // first column of a unit: up to uc columns
          const uint32_t m0 = h ? msk[warp][1][p] >> 16 : msk[warp][1][p] & 0xffffu;
          const uint32_t m1 = h ? msk[warp][2][p] >> 16 : msk[warp][2][p] & 0xffffu;
          uint32_t rest = m & ~((1u << j) - 1u), piece = 0u, sub = 0u;  // sub: 2-bit row-pair
          for (int k = 0; k < uc && rest; ++k) {                         // masks in column order
            const uint32_t bit = rest & (0u - rest);
            piece |= bit;
            if (k < 4) sub |= (((m0 & bit) ? 1u : 0u) | ((m1 & bit) ? 2u : 0u)) << (2 * k);
            rest &= rest - 1u;
          }
          const unsigned long long at = pos + (h ? np0 : 0) + r / uc;
          // {a << 16 | b, column mask | lane block << 16 | row-pair masks << 20 (KP = 4)}
          if (at < cap) list[at] = make_uint2(ab, ((uint32_t)(2 * p + h) << 16) | piece | (sub << 20));
        }
        pos += (unsigned long long)(np0 + np1);
      }
    }
    __syncthreads();  // wcnt / wpos are rewritten by the next round
  }
}

// ---- directory of tile pairs with words (for the union kernels) ------------------
// Per item: its row units [lo, hi) (culled: item_units of this shard's items; dense:
// the triangle order, clipped to the shard) own chunk entries [lo * WPR, hi * WPR);
// the item gets a directory entry if any of them holds words.
template <int KP>
__global__ void unit_dir_kernel(const UnitArgs A, int64_t all_items, const uint2* __restrict__ item_units,
                                const unsigned long long* __restrict__ kept, uint4* __restrict__ dir,
                                unsigned long long* __restrict__ dir_count) {
  griddep_wait();
  constexpr int LB = TILE / (32 * KP);
  long long r_lo, r_hi;
  unit_range(A, r_lo, r_hi);
  const int64_t K = A.unit_list ? (int64_t)*kept : all_items;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < K; q += nwarps) {
    long long lo, hi;
    if (A.unit_list) {
      if (q % A.shard_world != A.shard_rank) continue;
      const uint2 iu = item_units[q];
      lo = (long long)iu.x | ((long long)(iu.y >> 16) << 32);
      hi = lo + (long long)(iu.y & 0xffffu);
      if (hi > r_hi) hi = r_hi;  // list overflow: the host re-runs
    } else {
      lo = q * LB;
      hi = lo + LB;
      lo = lo > r_lo ? lo : r_lo;
      hi = hi < r_hi ? hi : r_hi;
    }
    if (lo >= hi) continue;
    const long long c_lo = lo * WPR, c_hi = hi * WPR;
    uint32_t words = 0;
    for (long long e = c_lo + lane; e < c_hi; e += 32) words += A.uchunks[e].y & 0xffffu;
#pragma unroll
    for (int off = 16; off; off >>= 1) words += __shfl_xor_sync(0xffffffffu, words, off);
    if (lane == 0 && words) {
      int a, b;
      if (A.item_list) {
        const uint32_t ab = A.item_list[q];
        a = (int)(ab >> 16);
        b = (int)(ab & 0xffffu);
      } else {
        decode_item(q, A.T, a, b);
      }
      const unsigned long long e = atomicAdd(dir_count, 1ull);
      dir[e] = make_uint4(((uint32_t)a << 16) | (uint32_t)b, (uint32_t)c_lo, (uint32_t)(c_hi - c_lo),
                          (uint32_t)((unsigned long long)c_lo >> 32));
    }
  }
}

// One point of the general prep path with the record width known at compile time: the
// point's d coordinates are loaded together (independent loads in flight, where the
// runtime-width loop was a chain of one load at a time: C4, 16-D, prep 70 us) and the
// record is written as float4s.
template <int DP>
__device__ __forceinline__ void prep_point(const double* __restrict__ coords, int64_t i, int d,
                                           float* __restrict__ rec, float (&mn)[4], float (&mx)[4],
                                           bool& bad) {
  constexpr int S = ((DP + 1) + 3) / 4 * 4;
  const double* src = coords + i * d;
  double x[DP];
#pragma unroll
  for (int c = 0; c < DP; ++c) x[c] = c < d ? src[c] : 0.0;
  float r[S];
  float p = 0.f;
#pragma unroll
  for (int c = 0; c < DP; ++c) {
    const float v = __double2float_rn(x[c]);  // kernels.py:148-150 (0.0 -> +0 padding)
    r[c] = v;
    if (c < 4) {  // NaN coordinates drop out of fminf / fmaxf
      mn[c] = fminf(mn[c], v);
      mx[c] = fmaxf(mx[c], v);
    }
    const float sq = __fmul_rn(v, v);
    p = (c == 0) ? sq : __fadd_rn(p, sq);  // kernels.py:388-391, left to right
    bad |= !(fabsf(v) <= SAFE_ABS);
  }
  r[DP] = p;
#pragma unroll
  for (int c = DP + 1; c < S; ++c) r[c] = 0.f;
  float4* dst = reinterpret_cast<float4*>(rec + i * S);
#pragma unroll
  for (int v = 0; v < S / 4; ++v) dst[v] = make_float4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
}

// ---- prep: narrow to float32 (RN), squared norms, padded records ------------------
// Also reduces the bounding box of the first min(d, 4) coordinates for the spatial
// sort (bbox != nullptr): grid-stride threads keep running min/max, then a warp and a
// block reduction and one atomic per block and dimension.
__global__ void __launch_bounds__(256) prep_kernel(const double* __restrict__ coords, int64_t n,
                                                   int d, int dpad, int S, float* __restrict__ rec,
                                                   uint32_t* unsafe_flag,
                                                   unsigned long long* stamps,
                                                   unsigned int* __restrict__ bbox,
                                                   int32_t* __restrict__ cnt) {
  griddep_wait();
  stamp(stamps, ST_PREP);
  float mn[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
  float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i_gen = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (d == 2 && dpad == 2 && S == 4 && (reinterpret_cast<uintptr_t>(coords) & 15u) == 0) {
    // 2-D: one 16-byte load and one 16-byte store per point, four points per thread in
    // flight (the general loop below is a chain of dependent loads per point)
    const double2* src2 = reinterpret_cast<const double2*>(coords);
    float4* dst4 = reinterpret_cast<float4*>(rec);
    for (; i_gen < n; i_gen += 4 * stride) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i_gen + u * stride;
        v[u] = i < n ? src2[i] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i_gen + u * stride;
        if (i >= n) continue;
        const float x = __double2float_rn(v[u].x), y = __double2float_rn(v[u].y);  // kernels.py:148-150
        const float p = __fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y));  // kernels.py:388-391
        dst4[i] = make_float4(x, y, p, 0.f);
        mn[0] = fminf(mn[0], x);
        mx[0] = fmaxf(mx[0], x);
        mn[1] = fminf(mn[1], y);
        mx[1] = fmaxf(mx[1], y);
        bad |= !(fabsf(x) <= SAFE_ABS) || !(fabsf(y) <= SAFE_ABS);
        if (cnt) cnt[i] = 0;
      }
    }
  }
  const bool fixed = S == ((dpad + 1) + 3) / 4 * 4 &&
                     (dpad == 4 || dpad == 8 || dpad == 16 || dpad == 32);
  if (fixed) {
    for (int64_t i = i_gen; i < n; i += stride) {
      if (dpad == 4) prep_point<4>(coords, i, d, rec, mn, mx, bad);
      else if (dpad == 8) prep_point<8>(coords, i, d, rec, mn, mx, bad);
      else if (dpad == 16) prep_point<16>(coords, i, d, rec, mn, mx, bad);
      else prep_point<32>(coords, i, d, rec, mn, mx, bad);
      if (cnt) cnt[i] = 0;
    }
    i_gen = n;  // done: skip the general loop
  }
  for (int64_t i = i_gen; i < n; i += stride) {
    const double* src = coords + i * d;
    float* dst = rec + i * S;
    float p = 0.f;
    for (int c = 0; c < dpad; ++c) {
      const float v = c < d ? __double2float_rn(src[c]) : 0.f;  // kernels.py:148-150
      dst[c] = v;
      if (c < 4) {  // NaN coordinates drop out of fminf / fmaxf
        mn[c] = fminf(mn[c], v);
        mx[c] = fmaxf(mx[c], v);
      }
      const float sq = __fmul_rn(v, v);
      p = (c == 0) ? sq : __fadd_rn(p, sq);  // kernels.py:388-391, left to right
      bad |= !(fabsf(v) <= SAFE_ABS);
    }
    dst[dpad] = p;
    for (int c = dpad + 1; c < S; ++c) dst[c] = 0.f;
    if (cnt) cnt[i] = 0;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(unsafe_flag, 1u);
  if (!bbox) return;
  __shared__ unsigned int smn[4], smx[4];  // smn holds ~ord(min): both reduce with max
  if (threadIdx.x < 4) {
    smn[threadIdx.x] = 0u;
    smx[threadIdx.x] = 0u;
  }
  __syncthreads();
  const int kd = d < 4 ? d : 4;
  for (int k = 0; k < kd; ++k) {
    float a = mn[k], b = mx[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      a = fminf(a, __shfl_xor_sync(0xffffffffu, a, off));
      b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, off));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMax(&smn[k], ~ord_bits(a));
      atomicMax(&smx[k], ord_bits(b));
    }
  }
  __syncthreads();
  if (threadIdx.x < kd) {
    atomicMax(&bbox[threadIdx.x], smn[threadIdx.x]);
    atomicMax(&bbox[4 + threadIdx.x], smx[threadIdx.x]);
  }
}

// ---- tile culling ------------------------------------------------------------------
// Per tile: coordinate bounding box (float32, exact) and max squared norm.
__global__ void tile_bounds_kernel(const float* __restrict__ rec, int64_t n, int dpad, int S,
                                   float* __restrict__ lo, float* __restrict__ hi,
                                   float* __restrict__ maxnorm, unsigned int* __restrict__ super) {
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
      if (super) super_box_add(super, tile, dpad, k, mn, mx);
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

// Row-wise culling for T <= CULL_ROWS_MAX tiles (two launches instead of flags + scan
// + scatter): pass 1 counts the kept pairs of each tile row a (CTA per row); pass 2
// sums the counts of the rows before a (every CTA itself: O(T) reads, L2-resident)
// and writes row a's kept pairs in order with a block scan. Same list, same order.
constexpr int64_t CULL_ROWS_MAX = 8192;
constexpr int CULL_T = 256;

__device__ __forceinline__ int block_sum(int v, int* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();  // red may still be read by a previous call
  if (lane == 0) red[wid] = v;
  __syncthreads();
  int t = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;
}

__global__ void __launch_bounds__(CULL_T) cull_rows_kernel(
    const float* __restrict__ lo, const float* __restrict__ hi, const float* __restrict__ maxnorm,
    int dpad, int64_t T, float eps32, int formula, const uint32_t* __restrict__ unsafe_flag,
    int32_t* __restrict__ rowcnt) {
  griddep_wait();
  __shared__ int red[CULL_T / 32];
  const bool unsafe = *unsafe_flag != 0;
  for (int64_t a = blockIdx.x; a < T; a += gridDim.x) {
    int c = 0;
    for (int64_t b = a + threadIdx.x; b < T; b += blockDim.x)
      c += keep_item(lo, hi, maxnorm, dpad, (int)a, (int)b, eps32, formula, unsafe) ? 1 : 0;
    const int t = block_sum(c, red);
    if (threadIdx.x == 0) rowcnt[a] = t;
  }
}

// One GPU (no shard needs the same order): each row's kept pairs are gathered in shared
// memory (T <= CULL_ROWS_MAX entries) and appended to the list with one reservation per
// row — one launch instead of cull_rows + cull_write; the list order across rows then
// depends on scheduling, which no result does.
__global__ void __launch_bounds__(CULL_T) cull_append_kernel(
    const float* __restrict__ lo, const float* __restrict__ hi, const float* __restrict__ maxnorm,
    int dpad, int64_t T, float eps32, int formula, const uint32_t* __restrict__ unsafe_flag,
    uint32_t* __restrict__ list, unsigned long long* __restrict__ count) {
  griddep_wait();
  extern __shared__ uint32_t kb[];  // T entries
  __shared__ int nkb;
  __shared__ unsigned long long kbase;
  const bool unsafe = *unsafe_flag != 0;
  const int lane = threadIdx.x & 31;
  for (int64_t a = blockIdx.x; a < T; a += gridDim.x) {
    if (threadIdx.x == 0) nkb = 0;
    __syncthreads();
    for (int64_t b0 = a; b0 < T; b0 += blockDim.x) {
      const int64_t b = b0 + threadIdx.x;
      const bool k = b < T && keep_item(lo, hi, maxnorm, dpad, (int)a, (int)b, eps32, formula, unsafe);
      const uint32_t bal = __ballot_sync(0xffffffffu, k);
      int at = 0;
      if (lane == 0 && bal) at = atomicAdd(&nkb, __popc(bal));
      at = __shfl_sync(0xffffffffu, at, 0);
      if (k) kb[at + __popc(bal & ((1u << lane) - 1u))] = ((uint32_t)a << 16) | (uint32_t)b;
    }
    __syncthreads();
    if (threadIdx.x == 0) kbase = nkb ? atomicAdd(count, (unsigned long long)nkb) : 0ull;
    __syncthreads();
    for (int e = threadIdx.x; e < nkb; e += blockDim.x) list[kbase + e] = kb[e];
    __syncthreads();  // nkb / kb are rewritten by the next row
  }
}

__global__ void __launch_bounds__(CULL_T) cull_write_kernel(
    const float* __restrict__ lo, const float* __restrict__ hi, const float* __restrict__ maxnorm,
    int dpad, int64_t T, float eps32, int formula, const uint32_t* __restrict__ unsafe_flag,
    const int32_t* __restrict__ rowcnt, uint32_t* __restrict__ list, int32_t* __restrict__ total_kept,
    unsigned long long* __restrict__ count) {
  griddep_wait();
  __shared__ int red[CULL_T / 32];
  __shared__ int wsum[CULL_T / 32];
  const bool unsafe = *unsafe_flag != 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t a = blockIdx.x; a < T; a += gridDim.x) {
    int p = 0;
    for (int64_t r = threadIdx.x; r < a; r += blockDim.x) p += rowcnt[r];
    int pos = block_sum(p, red);  // kept pairs of the rows before a
    for (int64_t b0 = a; b0 < T; b0 += blockDim.x) {
      const int64_t b = b0 + threadIdx.x;
      const bool k = b < T && keep_item(lo, hi, maxnorm, dpad, (int)a, (int)b, eps32, formula, unsafe);
      const uint32_t bal = __ballot_sync(0xffffffffu, k);
      __syncthreads();  // wsum of the previous chunk is consumed
      if (lane == 0) wsum[wid] = __popc(bal);
      __syncthreads();
      int before = 0, all = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        before += w < wid ? wsum[w] : 0;
        all += wsum[w];
      }
      if (k) list[pos + before + __popc(bal & ((1u << lane) - 1u))] = ((uint32_t)a << 16) | (uint32_t)b;
      pos += all;
    }
    if (a == T - 1 && threadIdx.x == 0) {
      *total_kept = pos;
      *count = (unsigned long long)pos;
    }
  }
}

// keep_item's bound in float with directed rounding (every operation rounds toward a
// smaller bound; see box_pairs), on box a = {alo, ahi, wa} and box b: the test of the
// hierarchical culling, d <= 4. Exact culling as keep_item (never drops a pair whose
// float32 result could be <= eps32).
template <int DP>
__device__ __forceinline__ bool keep_box(const float* alo, const float* ahi, float wa, const float* blo,
                                         const float* bhi, float wb, float eps32, int formula) {
  constexpr float u = 1.0f / 16777216.0f;
  constexpr float C1 = 1.0f - 12.0f * DP * u - 1e-6f;                   // (1 - 12 DP u)(1 - 1e-12)
  constexpr float C2 = 4.0f * (2.0f * DP + 3.0f) * u * 1.001f * 1.001f;  // 4 (2DP+3) u 1.001
  float L = 0.f;
#pragma unroll
  for (int k = 0; k < DP; ++k) {
    const float g = fmaxf(0.f, fmaxf(__fsub_rd(blo[k], ahi[k]), __fsub_rd(alo[k], bhi[k])));
    L = __fadd_rd(L, __fmul_rd(g, g));
  }
  float bound = __fmul_rd(L, C1);
  if (formula == DS_FORMULA_ALGEBRAIC) bound = __fsub_rd(bound, __fmul_ru(__fadd_ru(wa, wb), C2));
  return !(bound > eps32);  // NaN bounds keep the pair
}

// Hierarchical row culling (d <= 4): a CTA per tile row a tests the super tiles at or
// after a's first (one thread each), then one warp per kept super tile tests its 32
// tiles b >= a — the kept pairs come out in item order (super tiles in order, tiles in
// order within one), the same list as cull_rows / cull_write. MODE 0 counts the row's
// kept pairs (rowcnt), MODE 1 writes them at the row's offset (two kernels: the order
// every rank of a sharded run must share); MODE 2 (one GPU) appends them in any order,
// one list reservation per row (one kernel; count = the kept total).
template <int DP, int MODE>
__global__ void __launch_bounds__(CULL_T) cull_super_kernel(
    const float* __restrict__ lo, const float* __restrict__ hi, const float* __restrict__ maxnorm,
    const unsigned int* __restrict__ super, int64_t T, float eps32, int formula,
    const uint32_t* __restrict__ unsafe_flag, int32_t* __restrict__ rowcnt, uint32_t* __restrict__ list,
    int32_t* __restrict__ total_kept, unsigned long long* __restrict__ count) {
  griddep_wait();
  constexpr int W = CULL_T / 32;
  __shared__ int red[W];
  __shared__ int wsum[W];
  __shared__ int ks[CULL_T];  // kept super tiles of the row, in order
  __shared__ int nks;
  constexpr int KB = 1024;    // MODE 2: the row's kept tiles, flushed to the list in batches
  __shared__ uint32_t kb[MODE == 2 ? KB : 1];
  __shared__ int nkb;
  __shared__ unsigned long long kbase;
  const bool unsafe = *unsafe_flag != 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t NS = (T + SUPER - 1) / SUPER;
  for (int64_t a = blockIdx.x; a < T; a += gridDim.x) {
    float alo[DP], ahi[DP];
#pragma unroll
    for (int k = 0; k < DP; ++k) {
      alo[k] = lo[a * DP + k];
      ahi[k] = hi[a * DP + k];
    }
    const float wa = maxnorm[a];
    int pos = 0;
    if (MODE == 2 && threadIdx.x == 0) nkb = 0;
    if (MODE == 1) {  // kept pairs of the rows before a (O(T) reads, L2-resident)
      int p = 0;
      for (int64_t r = threadIdx.x; r < a; r += blockDim.x) p += rowcnt[r];
      pos = block_sum(p, red);
    }
    int row_total = 0;
    for (int64_t s0 = a / SUPER; s0 < NS; s0 += CULL_T) {  // super tiles, CULL_T at a time
      const int64_t sb = s0 + threadIdx.x;
      bool k = false;
      if (sb < NS) {
        if (unsafe) {
          k = true;
        } else {
          const unsigned int* b = super + sb * SUPER_BS;
          float blo[DP], bhi[DP];
#pragma unroll
          for (int q = 0; q < DP; ++q) {
            blo[q] = unord_bits(~b[q]);
            bhi[q] = unord_bits(b[DP + q]);
          }
          k = keep_box<DP>(alo, ahi, wa, blo, bhi, unord_bits(b[2 * DP]), eps32, formula);
        }
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, k);
      __syncthreads();  // ks / wsum of the previous round are consumed
      if (lane == 0) wsum[wid] = __popc(bal);
      __syncthreads();
      int before = 0, all = 0;
      for (int w = 0; w < W; ++w) {
        before += w < wid ? wsum[w] : 0;
        all += wsum[w];
      }
      if (k) ks[before + __popc(bal & ((1u << lane) - 1u))] = (int)sb;
      if (threadIdx.x == 0) nks = all;
      __syncthreads();
      const int nk = nks;
      for (int i0 = 0; i0 < nk; i0 += W) {  // one warp per kept super tile
        const int i = i0 + wid;
        const int64_t b = i < nk ? (int64_t)ks[i] * SUPER + lane : T;
        bool kt = false;
        if (b < T && b >= a) {
          if (unsafe || b == a) {
            kt = true;
          } else {
            float blo[DP], bhi[DP];
#pragma unroll
            for (int q = 0; q < DP; ++q) {
              blo[q] = lo[b * DP + q];
              bhi[q] = hi[b * DP + q];
            }
            kt = keep_box<DP>(alo, ahi, wa, blo, bhi, maxnorm[b], eps32, formula);
          }
        }
        const uint32_t tb = __ballot_sync(0xffffffffu, kt);
        if (MODE == 0) {
          row_total += lane == 0 ? __popc(tb) : 0;
        } else if (MODE == 2) {
          int at = 0;
          if (lane == 0 && tb) at = atomicAdd(&nkb, __popc(tb));
          at = __shfl_sync(0xffffffffu, at, 0);
          if (kt) kb[at + __popc(tb & ((1u << lane) - 1u))] = ((uint32_t)a << 16) | (uint32_t)b;
          __syncthreads();
          if (nkb > KB - CULL_T || i0 + W >= nk) {  // flush before the buffer could overflow
            if (threadIdx.x == 0) kbase = nkb ? atomicAdd(count, (unsigned long long)nkb) : 0ull;
            __syncthreads();
            for (int e = threadIdx.x; e < nkb; e += CULL_T) list[kbase + e] = kb[e];
            __syncthreads();
            if (threadIdx.x == 0) nkb = 0;
            __syncthreads();
          }
        } else {
          __syncthreads();
          if (lane == 0) wsum[wid] = __popc(tb);
          __syncthreads();
          int bw = 0, aw = 0;
          for (int w = 0; w < W; ++w) {
            bw += w < wid ? wsum[w] : 0;
            aw += wsum[w];
          }
          if (kt) list[pos + bw + __popc(tb & ((1u << lane) - 1u))] = ((uint32_t)a << 16) | (uint32_t)b;
          pos += aw;
        }
      }
    }
    if (MODE == 0) {
      const int t = block_sum(row_total, red);
      if (threadIdx.x == 0) rowcnt[a] = t;
    } else if (MODE == 1 && a == T - 1 && threadIdx.x == 0) {
      *total_kept = pos;
      *count = (unsigned long long)pos;
    }
  }
}

template <int DP>
cudaError_t launch_cull_super(const float* lo, const float* hi, const float* maxnorm,
                              const unsigned int* super, int64_t T, float eps32, int formula,
                              const uint32_t* unsafe_flag, int32_t* rowcnt, uint32_t* list,
                              int32_t* total_kept, unsigned long long* count, bool ordered,
                              cudaStream_t s) {
  const unsigned g = (unsigned)std::min<int64_t>(T, 148 * 8);
  if (!ordered)  // count starts at zero (the per-call zero region)
    return launch_pdl(cull_super_kernel<DP, 2>, dim3(g), dim3(CULL_T), 0, s, lo, hi, maxnorm,
                      super, T, eps32, formula, unsafe_flag, (int32_t*)nullptr, list,
                      (int32_t*)nullptr, count);
  cudaError_t e = launch_pdl(cull_super_kernel<DP, 0>, dim3(g), dim3(CULL_T), 0, s, lo, hi,
                             maxnorm, super, T, eps32, formula, unsafe_flag, rowcnt,
                             (uint32_t*)nullptr, (int32_t*)nullptr, (unsigned long long*)nullptr);
  if (e != cudaSuccess) return e;
  return launch_pdl(cull_super_kernel<DP, 1>, dim3(g), dim3(CULL_T), 0, s, lo, hi, maxnorm, super,
                    T, eps32, formula, unsafe_flag, rowcnt, list, total_kept, count);
}

int pad_dim(int d) {
  if (d <= 4) return d;
  if (d <= 8) return 8;
  if (d <= 16) return 16;
  if (d <= 32) return 32;
  return 64;
}

template <int D, int F>
cudaError_t launch_df(const UnitArgs& a, int sm_count, cudaStream_t s) {
  using G = Geo<D>;
  auto kern = eps_unit_kernel<D, F>;
  // kernel attributes are per device: configure once per device (idempotent if raced)
  static std::atomic<int> per_sm_dev[DS_MAX_DEVICES] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int per_sm = dev < DS_MAX_DEVICES ? per_sm_dev[dev].load() : 0;
  if (per_sm == 0) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::THREADS, G::SMEM);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    if (dev < DS_MAX_DEVICES) per_sm_dev[dev].store(per_sm);
  }
  return launch_pdl(kern, dim3((unsigned)(sm_count * per_sm)), dim3(G::THREADS), G::SMEM, s, a);
}

template <int D>
cudaError_t launch_d(const UnitArgs& a, int formula, int sm_count, cudaStream_t s) {
  return formula == DS_FORMULA_ALGEBRAIC ? launch_df<D, DS_FORMULA_ALGEBRAIC>(a, sm_count, s)
                                         : launch_df<D, DS_FORMULA_DIRECT>(a, sm_count, s);
}

}  // namespace

int padded_dim(int d) { return pad_dim(d); }

cudaError_t launch_prep(const double* coords, int64_t n, int d, float* rec, uint32_t* unsafe_flag,
                        unsigned long long* stamps, unsigned int* bbox, int32_t* cnt,
                        cudaStream_t s) {
  const int dp = pad_dim(d);
  const int S = ((dp + 1) + 3) / 4 * 4;
  const int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  return launch_pdl(prep_kernel, dim3((unsigned)blocks), dim3(threads), 0, s, coords, n, d, dp, S,
                    rec, unsafe_flag, stamps, bbox, cnt);
}

cudaError_t launch_cull(const float* rec, int64_t n, int d, float eps32, int formula,
                        const uint32_t* unsafe_flag, float* lo, float* hi, float* maxnorm,
                        unsigned int* super, int32_t* flags, int32_t* partials,
                        int32_t* total_kept, uint32_t* list, unsigned long long* count,
                        bool bounds_ready, bool ordered, cudaStream_t s) {
  const int dp = pad_dim(d);
  const int S = ((dp + 1) + 3) / 4 * 4;
  const int64_t T = (n + TILE - 1) / TILE;
  if (dp > 4) super = nullptr;
  if (!bounds_ready)
    tile_bounds_kernel<<<(unsigned)T, 256, 0, s>>>(rec, n, dp, S, lo, hi, maxnorm, super);
  if (super && T <= CULL_ROWS_MAX) {  // hierarchical: super tiles first (d <= 4)
    switch (dp) {
      case 1: return launch_cull_super<1>(lo, hi, maxnorm, super, T, eps32, formula, unsafe_flag,
                                          flags, list, total_kept, count, ordered, s);
      case 2: return launch_cull_super<2>(lo, hi, maxnorm, super, T, eps32, formula, unsafe_flag,
                                          flags, list, total_kept, count, ordered, s);
      case 3: return launch_cull_super<3>(lo, hi, maxnorm, super, T, eps32, formula, unsafe_flag,
                                          flags, list, total_kept, count, ordered, s);
      default: return launch_cull_super<4>(lo, hi, maxnorm, super, T, eps32, formula, unsafe_flag,
                                           flags, list, total_kept, count, ordered, s);
    }
  }
  if (T <= CULL_ROWS_MAX) {  // rowcnt lives in the flags buffer (T <= T(T+1)/2 ints)
    const unsigned g = (unsigned)std::min<int64_t>(T, 148 * 8);
    if (!ordered)  // count starts at zero (the per-call zero region)
      return launch_pdl(cull_append_kernel, dim3(g), dim3(CULL_T), (size_t)T * 4, s,
                        (const float*)lo, (const float*)hi, (const float*)maxnorm, dp, T, eps32,
                        formula, unsafe_flag, list, count);
    cudaError_t e = launch_pdl(cull_rows_kernel, dim3(g), dim3(CULL_T), 0, s, (const float*)lo,
                               (const float*)hi, (const float*)maxnorm, dp, T, eps32, formula,
                               unsafe_flag, flags);
    if (e != cudaSuccess) return e;
    return launch_pdl(cull_write_kernel, dim3(g), dim3(CULL_T), 0, s, (const float*)lo,
                      (const float*)hi, (const float*)maxnorm, dp, T, eps32, formula, unsafe_flag,
                      (const int32_t*)flags, list, total_kept, count);
  }
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

cudaError_t launch_units_kernel(const UnitArgs& a, int d, int formula, int sm_count,
                                cudaStream_t s) {
  switch (pad_dim(d)) {
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

cudaError_t launch_unit_list(const float* blk, int64_t n, int d, float eps32, int formula,
                             const uint32_t* unsafe_flag, const uint32_t* item_list,
                             const unsigned long long* kept, int64_t all_items, int rank, int world,
                             uint2* unit_list, unsigned long long units_cap,
                             unsigned long long* unit_count, uint2* item_units, uint2* diag_range,
                             cudaStream_t s) {
  const int dp = pad_dim(d);
  const int KP = unit_kp(d);
  const float* box = dp <= 4 ? blk : nullptr;  // block boxes only pay off in low dimension
  // one resident wave (the kernel strides over the kept items): empty CTAs beyond it
  // would only add launch waves
  int dev = 0;
  cudaGetDevice(&dev);
  static std::atomic<int> wave_dev[DS_MAX_DEVICES] = {};
  int wave = dev < DS_MAX_DEVICES ? wave_dev[dev].load() : 0;
  if (wave == 0) {
    int sms = 148, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, unit_list_kernel, 256, 0) != cudaSuccess ||
        per_sm < 1)
      per_sm = 2;
    wave = sms * per_sm;
    if (dev < DS_MAX_DEVICES) wave_dev[dev].store(wave);
  }
  int64_t blocks = (all_items / world * 32 + 255) / 256 + 1;
  if (blocks > wave) blocks = wave;
  return launch_pdl(unit_list_kernel, dim3((unsigned)blocks), dim3(256), 0, s, box, dp, n, KP, eps32,
                    formula, unsafe_flag, item_list, kept, rank, world, unit_list, units_cap,
                    unit_count, item_units, diag_range);
}

cudaError_t launch_unit_dir(const UnitArgs& a, int d, int64_t all_items, const uint2* item_units,
                            const unsigned long long* kept, uint4* dir,
                            unsigned long long* dir_count, cudaStream_t s) {
  int64_t blocks = (all_items * 32 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  switch (unit_kp(d)) {
    case 4:
      return launch_pdl(unit_dir_kernel<4>, dim3((unsigned)blocks), dim3(256), 0, s, a, all_items,
                        item_units, kept, dir, dir_count);
    case 2:
      return launch_pdl(unit_dir_kernel<2>, dim3((unsigned)blocks), dim3(256), 0, s, a, all_items,
                        item_units, kept, dir, dir_count);
    default:
      return launch_pdl(unit_dir_kernel<1>, dim3((unsigned)blocks), dim3(256), 0, s, a, all_items,
                        item_units, kept, dir, dir_count);
  }
  return cudaGetLastError();
}

}  // namespace ds
