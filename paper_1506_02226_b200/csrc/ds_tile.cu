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

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
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
  static constexpr int KP = D <= 8 ? 4 : (D <= 32 ? 2 : 1);  // lane points per lane
  static constexpr int S = ((D + 1) + 3) / 4 * 4;           // floats per record
  static constexpr int WARPS = 4;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int STAGE = 32 * S;                       // floats per staged block
  static constexpr size_t SMEM = (size_t)WARPS * 2 * STAGE * 4;
  static constexpr int UNROLL = D <= 4 ? 32 : 8;
  static constexpr int MINB = D <= 32 ? 4 : 3;  // 16 (d <= 32) or 12 resident warps per SM
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

// Unit -> (tile pair, lane block, column block); `self` = the column block lies
// inside the lane block of a diagonal tile. Units that need no evaluation (ragged
// tail, or below the diagonal of a diagonal tile: their pairs are covered by the
// mirrored unit) report skip.
struct UnitInfo {
  int a, b, lb, jw;
  bool self, skip;
};

// Walks a warp's slice of the units. Culled schedule: one 8-byte list entry
// {a << 16 | b, sub} per unit. Dense schedule: units are q * UPT + sub over the
// upper triangle in row order, so only the slice start is decoded (decode_item);
// later units step (sub, b, a) incrementally.
template <int KP>
struct UnitCursor {
  static constexpr int UPT = (TILE / (32 * KP)) * WPR;
  const uint2* list;
  int T, n;
  int a, b, sub;

  __device__ __forceinline__ void start(const UnitArgs& A, long long u) {
    list = A.unit_list;
    T = A.T;
    n = (int)A.n;
    if (!list) {
      const long long q = u / UPT;
      sub = (int)(u - q * UPT);
      decode_item(q, T, a, b);
    }
  }
  // info of unit u (the previous call, if any, was for u - 1)
  __device__ __forceinline__ UnitInfo get(long long u, bool first) {
    if (list) {
      const uint2 e = __ldg(list + u);
      a = (int)(e.x >> 16);
      b = (int)(e.x & 0xffffu);
      sub = (int)e.y;
    } else if (!first) {
      if (++sub == UPT) {
        sub = 0;
        if (++b == T) b = ++a;
      }
    }
    UnitInfo ui;
    ui.a = a;
    ui.b = b;
    ui.lb = sub / WPR;
    ui.jw = sub % WPR;
    const int na = min(TILE, n - a * TILE);
    const int nb = min(TILE, n - b * TILE);
    ui.skip = ui.jw * 32 >= nb || ui.lb * 32 * KP >= na || (a == b && ui.jw < ui.lb * KP);
    ui.self = a == b && ui.jw < (ui.lb + 1) * KP;
    return ui;
  }
};

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

// The eps-tile kernel. Every warp owns a contiguous slice of the unit list and works
// through it without any block-level synchronisation:
//   * the unit's 32 staged points (one contiguous 32*S*4-byte run of the record
//     array) are copied into the warp's double buffer with cp.async (one 16-byte
//     copy per lane and record quarter), issued one unit ahead;
//   * the lane block (32*KP consecutive points of tile a) is held in registers and
//     only reloaded when the slice moves to another lane block;
//   * per staged point every lane evaluates its KP points in the reference's exact
//     operation order (eval_d2) and packs the predicates (pack_bits);
//   * lane-side counts are popcounts accumulated in registers across the units of a
//     lane block; column-side counts (off-diagonal units only: each unordered pair
//     is evaluated once) come from column_counts, one atomic per column;
//   * the unit's non-zero words are appended with one warp-aggregated atomic and
//     the unit's chunk entry records where they went. Units without a single bit
//     (most of a dense schedule) skip both.
template <int D, int F, bool SAFE>
__global__ void __launch_bounds__(Geo<D>::THREADS, Geo<D>::MINB) eps_unit_kernel(const UnitArgs A) {
  using G = Geo<D>;
  constexpr int KP = G::KP;
  constexpr int S = G::S;
  constexpr int KC = Pack<KP, SAFE>::KC;

  if ((*A.unsafe_flag != 0) == SAFE) return;  // the other instantiation owns this input

  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  float* stage = reinterpret_cast<float*>(smem) + (size_t)warp * 2 * G::STAGE;

  const int n = (int)A.n;
  const float eps32 = A.eps32;
  long long U = A.dense_units;
  if (A.unit_list) {
    const unsigned long long c = *A.unit_count;
    U = (long long)(c < A.units_cap ? c : A.units_cap);
  }
  const long long r_lo = U * A.shard_rank / A.shard_world;
  const long long r_hi = U * (A.shard_rank + 1) / A.shard_world;
  const long long nw = (long long)gridDim.x * G::WARPS;
  const long long gw = (long long)blockIdx.x * G::WARPS + warp;
  const long long u_lo = r_lo + (r_hi - r_lo) * gw / nw;
  const long long u_hi = r_lo + (r_hi - r_lo) * (gw + 1) / nw;
  if (u_lo >= u_hi) return;

  UnitCursor<KP> cursor;
  cursor.start(A, u_lo);
  // next unit to evaluate after u (skipped units get an empty chunk)
  auto next_unit = [&](long long u, UnitInfo& ui, bool first) -> long long {
    for (; u < u_hi; ++u, first = false) {
      ui = cursor.get(u, first);
      if (!ui.skip) return u;
      if (lane == 0) A.uchunks[u] = make_uint2(0u, 0u);
    }
    return u;
  };
  auto issue = [&](const UnitInfo& ui, int buf) {  // all lanes: record `lane` of the block
    const int j = ui.b * TILE + ui.jw * 32 + lane;
    const bool v = j < n;
    const float* src = A.rec + (size_t)(v ? j : 0) * S;
    float* dst = stage + (size_t)buf * G::STAGE + lane * S;
#pragma unroll
    for (int q = 0; q < S / 4; ++q) cp_async16(dst + 4 * q, src + 4 * q, v ? 16u : 0u);
    cp_async_commit();
  };

  UnitInfo cur;
  long long u = next_unit(u_lo, cur, true);
  if (u < u_hi) issue(cur, 0);
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
  unsigned long long units_done = 0;

  auto flush = [&]() {
    if (la < 0) return;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (lcnt[k]) atomicAdd(&A.cnt[la * TILE + (llb * 32 + lane) * KP + k], (int)lcnt[k]);
      lcnt[k] = 0u;
    }
  };

  while (u < u_hi) {
    const int buf = it & 1;
    __syncwarp();  // every lane is done reading the other buffer
    UnitInfo nxt;
    const long long un = next_unit(u + 1, nxt, false);
    if (un < u_hi) issue(nxt, buf ^ 1);

    if (cur.a != la || cur.lb != llb) {  // (re)load the lane block into registers
      flush();
      la = cur.a;
      llb = cur.lb;
      const int na = min(TILE, n - la * TILE);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int il = (llb * 32 + lane) * KP + k;  // 32*KP consecutive points per block
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
#pragma unroll
        for (int q = 0; q < Lanes<D, KP>::DP; ++q) L.v2[k][q] = make_float2(c[2 * q], c[2 * q + 1]);
        L.v1[k] = c[D - 1];
        L.t[k] = tmp[D];
      }
    }

    if (un < u_hi) cp_async_wait<1>();  // this unit's group is complete
    else cp_async_wait<0>();
    __syncwarp();
    const float* st = stage + (size_t)buf * G::STAGE;
    uint32_t acc[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) acc[k] = 0u;
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
      eval_d2<D, F, KP>(L, xj, xj[D], d2);
      pack_bits<KP, SAFE>(d2, eps32, jj, acc);
    }
    ++units_done;

    const int nb = min(TILE, n - cur.b * TILE);
    const uint32_t vm = valid_mask(nb - cur.jw * 32);
    uint32_t w[KP];
    uint32_t any = 0u;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      w[k] = lvalid[k] ? ((k < KC ? acc[k] : ~acc[k]) & vm) : 0u;
      lcnt[k] += __popc(w[k]);
      any |= w[k];
    }
    unsigned long long base = 0;
    int total = 0;
    if (__any_sync(0xffffffffu, any != 0u)) {
      if (!cur.self) {
        const uint32_t v = column_counts<KP>(w, lane);
        if (v) atomicAdd(&A.cnt[cur.b * TILE + cur.jw * 32 + lane], (int)v);
      } else {
#pragma unroll
        for (int k = 0; k < KP; ++k)  // keep columns j >= row (incl. the self pair)
          w[k] &= diag_keep((llb * 32 + lane) * KP + k - cur.jw * 32);
      }
      // append the unit's non-zero words (one warp-aggregated atomic)
      int nz = 0;
#pragma unroll
      for (int k = 0; k < KP; ++k) nz += w[k] != 0u;
      int incl = nz;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      total = __shfl_sync(0xffffffffu, incl, 31);
      if (lane == 0) base = atomicAdd(A.words_count, (unsigned long long)total);
      base = __shfl_sync(0xffffffffu, base, 0);
      unsigned long long pos = base + (unsigned long long)(incl - nz);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        if (w[k]) {
          if (pos < A.words_cap)
            A.words[pos] = make_uint2(w[k], (uint32_t)(((llb * 32 + lane) * KP + k) << 4 | cur.jw));
          ++pos;
        }
      }
    }
    if (lane == 0)
      A.uchunks[u] = make_uint2((uint32_t)base, (uint32_t)total | ((uint32_t)(base >> 32) << 16));

    u = un;
    cur = nxt;
    ++it;
  }
  flush();
  if (lane == 0 && units_done)
    atomicAdd(A.pairs_done, units_done * 32ull * 32ull * (unsigned long long)KP);
}

// ---- culled schedule: unit list ------------------------------------------------------
// Unit (lb, jw) of kept tile pair (a, b) is kept unless it is structurally empty
// (UnitCursor's skip) or, for d <= 4, the union box of its lane block and the box
// of its column block are provably out of range: the bound of keep_item, in double,
// on the 32-point block boxes (block_bounds_kernel).
__device__ __forceinline__ bool unit_keep(const float* __restrict__ blk, int dpad, int64_t n, int KP,
                                          int a, int b, int lb, int jw, float eps32, int formula,
                                          bool unsafe) {
  const int64_t na = min((int64_t)TILE, n - (int64_t)a * TILE);
  const int64_t nb = min((int64_t)TILE, n - (int64_t)b * TILE);
  if (jw * 32 >= nb || lb * 32 * KP >= na) return false;
  if (a == b && jw < lb * KP) return false;
  if (unsafe || !blk || (a == b && jw < (lb + 1) * KP)) return true;
  const int BS = 2 * dpad + 1;
  const int64_t nblk = (n + 31) / 32;
  const float* cb = blk + ((int64_t)b * WPR + jw) * BS;
  const int64_t l0 = (int64_t)a * WPR + (int64_t)lb * KP;
  const int kl = (int)min((int64_t)KP, nblk - l0);
  const double u = 1.0 / 16777216.0;
  double L = 0.0, wn = (double)cb[2 * dpad];
  for (int k = 0; k < kl; ++k) wn = fmax(wn, (double)blk[(l0 + k) * BS + 2 * dpad]);
  for (int q = 0; q < dpad; ++q) {
    float lo = INFINITY, hi = -INFINITY;
    for (int k = 0; k < kl; ++k) {
      lo = fminf(lo, blk[(l0 + k) * BS + q]);
      hi = fmaxf(hi, blk[(l0 + k) * BS + dpad + q]);
    }
    const double g = fmax(0.0, fmax((double)cb[q] - (double)hi, (double)lo - (double)cb[dpad + q]));
    L += g * g;
  }
  double bound = L * (1.0 - 4.0 * 3.0 * dpad * u) * (1.0 - 1e-12);
  if (formula == DS_FORMULA_ALGEBRAIC) bound -= 4.0 * (2.0 * dpad + 3.0) * u * wn * 2.0 * 1.001;
  return !(bound > (double)eps32);  // NaN bounds keep the unit
}

// pass 1: units per kept item (warp per item); items past the kept count get 0
__global__ void unit_count_kernel(const float* __restrict__ blk, int dpad, int64_t n, int KP,
                                  float eps32, int formula, const uint32_t* __restrict__ unsafe_flag,
                                  const uint32_t* __restrict__ items,
                                  const unsigned long long* __restrict__ kept, int64_t all_items,
                                  int32_t* __restrict__ ucnt) {
  const int64_t K = (int64_t)*kept;
  const bool unsafe = *unsafe_flag != 0;
  const int upt = (TILE / (32 * KP)) * WPR;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = K + tid; q < all_items; q += nth) ucnt[q] = 0;
  const int lane = threadIdx.x & 31;
  for (int64_t q = tid >> 5; q < K; q += nth >> 5) {
    const uint32_t ab = items[q];
    const int a = (int)(ab >> 16), b = (int)(ab & 0xffffu);
    int c = 0;
    for (int s0 = 0; s0 < upt; s0 += 32) {
      const int sub = s0 + lane;
      const bool keep = unit_keep(blk, dpad, n, KP, a, b, sub / WPR, sub % WPR, eps32, formula, unsafe);
      c += __popc(__ballot_sync(0xffffffffu, keep));
    }
    if (lane == 0) ucnt[q] = c;
  }
}

// pass 3: scatter {item, sub} at the scanned offsets (deterministic, item order)
__global__ void unit_scatter_kernel(const float* __restrict__ blk, int dpad, int64_t n, int KP,
                                    float eps32, int formula,
                                    const uint32_t* __restrict__ unsafe_flag,
                                    const uint32_t* __restrict__ items,
                                    const unsigned long long* __restrict__ kept,
                                    const int32_t* __restrict__ off, const int32_t* __restrict__ total,
                                    uint2* __restrict__ list, unsigned long long cap,
                                    unsigned long long* __restrict__ count) {
  const int64_t K = (int64_t)*kept;
  const bool unsafe = *unsafe_flag != 0;
  const int upt = (TILE / (32 * KP)) * WPR;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0) *count = (unsigned long long)*total;
  const int lane = threadIdx.x & 31;
  for (int64_t q = tid >> 5; q < K; q += nth >> 5) {
    const uint32_t ab = items[q];
    const int a = (int)(ab >> 16), b = (int)(ab & 0xffffu);
    unsigned long long pos = (unsigned long long)off[q];
    for (int s0 = 0; s0 < upt; s0 += 32) {
      const int sub = s0 + lane;
      const bool keep = unit_keep(blk, dpad, n, KP, a, b, sub / WPR, sub % WPR, eps32, formula, unsafe);
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      const unsigned long long p = pos + __popc(bal & ((1u << lane) - 1u));
      if (keep && p < cap) list[p] = make_uint2(ab, (uint32_t)sub);
      pos += __popc(bal);
    }
  }
}

// ---- directory of tile pairs with words (for the union kernels) ------------------
template <int KP>
__global__ void unit_dir_kernel(const UnitArgs A, int64_t all_items, const int32_t* __restrict__ item_off,
                                const unsigned long long* __restrict__ kept, uint4* __restrict__ dir,
                                unsigned long long* __restrict__ dir_count) {
  constexpr int UPT = (TILE / (32 * KP)) * WPR;
  long long U = A.dense_units;
  int64_t K = all_items;
  if (A.unit_list) {
    const unsigned long long c = *A.unit_count;
    U = (long long)(c < A.units_cap ? c : A.units_cap);
    K = (int64_t)*kept;
  }
  const long long r_lo = U * A.shard_rank / A.shard_world;
  const long long r_hi = U * (A.shard_rank + 1) / A.shard_world;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < K; q += nwarps) {
    long long lo, hi;
    if (A.unit_list) {
      lo = item_off[q];
      hi = q + 1 < all_items ? (long long)item_off[q + 1] : (long long)*A.unit_count;
      if (q + 1 == K) hi = (long long)*A.unit_count;
    } else {
      lo = q * UPT;
      hi = lo + UPT;
    }
    lo = lo > r_lo ? lo : r_lo;
    hi = hi < r_hi ? hi : r_hi;
    if (lo >= hi) continue;
    uint32_t words = 0;
    for (long long u = lo + lane; u < hi; u += 32) words += A.uchunks[u].y & 0xffffu;
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
      const unsigned long long ci = atomicAdd(dir_count, 1ull);
      dir[ci] = make_uint4(((uint32_t)a << 16) | (uint32_t)b, (uint32_t)lo, (uint32_t)(hi - lo),
                           (uint32_t)((unsigned long long)lo >> 32));
    }
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
cudaError_t launch_one(const UnitArgs& a, int sm_count, cudaStream_t s) {
  using G = Geo<D>;
  auto kern = eps_unit_kernel<D, F, SAFE>;
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
  kern<<<(unsigned)(sm_count * per_sm), G::THREADS, G::SMEM, s>>>(a);
  return cudaGetLastError();
}

// Both instantiations are launched back to back; each reads the device flag set by
// the prep kernel and the one that does not own the input exits immediately, so
// the host never waits for the range check.
template <int D, int F>
cudaError_t launch_df(const UnitArgs& a, int sm_count, cudaStream_t s) {
  cudaError_t e = launch_one<D, F, true>(a, sm_count, s);
  if (e != cudaSuccess) return e;
  return launch_one<D, F, false>(a, sm_count, s);
}

template <int D>
cudaError_t launch_d(const UnitArgs& a, int formula, int sm_count, cudaStream_t s) {
  return formula == DS_FORMULA_ALGEBRAIC ? launch_df<D, DS_FORMULA_ALGEBRAIC>(a, sm_count, s)
                                         : launch_df<D, DS_FORMULA_DIRECT>(a, sm_count, s);
}

}  // namespace

int padded_dim(int d) { return pad_dim(d); }

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
                             const unsigned long long* kept, int64_t all_items, int32_t* ucnt,
                             int32_t* partials, int32_t* total32, uint2* unit_list,
                             unsigned long long units_cap, unsigned long long* unit_count,
                             cudaStream_t s) {
  const int dp = pad_dim(d);
  const int KP = unit_kp(d);
  const float* box = dp <= 4 ? blk : nullptr;  // block boxes only pay off in low dimension
  int64_t blocks = (all_items * 32 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  unit_count_kernel<<<(unsigned)blocks, 256, 0, s>>>(box, dp, n, KP, eps32, formula, unsafe_flag,
                                                     item_list, kept, all_items, ucnt);
  cudaError_t e = launch_exclusive_scan(ucnt, all_items, partials, total32, s);
  if (e != cudaSuccess) return e;
  unit_scatter_kernel<<<(unsigned)blocks, 256, 0, s>>>(box, dp, n, KP, eps32, formula, unsafe_flag,
                                                       item_list, kept, ucnt, total32, unit_list,
                                                       units_cap, unit_count);
  return cudaGetLastError();
}

cudaError_t launch_unit_dir(const UnitArgs& a, int d, int64_t all_items, const int32_t* item_off,
                            const unsigned long long* kept, uint4* dir,
                            unsigned long long* dir_count, cudaStream_t s) {
  int64_t blocks = (all_items * 32 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  switch (unit_kp(d)) {
    case 4:
      unit_dir_kernel<4><<<(unsigned)blocks, 256, 0, s>>>(a, all_items, item_off, kept, dir, dir_count);
      break;
    case 2:
      unit_dir_kernel<2><<<(unsigned)blocks, 256, 0, s>>>(a, all_items, item_off, kept, dir, dir_count);
      break;
    default:
      unit_dir_kernel<1><<<(unsigned)blocks, 256, 0, s>>>(a, all_items, item_off, kept, dir, dir_count);
  }
  return cudaGetLastError();
}

}  // namespace ds
