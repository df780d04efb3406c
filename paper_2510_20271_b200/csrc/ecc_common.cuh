// ecc_common.cuh -- shared device code for the B200 ECC engine.
//
// Semantics follow the reference ecckit 0.1.0 (see DESIGN.md for the full
// derivation); file:line citations are into /root/reference/pkg/src/ecckit.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ecc {


// ---------------------------------------------------------------------------
// cp.async (LDGSTS): global -> shared copies that bypass the registers;
// src_bytes < the copy size zero-fills the rest (0: nothing is read).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
// Lower-star Euler coefficient of one voxel from its 3x3x3 neighbourhood.
//
// v[dz][dy][dx], index 0/1/2 == offset -1/0/+1 along (axis0, axis1, axis2).
// Out-of-grid neighbours hold NaN: every comparison against NaN is false, so
// an out-of-grid neighbour never "precedes" p (coefficients.py:88-89 pads
// with +inf and forces positive offsets False at :101-104).
//
// "q precedes p" (coefficients.py:3-8, 77-82): X(q) <= X(p) for offsets whose
// first non-zero component is -1, X(q) < X(p) for +1.
//
// c(p) = 1 - #lower edges + #lower squares - #lower cubes (coefficients.py:
// 109-138).  We evaluate it through the identity
//     c3(p) = c2(P) - L- * c2(P & Q-) - L+ * c2(P & Q+)
// where P is the 8-bit in-plane lower mask, Q+- the 8-bit masks of the
// planes above/below (centre excluded), L+- the centre bits above/below,
// and c2(M) = 1 - #axis bits + #quadrant triples is the 2D coefficient of
// an 8-neighbour mask.  (Every xz/yz square and every cube in half-space s
// contains the edge p -> p + s e_z; factoring that edge out leaves exactly
// -c2 of the AND-ed masks.)  The masks are stored in a cyclic neighbour
// order E,NE,N,NW,W,SW,S,SE with E repeated as bit 8, three 9-bit lanes per
// 32-bit word, so the 12 square/cube triples are one shift-and-AND and the
// whole signed count is a single POPC.  Exhaustively checked against the
// oracle in tests (test_oracle_golden / GPU parity).
// ---------------------------------------------------------------------------
template <typename V>
__device__ __forceinline__ int coeff3(const V (&v)[3][3][3]) {
  const V p = v[1][1][1];
  // cyclic order over (dy, dx): 0:(0,+1) 1:(+1,+1) 2:(+1,0) 3:(+1,-1)
  //                             4:(0,-1) 5:(-1,-1) 6:(-1,0) 7:(-1,+1)
  // in-plane: offsets with dy<0 or (dy==0 && dx<0) are lexicographically
  // negative (<=), the others positive (<).
  uint32_t P = (uint32_t)(v[1][1][2] < p) | ((uint32_t)(v[1][2][2] < p) << 1) |
               ((uint32_t)(v[1][2][1] < p) << 2) | ((uint32_t)(v[1][2][0] < p) << 3) |
               ((uint32_t)(v[1][1][0] <= p) << 4) | ((uint32_t)(v[1][0][0] <= p) << 5) |
               ((uint32_t)(v[1][0][1] <= p) << 6) | ((uint32_t)(v[1][0][2] <= p) << 7);
  // plane below (dz = -1): all offsets negative
  uint32_t Qm = (uint32_t)(v[0][1][2] <= p) | ((uint32_t)(v[0][2][2] <= p) << 1) |
                ((uint32_t)(v[0][2][1] <= p) << 2) | ((uint32_t)(v[0][2][0] <= p) << 3) |
                ((uint32_t)(v[0][1][0] <= p) << 4) | ((uint32_t)(v[0][0][0] <= p) << 5) |
                ((uint32_t)(v[0][0][1] <= p) << 6) | ((uint32_t)(v[0][0][2] <= p) << 7);
  // plane above (dz = +1): all offsets positive
  uint32_t Qp = (uint32_t)(v[2][1][2] < p) | ((uint32_t)(v[2][2][2] < p) << 1) |
                ((uint32_t)(v[2][2][1] < p) << 2) | ((uint32_t)(v[2][2][0] < p) << 3) |
                ((uint32_t)(v[2][1][0] < p) << 4) | ((uint32_t)(v[2][0][0] < p) << 5) |
                ((uint32_t)(v[2][0][1] < p) << 6) | ((uint32_t)(v[2][0][2] < p) << 7);
  const uint32_t Lm = (uint32_t)(v[0][1][1] <= p);
  const uint32_t Lp = (uint32_t)(v[2][1][1] < p);
  const uint32_t P9 = P | ((P & 1u) << 8);
  const uint32_t Qm9 = Qm | ((Qm & 1u) << 8);
  const uint32_t Qp9 = Qp | ((Qp & 1u) << 8);
  const uint32_t W = P9 | ((P9 & Qm9 & (0u - Lm)) << 9) | ((P9 & Qp9 & (0u - Lp)) << 18);
  const uint32_t sq = W & (W >> 1) & (W >> 2);
  constexpr uint32_t EV0 = 0x55u, EV12 = (0x55u << 9) | (0x55u << 18), EVA = EV0 | EV12;
  const uint32_t pos = (W & EV12) | (sq & EV0);
  const uint32_t neg = (W & EV0) | (sq & EV12);
  return __popc(pos | ((~neg & EVA) << 1) | ((Lm ^ 1u) << 28) | ((Lp ^ 1u) << 29)) - 13;
}

// coeff3 on float64 values with the compare results taken from sign bits:
// bit 31 of hi(RD(q - p)) is [q <= p] and of hi(RN(q - p)) is [q < p] when
// no value is -0 (callers canonicalise: v + 0.0); an out-of-grid NaN gives
// +NaN, i.e. "not lower", as the IEEE compares do.  A funnel shift moves
// each sign into its mask (one SHF per compare instead of a predicate select
// and an OR); the masks and the count are coeff3's.
__device__ __forceinline__ uint32_t hi_le(double q, double p) { return (uint32_t)__double2hiint(__dsub_rd(q, p)); }
__device__ __forceinline__ uint32_t hi_lt(double q, double p) { return (uint32_t)__double2hiint(__dsub_rn(q, p)); }
__device__ __forceinline__ uint32_t push_sign(uint32_t acc, uint32_t h) { return __funnelshift_l(h, acc, 1); }
__device__ __forceinline__ int coeff3_sgn(const double (&v)[3][3][3]) {
  const double p = v[1][1][1];
  // 9-bit cyclic masks, bit 8 = bit 0 (E repeated): push E first, then bits 7 .. 0
  const uint32_t e = hi_lt(v[1][1][2], p);
  uint32_t P9 = e >> 31;
  P9 = push_sign(P9, hi_le(v[1][0][2], p));   // 7 (-1,+1)
  P9 = push_sign(P9, hi_le(v[1][0][1], p));   // 6 (-1, 0)
  P9 = push_sign(P9, hi_le(v[1][0][0], p));   // 5 (-1,-1)
  P9 = push_sign(P9, hi_le(v[1][1][0], p));   // 4 ( 0,-1)
  P9 = push_sign(P9, hi_lt(v[1][2][0], p));   // 3 (+1,-1)
  P9 = push_sign(P9, hi_lt(v[1][2][1], p));   // 2 (+1, 0)
  P9 = push_sign(P9, hi_lt(v[1][2][2], p));   // 1 (+1,+1)
  P9 = push_sign(P9, e);                      // 0 ( 0,+1)
  const uint32_t em = hi_le(v[0][1][2], p);
  uint32_t Qm9 = em >> 31;
  Qm9 = push_sign(Qm9, hi_le(v[0][0][2], p));
  Qm9 = push_sign(Qm9, hi_le(v[0][0][1], p));
  Qm9 = push_sign(Qm9, hi_le(v[0][0][0], p));
  Qm9 = push_sign(Qm9, hi_le(v[0][1][0], p));
  Qm9 = push_sign(Qm9, hi_le(v[0][2][0], p));
  Qm9 = push_sign(Qm9, hi_le(v[0][2][1], p));
  Qm9 = push_sign(Qm9, hi_le(v[0][2][2], p));
  Qm9 = push_sign(Qm9, em);
  const uint32_t ep = hi_lt(v[2][1][2], p);
  uint32_t Qp9 = ep >> 31;
  Qp9 = push_sign(Qp9, hi_lt(v[2][0][2], p));
  Qp9 = push_sign(Qp9, hi_lt(v[2][0][1], p));
  Qp9 = push_sign(Qp9, hi_lt(v[2][0][0], p));
  Qp9 = push_sign(Qp9, hi_lt(v[2][1][0], p));
  Qp9 = push_sign(Qp9, hi_lt(v[2][2][0], p));
  Qp9 = push_sign(Qp9, hi_lt(v[2][2][1], p));
  Qp9 = push_sign(Qp9, hi_lt(v[2][2][2], p));
  Qp9 = push_sign(Qp9, ep);
  const uint32_t hm = hi_le(v[0][1][1], p), hp = hi_lt(v[2][1][1], p);
  const uint32_t mLm = (uint32_t)((int32_t)hm >> 31), mLp = (uint32_t)((int32_t)hp >> 31);
  const uint32_t W = P9 | ((P9 & Qm9 & mLm) << 9) | ((P9 & Qp9 & mLp) << 18);
  const uint32_t sq = W & (W >> 1) & (W >> 2);
  constexpr uint32_t EV0 = 0x55u, EV12 = (0x55u << 9) | (0x55u << 18), EVA = EV0 | EV12;
  const uint32_t pos = (W & EV12) | (sq & EV0);
  const uint32_t neg = (W & EV0) | (sq & EV12);
  return __popc(pos | ((~neg & EVA) << 1) | ((~mLm & 1u) << 28) | ((~mLp & 1u) << 29)) - 13;
}

// 2D coefficient (coefficients.py:109-126 on a 3x3 window v[dy][dx]):
// c2(P) = 1 - #lower axis neighbours + #lower quadrant triples.
template <typename V>
__device__ __forceinline__ int coeff2(const V (&v)[3][3]) {
  const V p = v[1][1];
  const uint32_t P = (uint32_t)(v[1][2] < p) | ((uint32_t)(v[2][2] < p) << 1) | ((uint32_t)(v[2][1] < p) << 2) |
                     ((uint32_t)(v[2][0] < p) << 3) | ((uint32_t)(v[1][0] <= p) << 4) |
                     ((uint32_t)(v[0][0] <= p) << 5) | ((uint32_t)(v[0][1] <= p) << 6) |
                     ((uint32_t)(v[0][2] <= p) << 7);
  const uint32_t P9 = P | ((P & 1u) << 8);
  const uint32_t sq = P9 & (P9 >> 1) & (P9 >> 2);
  return __popc((sq & 0x55u) | ((~P & 0x55u) << 1)) - 3;
}

// ---------------------------------------------------------------------------
// Binning: smallest j with x <= tau_j (grid.py:168-180, searchsorted-left).
// The table holds the thresholds in the compare type with sentinels:
// tab[0] = -inf, tab[1..nb] = taus, tab[nb+1] = +inf.  For float32/uint8
// inputs the device thresholds are t32_j = the largest float32 <= tau_j
// (float64), which makes fp32 compares reproduce the float64 ones exactly
// (x is float32: x <= tau <=> x <= RD_f32(tau)).  The affine guess is only a
// starting point; the two correction loops make the result exact for any
// non-decreasing table, and the host picks binary search when the guess is
// poor (non-uniform thresholds).
// ---------------------------------------------------------------------------
struct BinParams {
  double t0;      // first threshold (compare type precision)
  double inv_w;   // (nb-1)/(t_last - t0), 0 when nb == 1
  int64_t nb;     // number of thresholds
  int mode;       // 0 = affine guess + correction, 1 = binary search
  int pad;
};

template <typename V>
__device__ __forceinline__ int bin_of(V x, const V* __restrict__ tab, int nb, V t0, V inv_w, int mode) {
  int j;
  if (mode == 0) {
    V g = (x - t0) * inv_w;
    g = g < V(0) ? V(0) : g;
    g = g > V(nb) ? V(nb) : g;
    j = (int)g;
    if (!(j >= 0 && j <= nb)) j = 0;   // NaN (non-finite grids are rejected, but must not fault)
    // tab is offset by one: tab[j+1] == tau_j
    while (x > tab[j + 1]) ++j;            // stops at tab[nb+1] = +inf
    while (j > 0 && x <= tab[j]) --j;      // stops at tab[0] = -inf (x = -inf: bin 0)
  } else {
    int lo = 0, hi = nb;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (tab[mid + 1] < x) lo = mid + 1; else hi = mid;
    }
    j = lo;
  }
  return j;
}

// float -> totally ordered uint32 key (finite values; -0 canonicalised)
__device__ __forceinline__ uint32_t f32_key(float f) {
  uint32_t b = __float_as_uint(f + 0.0f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key_f32(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
__device__ __forceinline__ unsigned long long f64_key(double f) {
  unsigned long long b = (unsigned long long)__double_as_longlong(f + 0.0);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_f64(unsigned long long k) {
  return __longlong_as_double((long long)((k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k));
}

// pixel_coordinates (soft.py:79-94): idx * (2/(d-1)) - 1 (two roundings), 0 if d == 1
__device__ __forceinline__ double coord64(int64_t idx, int64_t d) {
  if (d == 1) return 0.0;
  double s = __ddiv_rn(2.0, (double)(d - 1));
  return __dadd_rn(__dmul_rn((double)idx, s), -1.0);
}

}  // namespace ecc
