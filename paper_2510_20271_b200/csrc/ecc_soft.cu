// ecc_soft.cu -- soft (sigmoid-relaxed) ECC forward / backward for sm_100a.
//
//   K5 ecc_soft_kernel<BWD=false>  chi_j  = sum_p c_p s_jp            (soft.py:154-196)
//   K6 ecc_soft_kernel<BWD=true>   w_p    = sum_j up_j lam s(1-s)    (soft.py:199-257)
//                                  dX_p   = -c_p w_p
//                                  dtau_j = up_j sum_p c_p lam s(1-s)
//                                  G      = sum_p c_p w_p pos_p      (d_u = -alpha G, d_alpha = -G.u)
//   K7 ecc_soft_reduce             fixed-order float64 sum of per-CTA partials
//
// The work is (voxel, threshold) pairs and is SFU-bound: each pair needs one
// sigmoid.  With the centred factorisation
//     exp(-lam (tau_j - f_p)) = a_j * b_p,  a_j = e^{-lam (tau_j - m)},  b_p = e^{lam (f_p - m)}
// a sigmoid is one FFMA + one MUFU.RCP (forward) instead of ex2 + rcp.
// Voxels with c_p == 0 contribute nothing to any output except dX_p = 0,
// so each CTA compacts its chunk to the non-zero voxels first.
//
// Layout: a CTA owns a chunk of CH voxels of one batch item; a lane holds
// TT = 32 thresholds in registers (a_j and accumulators); Lv lanes (power of
// two) cover one voxel's thresholds, 32/Lv voxels per warp in flight.
// Partials are reduced in a fixed order (deterministic, bit-reproducible
// across runs), fp32 within a lane over its voxels, fp64 across lanes/CTAs.
#include <math.h>
#include <stdlib.h>

#include "ecc_common.cuh"
#include "ecc_internal.h"
#include <algorithm>
#include <type_traits>
#include <mutex>
#include <map>
#include <tuple>

namespace ecc {

constexpr int SNT = 256;   // threads per CTA
constexpr int SNW = SNT / 32;
constexpr int TT = 32;     // thresholds per lane
constexpr int CH = 4096;   // voxels per CTA chunk
constexpr int MAXB_PASS = 32 * TT;  // thresholds per pass (Lv <= 32)
constexpr double LOG2E = 1.4426950408889634;

struct SoftArgs {
  const int8_t* c;        // [N][n]
  const float* fc;        // [N][n] centred field f - m (float32)
  const float* fclo;      // [N][n] f - m - fc (direct mode only)
  int64_t n;              // voxels per item
  int64_t chunks;         // ceil(n / CH)
  int64_t G;              // chunks per CTA (a unit)
  int64_t units;          // ceil(chunks / G): CTAs per item, partial rows per item
  int64_t D, H, W;
  int ndim;
  int nb;                 // B
  int factorized;
  float kscale;           // lam * log2(e)
  double lam, m;
  const double* taus;     // [B]
  const double* up;       // [N][B]   (backward)
  double* part;           // [N][chunks][B]
  double* gpart;          // [N][chunks][4]   (backward)
  float* dX;              // [N][n]   (backward)
  const ecc_soft_params* pd;   // parameters resident on the device (sync-free path), else nullptr
  int band;               // the windowed kernel was launched alongside: this one exits where it runs
  int2* recs;             // band kernels: the forward's band-sorted records [N][chunks][SNW][BREG], or nullptr
  int* rcnt;              //   and their counts [N][chunks][SNW]; the backward reads them instead of sorting
  int64_t unit0 = 0;      // this launch's first unit (units [unit0, unit0 + lunits) of every item)
  int64_t lunits = 0;     // units per item in this launch (== units unless a unit range is launched)
  int64_t item0 = 0;      // this launch's first item (items [item0, item0 + gridDim.x / lunits))
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA pipe for |x| <= 126 (the per-voxel factor b_p): x = n + f
// with n = rint(x) from the 1.5 * 2^23 magic add, 2^f by its degree-6 Taylor
// polynomial on [-1/2, 1/2] (relative error ~1.2e-7, like ex2.approx), and n
// added to the exponent field.  Frees the XU pipe, which the reciprocals
// saturate in the backward pass.
__device__ __forceinline__ float ex2_fma(float x) {
  const float r = __fadd_rn(x, 12582912.0f);
  const float f = __fsub_rn(x, __fsub_rn(r, 12582912.0f));
  float p = 1.5403530e-4f;
  p = __fmaf_rn(p, f, 1.3333558e-3f);
  p = __fmaf_rn(p, f, 9.6181291e-3f);
  p = __fmaf_rn(p, f, 5.5504109e-2f);
  p = __fmaf_rn(p, f, 2.4022651e-1f);
  p = __fmaf_rn(p, f, 6.9314718e-1f);
  p = __fmaf_rn(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(r) - 0x4B400000) << 23));
}
#ifndef ECC_SOFT_EX2_FMA
#define ECC_SOFT_EX2_FMA 0   // 0: MUFU.EX2 (default); 1: FMA-pipe 2^x in the backward, 2: in both (measured slower: 830 / 577 vs 808 / 527 us)
#endif
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 1/x on the FMA pipe for x in [1, 2^126] (the sigmoid denominators): bit-trick
// seed (relative error < 12.5%) and three Newton steps (< 1e-7 relative).
// Issuing a share of the reciprocals here instead of on MUFU balances the
// SFU against the FMA pipe (the pair loop is otherwise MUFU-bound).
__device__ __forceinline__ float rcp_fma(float x) {
  float r = __int_as_float(0x7EF311C3 - __float_as_int(x));
#pragma unroll
  for (int k = 0; k < 3; ++k) r = r * __fmaf_rn(-x, r, 2.f);
  return r;
}

// smem layout of a chunk after compaction
struct ChunkSmem {
  float fc[CH];     // centred field f_p - m of the non-zero voxels
  int pk[CH];       // voxel index within the chunk | (c << 16)
  int count;
  int pad[3];
};
// after ChunkSmem: factorised mode  atab[MAXB_PASS] (float)
//                  direct mode      fclo[CH] (float remainders), kt[MAXB_PASS] (double)
constexpr size_t CHUNK_BYTES = sizeof(ChunkSmem);

// log2 bound of the per-lane factor a_j; b_p is clamped to 2^+-(126 - A_MAX)
// so a_j b_p stays inside [2^-126, 2^126] (no overflow, no inf*0)
constexpr float A_MAX = 40.f;
#ifndef ECC_SOFT_PAIR
#define ECC_SOFT_PAIR 1   // paired reciprocals (pair_loop_prod) when the margin allows: bit 0 forward,
                          // bit 1 backward (measured: forward 816 vs 875 us, backward 1.43 vs 1.36 ms
                          // on 16 x 1024^2 -- the backward is latency-bound and the pairing lengthens
                          // its dependency chain, so it keeps one reciprocal per pair)
#endif
constexpr float B_MAX = 126.f - A_MAX;

template <bool BWD, int T, int EMU_EVERY>
__device__ __forceinline__ void pair_loop_fact(const float (&at)[T], const float (&upv)[T], float (&acc)[T], float b,
                                               float cf, float& w) {
  // sigma = r = 1 / (1 + a_j b_p): one FFMA + one MUFU.RCP; sigma (1 - sigma)
  // = r - r^2 (one FFMA; its absolute error ~1 ulp(1) is far below the
  // normwise tolerance).  All reciprocals are issued before any is consumed
  // so the MUFU latency overlaps; two partial sums break the w chain.
  float r[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const float den = __fmaf_rn(at[t], b, 1.f);
    r[t] = (t % EMU_EVERY == EMU_EVERY - 1) ? rcp_fma(den) : rcp_approx(den);
  }
  float w0 = 0.f, w1 = 0.f;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    if (!BWD) {
      acc[t] = __fmaf_rn(cf, r[t], acc[t]);
    } else {
      const float s1 = __fmaf_rn(-r[t], r[t], r[t]);
      if (t & 1) w1 = __fmaf_rn(upv[t], s1, w1); else w0 = __fmaf_rn(upv[t], s1, w0);
      acc[t] = __fmaf_rn(cf, s1, acc[t]);
    }
  }
  w = w0 + w1;
}

// ---- packed f32x2 variant (sm_100 FFMA2/FMUL2): one issue slot per two
// lane-FMAs.  The FMA pipe's lane throughput is unchanged, but the issue
// slots freed let a larger share of the reciprocals move from MUFU to
// Newton iterations on the FMA pipe, which is what balances the pair loop.
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float x, float y) {
  f2_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(x), "f"(y));
  return d;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// c - a*b as ONE FFMA2 with a negated operand (single rounding, = fma(-a, b, c))
__device__ __forceinline__ f2_t fnma2(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("{\n.reg .b64 na;\n"
      "xor.b64 na, %1, 0x8000000080000000;\n"
      "fma.rn.f32x2 %0, na, %2, %3;\n}\n" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
// slots (pairs of thresholds) whose reciprocals run as Newton iterations
#ifndef ECC_EMU_FWD
#define ECC_EMU_FWD 3   // emulated slots per 8 (forward)
#endif
#ifndef ECC_EMU_BWD
#define ECC_EMU_BWD 1   // emulated slots per 8 (backward): 1 measured 10.73 vs 10.83 ms on C3 (3 runs each);
                        // 2 was slower (before the sign-flip-free FMAs: 11.41 vs 11.10)
#endif
template <bool BWD>
__device__ __forceinline__ constexpr bool emu_slot(int i) {
  // spread the emulated slots evenly over each group of 8
  return ((i % 8) * (BWD ? ECC_EMU_BWD : ECC_EMU_FWD)) % 8 + (BWD ? ECC_EMU_BWD : ECC_EMU_FWD) > 7 &&
         (BWD ? ECC_EMU_BWD : ECC_EMU_FWD) > 0;
}

// The a-pairs arrive NEGATED (nat = -a_j): den = 1 + a b is formed as
// nden = fma(-a, b, -1) = -den, so no operand ever needs a sign flip (an
// f32x2 FMA has no negate modifier; a 64-bit XOR costs two LOP3 per pair of
// lanes).  Forward: r = rcp(-nden) (MUFU takes the negation for free),
// Newton steps r (2 + nden r).  Backward: rn = rcp(nden) = -sigma and
// fma(rn, rn, rn) = sigma^2 - sigma = -sigma (1 - sigma), so the backward
// accumulates negated w and d_tau partials; w is negated on return and acc
// by the caller.  Every rounding is the sign mirror of the positive form,
// so the results are bit-identical to it.
template <bool BWD, int T>
__device__ __forceinline__ void pair_loop_fact2(const f2_t (&nat)[T / 2], const f2_t (&up)[T / 2], f2_t (&acc)[T / 2],
                                                float b, float cf, float& w) {
  const f2_t b2 = f2_pack(b, b), mone2 = f2_pack(-1.f, -1.f), two2 = f2_pack(2.f, 2.f), cf2 = f2_pack(cf, cf);
  f2_t r[T / 2];   // forward: sigma; backward: -sigma
#pragma unroll
  for (int i = 0; i < T / 2; ++i) {
    const f2_t nden = fma2(nat[i], b2, mone2);
    float dx, dy;
    f2_unpack(nden, dx, dy);
    if (emu_slot<BWD>(i)) {
      // seed 0x7EF311C3 - bits(den) = 0xFEF311C3 - bits(-den) (< 12.5 % error),
      // three Newton steps r (2 - den r)
      f2_t q = f2_pack(__int_as_float((int)(0xFEF311C3u - (uint32_t)__float_as_int(dx))),
                       __int_as_float((int)(0xFEF311C3u - (uint32_t)__float_as_int(dy))));
#pragma unroll
      for (int k = 0; k < 3; ++k) q = mul2(q, fma2(nden, q, two2));
      r[i] = BWD ? mul2(q, mone2) : q;
    } else {
      r[i] = BWD ? f2_pack(rcp_approx(dx), rcp_approx(dy)) : f2_pack(rcp_approx(-dx), rcp_approx(-dy));
    }
  }
  if (!BWD) {
#pragma unroll
    for (int i = 0; i < T / 2; ++i) acc[i] = fma2(cf2, r[i], acc[i]);
  } else {
    f2_t w0 = 0ull, w1 = 0ull;
#pragma unroll
    for (int i = 0; i < T / 2; ++i) {
      const f2_t ns1 = fma2(r[i], r[i], r[i]);   // sigma^2 - sigma = -sigma (1 - sigma)
      if (i & 1) w1 = fma2(up[i], ns1, w1); else w0 = fma2(up[i], ns1, w0);
      acc[i] = fma2(cf2, ns1, acc[i]);
    }
    float a0, a1, c0, c1;
    f2_unpack(w0, a0, a1);
    f2_unpack(w1, c0, c1);
    w = -((a0 + c0) + (a1 + c1));
  }
}

// Paired reciprocals (factorised mode, the default when the thresholds allow
// it): slot i (thresholds 2i, 2i+1) is paired lane-wise with slot T/2-1-i
// (T-2-2i, T-1-2i), whose factors a_j are near the reciprocals of slot i's
// (the block is centred), and one reciprocal R = 1 / (d d') of the product of
// the two denominators serves both: sigma = d' R, sigma' = d R.  One MUFU per
// two (voxel, threshold) pairs instead of one per pair, for two FMULs.  The
// product stays finite because b_p is clamped to 2^(+-bc), bc = (126 -
// max log2(a a')) / 2 - 1 (computed per lane block in the kernel), and the
// clamp changes sigma by at most 2^(A - bc) <= 2^-24 (A = max |log2 a|); the
// kernel falls back to pair_loop_fact2 when that margin is not met.
// Negated factors as in pair_loop_fact2 (nd = -d): forward sigma = nd' *
// rcp(-P), backward -sigma = nd' * rcp(P).
#ifndef ECC_BAND_EX2_FMA
#define ECC_BAND_EX2_FMA 0   // band forward: 2^kf on the FMA pipe instead of MUFU.EX2 (measured slower: C4 module
                             // forward 3.99 vs 3.87 ms)
#endif
#ifndef ECC_PROD_UNP
#define ECC_PROD_UNP 2   // band backward: slot pairs (of T / 4) kept unpaired -- one MUFU per pair, fewer FMA-pipe
                         // ops; balances the two pipes (0 / 1 / 2 / 3 / 4: 3.50 / 3.42 / 3.39 / 3.45 / 3.55 ms, 128 x 1024^2)
#endif
template <bool BWD, int T, int UNP = 0>
__device__ __forceinline__ void pair_loop_prod(const f2_t (&nat)[T / 2], const f2_t (&up)[T / 2], f2_t (&acc)[T / 2],
                                               float b, float cf, float& w) {
  const f2_t b2 = f2_pack(b, b), mone2 = f2_pack(-1.f, -1.f), cf2 = f2_pack(cf, cf);
  f2_t r[T / 2];   // forward: sigma; backward: -sigma
#pragma unroll
  for (int i = 0; i < T / 4; ++i) {
    const int ip = T / 2 - 1 - i;
    const f2_t nd = fma2(nat[i], b2, mone2), ndp = fma2(nat[ip], b2, mone2);
    if (i < UNP) {   // unpaired: rcp(-den) = sigma, rcp(den)... (as pair_loop_fact2)
      float dx, dy, ex, ey;
      f2_unpack(nd, dx, dy);
      f2_unpack(ndp, ex, ey);
      r[i] = BWD ? f2_pack(rcp_approx(dx), rcp_approx(dy)) : f2_pack(rcp_approx(-dx), rcp_approx(-dy));
      r[ip] = BWD ? f2_pack(rcp_approx(ex), rcp_approx(ey)) : f2_pack(rcp_approx(-ex), rcp_approx(-ey));
      continue;
    }
    float px, py;
    f2_unpack(mul2(nd, ndp), px, py);   // d d' > 0
    const f2_t R = BWD ? f2_pack(rcp_approx(px), rcp_approx(py)) : f2_pack(rcp_approx(-px), rcp_approx(-py));
    r[i] = mul2(ndp, R);
    r[ip] = mul2(nd, R);
  }
  if (!BWD) {
#pragma unroll
    for (int i = 0; i < T / 2; ++i) acc[i] = fma2(cf2, r[i], acc[i]);
  } else {
    f2_t w0 = 0ull, w1 = 0ull;
#pragma unroll
    for (int i = 0; i < T / 2; ++i) {
      const f2_t ns1 = fma2(r[i], r[i], r[i]);   // -sigma (1 - sigma)
      if (i & 1) w1 = fma2(up[i], ns1, w1); else w0 = fma2(up[i], ns1, w0);
      acc[i] = fma2(cf2, ns1, acc[i]);
    }
    float a0, a1, c0, c1;
    f2_unpack(w0, a0, a1);
    f2_unpack(w1, c0, c1);
    w = -((a0 + c0) + (a1 + c1));
  }
}

// direct mode (large lambda * threshold spread): the exponent
// lam log2(e) (f_p - tau_j) is formed in float64 (f_p carried as two floats,
// kt_j = lam log2(e) (tau_j - m) from a transposed shared table), then ex2 + rcp
template <bool BWD, int T>
__device__ __forceinline__ void pair_loop_direct(const double* __restrict__ kt, int Lv, int l, const float (&upv)[T],
                                                 float (&acc)[T], double kf, float cf, float& w) {
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const double z = kf - kt[t * Lv + l];
    const float e = ex2_approx(fminf((float)z, 100.f));
    const float r = rcp_approx(e + 1.f);
    if (!BWD) {
      acc[t] = __fmaf_rn(cf, r, acc[t]);
    } else {
      const float s1 = (e * r) * r;
      w = __fmaf_rn(upv[t], s1, w);
      acc[t] = __fmaf_rn(cf, s1, acc[t]);
    }
  }
}


// G = sum_p c_p w_p pos_p = -sum_p dX_p pos_p.  soft_run_G_acc adds the
// voxels [i0, i1) of a chunk (their dX just written by this CTA or warp;
// zero-coefficient voxels hold 0), walking their coordinates;
// soft_chunk_G_acc gives each thread a contiguous run of the chunk.
// soft_unit_G_write reduces the per-thread sums of the CTA's chunks in a
// fixed order.
__device__ __forceinline__ void soft_run_G_acc(const SoftArgs& a, int64_t item, int64_t v0, int i0, int i1,
                                               double (&gacc)[3]) {
  float g0 = 0.f, g1 = 0.f, g2 = 0.f;
  if (i0 < i1) {
    const float sH = a.H > 1 ? (float)(2.0 / (double)(a.H - 1)) : 0.f;
    const float sW = a.W > 1 ? (float)(2.0 / (double)(a.W - 1)) : 0.f;
    const float sD = a.D > 1 ? (float)(2.0 / (double)(a.D - 1)) : 0.f;
    const int64_t vi = v0 + i0;
    int64_t z = vi / (a.H * a.W), r = vi - z * a.H * a.W, y = r / a.W, x = r - y * a.W;
    const float* dxp = a.dX + item * a.n + v0;
    for (int i = i0; i < i1; ++i) {
      const float d = dxp[i];
      if (d != 0.f) {
        const float pz = a.D > 1 ? __fmaf_rn((float)z, sD, -1.f) : 0.f;
        const float py = a.H > 1 ? __fmaf_rn((float)y, sH, -1.f) : 0.f;
        const float px = a.W > 1 ? __fmaf_rn((float)x, sW, -1.f) : 0.f;
        if (a.ndim == 2) {
          g0 = __fmaf_rn(-d, py, g0);
          g1 = __fmaf_rn(-d, px, g1);
        } else {
          g0 = __fmaf_rn(-d, pz, g0);
          g1 = __fmaf_rn(-d, py, g1);
          g2 = __fmaf_rn(-d, px, g2);
        }
      }
      if (++x == a.W) {
        x = 0;
        if (++y == a.H) { y = 0; ++z; }
      }
    }
  }
  gacc[0] += g0;
  gacc[1] += g1;
  gacc[2] += g2;
}
__device__ __forceinline__ void soft_chunk_G_acc(const SoftArgs& a, int64_t item, int64_t v0, int nvox,
                                                 double (&gacc)[3]) {
  const int per = (CH + SNT - 1) / SNT;
  const int i0 = threadIdx.x * per;
  soft_run_G_acc(a, item, v0, i0, min(i0 + per, nvox), gacc);
}

__device__ __forceinline__ void soft_unit_G_write(const SoftArgs& a, int64_t slotidx, const double (&gacc)[3],
                                                  double (*s_g)[4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v0d = gacc[0], v1d = gacc[1], v2d = gacc[2];
  for (int o = 16; o; o >>= 1) {
    v0d += __shfl_xor_sync(0xffffffffu, v0d, o);
    v1d += __shfl_xor_sync(0xffffffffu, v1d, o);
    v2d += __shfl_xor_sync(0xffffffffu, v2d, o);
  }
  if (lane == 0) { s_g[warp][0] = v0d; s_g[warp][1] = v1d; s_g[warp][2] = v2d; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double sg = 0.0;
    for (int w = 0; w < SNW; ++w) sg += s_g[w][threadIdx.x];
    a.gpart[slotidx * 4 + threadIdx.x] = sg;
  }
}

// ---- windowed ("band") mode ------------------------------------------------
// With a sharp sigmoid most (voxel, threshold) pairs are saturated:
// sigma(lam (tau - f)) < 2^-24 for tau < f - W and > 1 - 2^-24 for
// tau > f + W, W = 24 ln 2 / lam.  The band kernel evaluates only a window of
// NWB consecutive 16-threshold blocks per voxel, chosen so that every
// threshold below it lies below f - W and every threshold above it above
// f + W; the pairs above contribute sigma = 1 (forward: c_p per threshold,
// summed per band and added once per chunk), those below 0, and in the
// backward both contribute sigma (1 - sigma) = 0.  The error per skipped pair
// is < 2^-24 -- the float32 rounding the pair loop already has (a
// denominator 1 + a b with a b < 2^-24 rounds to 1).  Each CTA sorts its
// non-zero voxels by window start ("band") while compacting, so a lane keeps
// one block's factors and accumulators in registers for a whole band.  Valid
// when the thresholds are sorted and every NWB - 1 blocks span more than 2 W
// (band_ok, evaluated identically by this kernel and the full one, so exactly
// one of the two does the work); for C3 / C4 (B = 256, lam = 50) the window
// is 8 of 16 blocks.
constexpr int BT = 16;                          // thresholds per lane block
constexpr int NWB = 8;                          // blocks (lanes) per voxel window
constexpr int BVW = 32 / NWB;                   // voxels per warp in flight
constexpr int BSLOTS = SNW * BVW;               // voxel slots per CTA
constexpr int BAND_MAXB = 368;                  // thresholds: at most 16 bands of NWB blocks
constexpr int BAND_MAXBLK = BAND_MAXB / BT;
constexpr int BAND_MAXBANDS = 16;               // band index: 4 bits of the voxel record
constexpr double BAND_ZCUT = 16.635532333438686;   // 24 ln 2

__device__ __forceinline__ bool band_ok(const SoftArgs& a) {
  const int nb = a.nb, nblk = (nb + BT - 1) / BT, nbands = nblk - NWB + 1;
  if (nb > BAND_MAXB || nbands < 2 || nbands > BAND_MAXBANDS) return false;   // uniform over the grid
  if (a.W >= (1 << 22) || a.H >= (1 << 22) || a.D >= (1 << 22)) return false;   // fused G's 2^23 conversions
  const double w2 = 2.0 * BAND_ZCUT / a.lam * (1.0 + 1e-3);
  bool ok = true;
  for (int j = threadIdx.x; j + 1 < nb; j += blockDim.x) ok = ok && a.taus[j] <= a.taus[j + 1];
  for (int b = threadIdx.x; b + 1 < nbands; b += blockDim.x)
    ok = ok && a.taus[(b + NWB) * BT] - a.taus[(b + 1) * BT] > w2;
  return __syncthreads_and(ok) != 0;
}

static size_t band_smem(int nb);

template <bool BWD, bool FACT, int T>
__global__ void __launch_bounds__(SNT, (T == 8 ? 4 : (T == 16 ? 3 : 2)))
ecc_soft_kernel(SoftArgs a) {
  if (a.pd) {   // device-resident parameters: both modes are launched, the other one exits here
    if ((a.pd->factorized != 0) != FACT) return;
    a.lam = a.pd->lam;
    a.m = a.pd->center;
    a.kscale = (float)(a.lam * LOG2E);
  }
  if (FACT && T == BT && a.band && band_ok(a)) return;   // the band kernel does this problem
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ChunkSmem& S = *reinterpret_cast<ChunkSmem*>(smem_raw);
  unsigned char* tail = smem_raw + CHUNK_BYTES;
  float* s_fclo = reinterpret_cast<float*>(tail);                                   // direct mode
  double* kt = reinterpret_cast<double*>(tail + sizeof(float) * CH);                 // direct mode
  float* atab = reinterpret_cast<float*>(tail);                                      // factorised
  float* red = reinterpret_cast<float*>(smem_raw);   // reused after the main loop
  __shared__ int s_wcount[SNW];
  __shared__ double s_g[SNW][4];

  // this CTA: chunks [c0, c1) of one item (a unit of G chunks)
  const int64_t item = a.item0 + blockIdx.x / a.lunits;
  const int64_t unit = a.unit0 + blockIdx.x % a.lunits;
  const int64_t c0 = unit * a.G, c1 = min(c0 + a.G, a.chunks);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;


  // ---- lane groups: Lv lanes cover one voxel's thresholds -----------------
  const int nb = a.nb;
  int Lv = 1;
  while (Lv * T < nb) Lv <<= 1;
  const int VW = 32 / Lv;               // voxels per warp in flight
  const int g = lane / Lv;              // voxel slot within the warp
  const int l = lane % Lv;              // threshold block of this lane
  const int slot = warp * VW + g;
  const int nslots = SNW * VW;

  // thresholds of this lane: j = l*T + t, centred on the block's own centre
  // m_l (factorised: a_j = 2^{-k (tau_j - m_l)}, b_{p,l} = 2^{k (f_p - m_l)}).
  // The per-threshold factors are computed once per CTA into shared memory.
  const double ks = a.lam * LOG2E;
  if (FACT) {
    for (int j = threadIdx.x; j < Lv * T; j += SNT) {
      float av = 0.f;
      if (j < nb) {
        const int b0 = (j / T) * T, b1 = min(b0 + T, nb) - 1;
        av = (float)exp2(-ks * (a.taus[j] - 0.5 * (a.taus[b0] + a.taus[b1])));
      }
      atab[j] = av;
    }
  } else {
    // kt[t * Lv + l] = ks (tau_{l T + t} - m); padded thresholds -> +inf (sigma = 1, discarded)
    for (int q = threadIdx.x; q < Lv * T; q += SNT) {
      const int tt = q / Lv, ll = q % Lv, j = ll * T + tt;
      kt[q] = j < nb ? ks * (a.taus[j] - a.m) : (double)INFINITY;
    }
  }
  __syncthreads();
  // paired-reciprocal mode (factorised): this lane block's b clamp and margin
  float bc = B_MAX;
  bool prod = false;
  if (FACT && (ECC_SOFT_PAIR & (BWD ? 2 : 1))) {
    float amax = 0.f, dmax = 0.f;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int tp = (T - 2 - 2 * (t >> 1)) + (t & 1);   // lane-wise partner (slot T/2-1-i)
      const float x0 = atab[l * T + t], x1 = atab[l * T + tp];
      const float l0 = x0 > 0.f ? __log2f(x0) : 0.f, l1 = x1 > 0.f ? __log2f(x1) : 0.f;
      amax = fmaxf(amax, fabsf(l0));
      dmax = fmaxf(dmax, l0 + l1);
    }
    bc = fminf(B_MAX, 0.5f * (126.f - dmax) - 1.f);
    prod = __syncthreads_and(bc - amax >= 24.f);
    if (!prod) bc = B_MAX;
  }
  float at[T], upv[T], acc[T];          // direct mode
  f2_t at2[T / 2], up2[T / 2], acc2[T / 2];  // factorised mode (packed pairs)
  const int j0 = l * T;
  const int jl = min(j0 + T, nb) - 1;
  const double ml = (j0 < nb) ? 0.5 * (a.taus[j0] + a.taus[jl]) : a.m;
  // the factors are (re)loaded per chunk after its compaction, so they are
  // not live across it; the accumulators persist over the CTA's chunks
  auto load_lane = [&]() {
#pragma unroll
    for (int t = 0; t < T; ++t) {
      at[t] = FACT ? atab[j0 + t] : 0.f;
      upv[t] = (BWD && j0 + t < nb) ? (float)a.up[item * nb + j0 + t] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < T / 2; ++i) {
      at2[i] = f2_pack(-at[2 * i], -at[2 * i + 1]);   // negated: see pair_loop_fact2
      up2[i] = f2_pack(upv[2 * i], upv[2 * i + 1]);
    }
  };
#pragma unroll
  for (int t = 0; t < T; ++t) acc[t] = 0.f;
#pragma unroll
  for (int i = 0; i < T / 2; ++i) acc2[i] = 0ull;
  const float koff = FACT ? (float)(ks * (a.m - ml)) : 0.f;   // k f_p - k m_l = k fc + koff

  auto voxel_w = [&](int k, bool valid) -> float {
    const float f = valid ? S.fc[k] : 0.f;
    const float cf = valid ? __uint_as_float((uint32_t)S.pk[k] & 0xFFFF0000u) : 0.f;
    float w = 0.f;
    if (FACT) {
      const float kf = fminf(fmaxf(__fmaf_rn(a.kscale, f, koff), -bc), bc);
      // forward: paired reciprocals (pair_loop_prod) when the margin allows,
      // else packed FFMA2 pairs with 3/8 of the reciprocals as Newton
      // iterations; backward: packed FFMA2 with 1/8 of the reciprocals as
      // Newton iterations (ECC_EMU_BWD).  The scalar loop stays as the A/B
      // reference.
#ifndef ECC_BWD_PACKED
#define ECC_BWD_PACKED 1   // packed FFMA2 backward (801 vs 838 us at 16 thresholds per lane)
#endif
      if (BWD && !ECC_BWD_PACKED)
        pair_loop_fact<BWD, T, 1024>(at, upv, acc, ECC_SOFT_EX2_FMA >= 1 ? ex2_fma(kf) : ex2_approx(kf), cf, w);
      else if (prod)
        pair_loop_prod<BWD, T>(at2, up2, acc2, ex2_approx(kf), cf, w);
      else
        pair_loop_fact2<BWD, T>(at2, up2, acc2,
                                (BWD ? ECC_SOFT_EX2_FMA >= 1 : ECC_SOFT_EX2_FMA >= 2) ? ex2_fma(kf) : ex2_approx(kf),
                                cf, w);
    } else {
      const double fd = (double)f + (double)(valid ? s_fclo[k] : 0.f);
      pair_loop_direct<BWD, T>(kt, Lv, l, upv, acc, ks * fd, cf, w);
    }
    return w;
  };
  const float lamf = (float)a.lam;
  double gacc[3] = {0.0, 0.0, 0.0};
  for (int64_t chunk = c0; chunk < c1; ++chunk) {
  const int64_t v0 = chunk * CH;
  const int nvox = (int)min((int64_t)CH, a.n - v0);
  const int8_t* cg = a.c + item * a.n + v0;
  const float* fg = a.fc + item * a.n + v0;
  // ---- compaction of the chunk to c != 0 voxels (order-preserving) -------
  // Each warp owns CITER x 32 consecutive voxels; all of its coefficient and
  // field loads are issued up front (one memory latency, not CITER).
  {
    constexpr int CITER = CH / SNW / 32;
    const int w0 = warp * (CITER * 32), w1 = min(w0 + CITER * 32, nvox);
    int cvr[CITER];
    float fvr[CITER];
#pragma unroll
    for (int it = 0; it < CITER; ++it) {
      const int i = w0 + it * 32 + lane;
      cvr[it] = i < w1 ? (int)cg[i] : 0;
      fvr[it] = i < w1 ? fg[i] : 0.f;
    }
    int cnt = 0;
#pragma unroll
    for (int it = 0; it < CITER; ++it) cnt += __popc(__ballot_sync(0xffffffffu, cvr[it] != 0));
    if (lane == 0) s_wcount[warp] = cnt;
    __syncthreads();
    int off = 0;
    for (int w = 0; w < warp; ++w) off += s_wcount[w];
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < SNW; ++w) tot += s_wcount[w];
      S.count = tot;
    }
#pragma unroll
    for (int it = 0; it < CITER; ++it) {
      const int i = w0 + it * 32 + lane;
      const int cv = cvr[it];
      const unsigned m = __ballot_sync(0xffffffffu, cv != 0);
      if (cv != 0) {
        const int k = off + __popc(m & ((1u << lane) - 1u));
        S.fc[k] = fvr[it];
        if (!FACT) s_fclo[k] = a.fclo[item * a.n + v0 + i];
        // upper half: the float32 bits of c (small integers have a zero low
        // half), so the pair loop reads c with one AND instead of an I2F on
        // the XU pipe that the reciprocals saturate; lower half: the voxel
        S.pk[k] = i | (int)(__float_as_uint((float)cv) & 0xFFFF0000u);
      } else if (BWD && i < w1) {
        a.dX[item * a.n + v0 + i] = 0.f;
      }
      off += __popc(m);
    }
    __syncthreads();
  }
  const int count = S.count;
  load_lane();
  int kb0 = warp * VW;
  if (BWD && FACT && Lv >= 8) {
    // deferred group reduction: 8 voxel rounds, then (Lv > 8) a butterfly
    // over the lane offsets >= 8 and one reduce-scatter over 8 lanes (7
    // shuffles for 8 voxels instead of 3 per voxel); lane l < 8 ends with the
    // full w of round l and writes that voxel's dX
    for (; kb0 < count; kb0 += 8 * nslots) {
      float wv[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int k = kb0 + r * nslots + g;
        wv[r] = voxel_w(k, k < count);
      }
#pragma unroll
      for (int o = 16; o >= 8; o >>= 1)
        if (o < Lv) {
#pragma unroll
          for (int r = 0; r < 8; ++r) wv[r] += __shfl_xor_sync(0xffffffffu, wv[r], o);
        }
#pragma unroll
      for (int o = 4, n = 4; o; o >>= 1, n >>= 1) {
        const bool up = (l & o) != 0;
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const float mine = up ? wv[n + i] : wv[i];
          const float give = up ? wv[i] : wv[n + i];
          wv[i] = mine + __shfl_xor_sync(0xffffffffu, give, o);
        }
      }
      const int k = kb0 + (l & 7) * nslots + g;
      if (l < 8 && k < count) {
        const int pk = S.pk[k];
        a.dX[item * a.n + v0 + (pk & 0xffff)] = -__uint_as_float((uint32_t)pk & 0xFFFF0000u) * (lamf * wv[0]);
      }
    }
  } else {
    // warp-uniform trip count: the group reduction shuffles across the warp
    for (int kb = kb0; kb < count; kb += nslots) {
      const int k = kb + g;
      const bool valid = k < count;
      float w = voxel_w(k, valid);
      if (BWD) {
#pragma unroll
        for (int o = 16; o; o >>= 1)
          if (o < Lv) w += __shfl_xor_sync(0xffffffffu, w, o);   // Lv is warp-uniform
        if (l == 0 && valid) {
          const int pk = S.pk[k];
          a.dX[item * a.n + v0 + (pk & 0xffff)] = -__uint_as_float((uint32_t)pk & 0xFFFF0000u) * (lamf * w);
        }
      }
    }
  }

  __syncthreads();   // the next chunk's compaction overwrites S; dX of this chunk is visible
  if (BWD) soft_chunk_G_acc(a, item, v0, nvox, gacc);
  }
  // ---- fixed-order reduction of acc over the CTA's voxel slots ------------
  const int rowlen = Lv * T;
  if (FACT && (!BWD || ECC_BWD_PACKED)) {
#pragma unroll
    for (int i = 0; i < T / 2; ++i) f2_unpack(acc2[i], acc[2 * i], acc[2 * i + 1]);
    if (BWD) {   // the packed backward accumulates -d_tau (see pair_loop_fact2)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[t] = -acc[t];
    }
  }
#pragma unroll
  for (int t = 0; t < T; ++t) red[slot * rowlen + l * T + t] = acc[t];
  __syncthreads();
  double* out = a.part + (item * a.units + unit) * nb;
  for (int j = threadIdx.x; j < nb; j += SNT) {
    double sacc = 0.0;
    for (int q = 0; q < nslots; ++q) sacc += (double)red[q * rowlen + j];
    out[j] = sacc;
  }

  if (BWD) soft_unit_G_write(a, item * a.units + unit, gacc, s_g);
}

// K5/K6 windowed: see the band-mode comment above.  Per-pair arithmetic
// (a_j, block centres, the b clamp, paired reciprocals) is the full kernel's
// with T = 16, so evaluated pairs give the same float32 values.
//
// A CTA takes G consecutive chunks of one item (the per-threshold tables are
// built once per CTA).  Per chunk each warp compacts its own 512 voxels into
// its own region of the record array, sorted by band (a counting sort with
// match.any groups and shared atomics) and with every band padded to a
// multiple of four records (zero-coefficient fillers), so the warp's four
// voxel slots of eight lanes change band together; lane o of a slot holds
// block (band + o).  Blocks of 16 floats in shared memory are read and
// written as four 16-byte quads whose order is swizzled by the block index,
// so the eight lanes of a slot (consecutive blocks) hit distinct banks.
constexpr int BPAD = 2 * BVW;                        // records per warp iteration: bands are padded to it
constexpr int BREG = CH / SNW + (BPAD - 1) * BAND_MAXBANDS + BPAD;   // per-warp record region: fillers, prefetch slack

constexpr int BSTAGE = (CH / SNW) * 5;               // per-warp staging: 512 int8 + 512 float


// exact float of 0 <= i < 2^23 without an I2F (XU pipe)
__device__ __forceinline__ float i2f23(int i) { return __int_as_float(0x4B000000 | i) - 8388608.f; }

__device__ __forceinline__ int bq(int blk, int q) {   // float offset of quad q of block blk
  return blk * BT + 4 * (q ^ ((blk >> 1) & 3));
}

template <bool BWD>
#ifndef ECC_BAND_PAIR
#define ECC_BAND_PAIR 3   // paired reciprocals in both band kernels (backward: 4.82 vs 5.05 ms on 128 x 1024^2;
                          // with two voxels per lane in flight the longer chain no longer costs)
#endif
#ifndef ECC_BAND_DEFER
#define ECC_BAND_DEFER 1   // deferred w reduction (reduce-scatter over 8 voxels): backward 4.41 vs 4.99 ms (128 x 1024^2)
#endif
#ifndef ECC_BAND_GFUSE
#define ECC_BAND_GFUSE 1   // G accumulated where dX is written (no per-chunk barrier and re-read)
#endif
#ifndef ECC_BAND_WARPG
#define ECC_BAND_WARPG 0   // G per warp slice without the CTA barrier: measured slower (5.28 vs 4.41 ms)
#endif
#ifndef ECC_BAND_RPF
#define ECC_BAND_RPF 1   // backward: prefetch the next chunk's records into the staging area
#endif
#ifndef ECC_BAND_BALLOT
#define ECC_BAND_BALLOT 1   // band sort from ballots (0: MATCH groups + shared-memory atomics)
#endif
#ifndef ECC_BAND_MINB
#define ECC_BAND_MINB 2   // 128 registers: two voxels per lane in flight, no spills
#endif
__global__ void __launch_bounds__(SNT, ECC_BAND_MINB) ecc_soft_band_kernel(SoftArgs a) {
  if (a.pd) {
    if (!a.pd->factorized) return;
    a.lam = a.pd->lam;
    a.m = a.pd->center;
    a.kscale = (float)(a.lam * LOG2E);
  }
  if (!band_ok(a)) return;   // the full kernel does this problem
  const int nb = a.nb, nblk = (nb + BT - 1) / BT, nbands = nblk - NWB + 1, rowlen = nblk * BT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int2* rec = reinterpret_cast<int2*>(smem_raw);                    // [SNW][BREG] {fc bits, voxel | band << 12 | c bits}
  float* red = reinterpret_cast<float*>(rec + SNW * BREG);          // [BSLOTS][rowlen] per-slot partials
  float* natab = red + BSLOTS * rowlen;                             // [rowlen] -a_j
  float* s_up = natab + rowlen;                                     // [rowlen] (backward)
  __shared__ float s_edge[BAND_MAXBANDS + 1], s_koff[BAND_MAXBLK], s_bc[BAND_MAXBLK], s_above[BAND_MAXBLK];
#if !ECC_BAND_BALLOT
  __shared__ int s_cnt[SNW][BAND_MAXBANDS];
#endif
  __shared__ int s_csb[BAND_MAXBANDS];
  __shared__ double s_g[SNW][4];

  const int64_t item = a.item0 + blockIdx.x / a.lunits;
  const int64_t unit = a.unit0 + blockIdx.x % a.lunits;
  const int64_t c0 = unit * a.G, c1 = min(c0 + a.G, a.chunks);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double ks = a.lam * LOG2E;

  // ---- per-threshold factors and per-block parameters (once per CTA) -------
  for (int j = threadIdx.x; j < rowlen; j += SNT) {
    float av = 0.f;
    if (j < nb) {
      const int b0 = (j / BT) * BT, b1 = min(b0 + BT, nb) - 1;
      av = (float)exp2(-ks * (a.taus[j] - 0.5 * (a.taus[b0] + a.taus[b1])));
    }
    const int q = bq(j / BT, (j % BT) >> 2) + (j & 3);
    natab[q] = -av;   // negated: see pair_loop_fact2
    s_up[q] = (BWD && j < nb) ? (float)a.up[item * nb + j] : 0.f;
  }
  for (int i = threadIdx.x; i < BSLOTS * rowlen; i += SNT) red[i] = 0.f;
  if (threadIdx.x < nblk)
    s_koff[threadIdx.x] = (float)(ks * (a.m - 0.5 * (a.taus[threadIdx.x * BT] + a.taus[min(threadIdx.x * BT + BT, nb) - 1])));
  if (threadIdx.x <= BAND_MAXBANDS) {
    // band b >= 1 starts where f - m >= tau_{16 b} - m + W; +inf past the last band
    const int b = threadIdx.x;
    s_edge[b] = (b >= 1 && b < nbands) ? (float)(a.taus[b * BT] - a.m + BAND_ZCUT / a.lam) : INFINITY;
  }
  if (threadIdx.x < BAND_MAXBANDS) s_csb[threadIdx.x] = 0;
  __syncthreads();
  float bcv = B_MAX;
  bool prod = false;
  if (ECC_BAND_PAIR & (BWD ? 2 : 1)) {
    bool okp = true;
    if (threadIdx.x < nblk) {
      float amax = 0.f, dmax = 0.f;
#pragma unroll
      for (int t = 0; t < BT; ++t) {
        const int tp = (BT - 2 - 2 * (t >> 1)) + (t & 1);
        const float x0 = -natab[bq(threadIdx.x, t >> 2) + (t & 3)], x1 = -natab[bq(threadIdx.x, tp >> 2) + (tp & 3)];
        const float l0 = x0 > 0.f ? __log2f(x0) : 0.f, l1 = x1 > 0.f ? __log2f(x1) : 0.f;
        amax = fmaxf(amax, fabsf(l0));
        dmax = fmaxf(dmax, l0 + l1);
      }
      bcv = fminf(B_MAX, 0.5f * (126.f - dmax) - 1.f);
      okp = bcv - amax >= 24.f;
    }
    prod = __syncthreads_and(okp) != 0;
  }
  if (threadIdx.x < nblk) s_bc[threadIdx.x] = prod ? bcv : B_MAX;
  // (made visible by the first chunk's barrier)

  const int g = lane / NWB, o = lane % NWB;
  const int slot = warp * BVW + g;
  float* myred = red + slot * rowlen;
  int2* wrec = rec + warp * BREG;
  f2_t nat2[BT / 2], up2[BT / 2], acc2[BT / 2];
  float koff = 0.f, bc = B_MAX, csum = 0.f;
  int curb = -1;
  auto load_block = [&](int b) {
    const int blk = b + o;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 av = *reinterpret_cast<const float4*>(natab + bq(blk, q));
      nat2[2 * q] = f2_pack(av.x, av.y);
      nat2[2 * q + 1] = f2_pack(av.z, av.w);
      if (BWD) {
        const float4 uv = *reinterpret_cast<const float4*>(s_up + bq(blk, q));
        up2[2 * q] = f2_pack(uv.x, uv.y);
        up2[2 * q + 1] = f2_pack(uv.z, uv.w);
      }
    }
#pragma unroll
    for (int i = 0; i < BT / 2; ++i) acc2[i] = 0ull;
    koff = s_koff[blk];
    bc = s_bc[blk];
  };
  auto flush = [&]() {
    const int blk = curb + o;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float4* p = reinterpret_cast<float4*>(myred + bq(blk, q));
      float4 v = *p;
      float x0, x1, x2, x3;
      f2_unpack(acc2[2 * q], x0, x1);
      f2_unpack(acc2[2 * q + 1], x2, x3);
      if (BWD) { v.x -= x0; v.y -= x1; v.z -= x2; v.w -= x3; }   // the packed backward accumulates -d_tau
      else { v.x += x0; v.y += x1; v.z += x2; v.w += x3; }
      *p = v;
    }
    if (!BWD && o == 0) atomicAdd(&s_csb[curb], (int)csum);
    csum = 0.f;
  };
  if (!BWD) {
#pragma unroll
    for (int i = 0; i < BT / 2; ++i) up2[i] = 0ull;
  }
  const float lamf = (float)a.lam;
  double gacc[3] = {0.0, 0.0, 0.0};
  constexpr int CITER = CH / SNW / 32;
  const int Wi = (int)a.W, Hi = (int)a.H;
  const float invW = 1.0f / (float)a.W;
  const float sHf = a.H > 1 ? (float)(2.0 / (double)(a.H - 1)) : 0.f;
  const float sWf = a.W > 1 ? (float)(2.0 / (double)(a.W - 1)) : 0.f;
  const float sDf = a.D > 1 ? (float)(2.0 / (double)(a.D - 1)) : 0.f;
  // The warp's next slice of coefficients and field values is fetched into
  // its shared staging buffer with cp.async while it sorts and walks the
  // current one (16-byte copies: needs 16-byte aligned slices).
  const bool staged = !(BWD && a.recs) && (a.n % 16) == 0 && (((uintptr_t)a.c | (uintptr_t)a.fc) & 15) == 0;
  int8_t* st_c = reinterpret_cast<int8_t*>(s_up + rowlen) + warp * BSTAGE;   // [512] coefficients
  float* st_f = reinterpret_cast<float*>(st_c + CITER * 32);                  // [512] field values
  auto stage_issue = [&](int64_t ch) {
    const int w0s = warp * (CITER * 32);
    const int nv = (int)min((int64_t)CITER * 32, max((int64_t)0, min((int64_t)CH, a.n - ch * CH) - w0s));
    const int64_t vb = item * a.n + ch * CH + w0s;
    const int off = 16 * lane;
    const int cb = max(0, min(16, nv - off));
    cp_async16(st_c + off, a.c + vb + (cb ? off : 0), cb);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int fo = off + 4 * q;
      const int fb = 4 * max(0, min(4, nv - fo));
      cp_async16(st_f + fo, a.fc + vb + (fb ? fo : 0), fb);
    }
    cp_async_commit();
  };
  if (staged) stage_issue(c0);
  // Backward with the forward's records: the first RPF records of the warp's
  // next chunk are fetched into the (otherwise idle) staging area with
  // cp.async while the current chunk walks, so only the rest of a chunk's
  // records is read with the walk waiting (a fixed count: no wait on the
  // next chunk's record count; the region holds BREG records, all in bounds).
  constexpr int RPF = ECC_BAND_RPF ? (BSTAGE / 16) * 2 : 0;   // records (8 B) that fit the staging area
  int4* rpf = reinterpret_cast<int4*>(st_c);
  auto rpf_issue = [&](int64_t ch) {
    const int4* src4 = reinterpret_cast<const int4*>(a.recs + ((item * a.chunks + ch) * SNW + warp) * BREG);
    for (int q = lane; q < RPF / 2; q += 32) cp_async16(rpf + q, src4 + q, 16);
    cp_async_commit();
  };
  if (BWD && a.recs && RPF && c0 < c1) rpf_issue(c0);
  const float e1 = s_edge[1];
  const float einv = nbands > 2 ? (float)(nbands - 2) / (s_edge[nbands - 1] - e1) : 0.f;

  for (int64_t chunk = c0; chunk < c1; ++chunk) {
    const int64_t v0 = chunk * CH;
    const int nvox = (int)min((int64_t)CH, a.n - v0);
    const int8_t* cg = a.c + item * a.n + v0;
    const float* fg = a.fc + item * a.n + v0;
    // ---- per-warp compaction to c != 0 voxels, sorted by band (stable) -----
    const int w0 = warp * (CITER * 32), w1 = min(w0 + CITER * 32, nvox);
    int nlist = 0;   // records in this warp's region, fillers included
    const int64_t rbase = (item * a.chunks + chunk) * SNW + warp;   // saved records of this warp and chunk
    if (BWD && a.recs) {
      // the forward's sorted records: no compaction, no sort
      nlist = a.rcnt[rbase];
      const int4* src4 = reinterpret_cast<const int4*>(a.recs + rbase * BREG);
      int pre = 0;
      if (RPF) {   // the prefetched head of the list, then the next chunk's head
        pre = min(nlist, RPF) / 2;
        cp_async_wait_all();
        __syncwarp();
        for (int q = lane; q < pre; q += 32) reinterpret_cast<int4*>(wrec)[q] = rpf[q];
        __syncwarp();
        if (chunk + 1 < c1) rpf_issue(chunk + 1);
      }
      for (int q = pre + lane; q < nlist / 2; q += 32) reinterpret_cast<int4*>(wrec)[q] = src4[q];
      for (int i = w0 + lane; i < w1; i += 32) a.dX[item * a.n + v0 + i] = 0.f;   // c = 0 voxels
      __syncwarp();
    } else {
      int kvr[CITER];     // band | c << 8  (c == 0: band field 0xFF)
      float fvr[CITER];
      if (staged) {
        cp_async_wait_all();
        __syncwarp();
  #pragma unroll
        for (int it = 0; it < CITER; ++it) {
          const int i = w0 + it * 32 + lane;
          const int cv = i < w1 ? (int)st_c[it * 32 + lane] : 0;
          fvr[it] = i < w1 ? st_f[it * 32 + lane] : 0.f;
          kvr[it] = (cv << 8) | 0xFF;
        }
        __syncwarp();
        if (chunk + 1 < c1) stage_issue(chunk + 1);   // overlaps this chunk's sort and window loop
      } else {
  #pragma unroll
        for (int it = 0; it < CITER; ++it) {
          const int i = w0 + it * 32 + lane;
          const int cv = i < w1 ? (int)cg[i] : 0;
          fvr[it] = i < w1 ? fg[i] : 0.f;
          kvr[it] = (cv << 8) | 0xFF;
        }
      }
#if !ECC_BAND_BALLOT
      if (lane < BAND_MAXBANDS) s_cnt[warp][lane] = 0;
      __syncwarp();
#endif
  #pragma unroll
      for (int it = 0; it < CITER; ++it) {
        const float f = fvr[it];
        if ((kvr[it] >> 8) != 0) {
          // band guess for near-uniform thresholds, then fixed against the edges
          int bb = 0;
          if (f >= e1) {
            const float gss = __fmul_rn(f - e1, einv);
            bb = min(1 + (gss < (float)nbands ? (int)gss : nbands), nbands - 1);
            // one step each way covers a guess off by one; exact otherwise
            const float lo = s_edge[bb], hi = s_edge[bb + 1], lo1 = s_edge[bb - 1];
            if (lo > f) {
              --bb;
              if (lo1 > f) { while (bb > 0 && s_edge[bb] > f) --bb; }
            } else if (hi <= f) {
              ++bb;
              while (s_edge[bb + 1] <= f) ++bb;
            }
          }
          kvr[it] = (kvr[it] & ~0xFF) | bb;
        }
      }
#if ECC_BAND_BALLOT
      // Stable counting sort by band from five ballots per iteration (valid,
      // band bits 0..3): lane b holds band b's voxel mask, so the counts, the
      // slots and each voxel's peers come from popc / shfl -- no MATCH, no
      // shared-memory atomics.
      const uint32_t FULLM = 0xffffffffu;
      const uint32_t lm0 = (lane & 1) ? ~0u : 0u, lm1 = (lane & 2) ? ~0u : 0u;
      const uint32_t lm2 = (lane & 4) ? ~0u : 0u, lm3 = (lane & 8) ? ~0u : 0u;
      auto band_mask = [&](int kv) -> uint32_t {   // voxels of band `lane` in one iteration
        const uint32_t V = __ballot_sync(FULLM, (kv >> 8) != 0);
        const uint32_t B0 = __ballot_sync(FULLM, kv & 1), B1 = __ballot_sync(FULLM, kv & 2);
        const uint32_t B2 = __ballot_sync(FULLM, kv & 4), B3 = __ballot_sync(FULLM, kv & 8);
        return V & ~(B0 ^ lm0) & ~(B1 ^ lm1) & ~(B2 ^ lm2) & ~(B3 ^ lm3);
      };
      int pos;
      __syncwarp();   // the previous chunk's walk is done with wrec
      {
        int run = 0;
  #pragma unroll
        for (int it = 0; it < CITER; ++it) run += __popc(band_mask(kvr[it]));
        const int c = lane < nbands ? run : 0;
        const int cpad = (c + BPAD - 1) & ~(BPAD - 1);
        int incl = cpad;
  #pragma unroll
        for (int sh = 1; sh < 32; sh <<= 1) {
          const int y = __shfl_up_sync(FULLM, incl, sh);
          if (lane >= sh) incl += y;
        }
        // fillers at the end of each band: zero coefficient, the band's index
        for (int q = incl - cpad + c; q < incl; ++q) wrec[q] = make_int2(0, lane << 12);
        pos = incl - cpad;   // next slot of band `lane`
        nlist = __shfl_sync(FULLM, incl, 31);
      }
      const uint32_t ltmask = (1u << lane) - 1u;
  #pragma unroll
      for (int it = 0; it < CITER; ++it) {
        const uint32_t M = band_mask(kvr[it]);
        const int i = w0 + it * 32 + lane;
        const int kv = kvr[it], cv = kv >> 8, bb = kv & 0xFF;
        const uint32_t peers = __shfl_sync(FULLM, M, bb & 31);
        const int base = __shfl_sync(FULLM, pos, bb & 31);
        if (cv != 0) {
          const int k = base + __popc(peers & ltmask);
          wrec[k] = make_int2(__float_as_int(fvr[it]), i | (bb << 12) | (int)(__float_as_uint((float)cv) & 0xFFFF0000u));
        } else if (BWD && i < w1) {
          a.dX[item * a.n + v0 + i] = 0.f;
        }
        pos += __popc(M);
      }
#else
      // band groups of all iterations first (independent MATCHes in flight),
      // then the counts.  The backward, whose window loop needs more registers,
      // recomputes the groups in the scatter instead of keeping them (spills).
      constexpr bool KEEP = !BWD;
      unsigned pvr[CITER];
  #pragma unroll
      for (int it = 0; it < CITER; ++it) pvr[it] = __match_any_sync(0xffffffffu, kvr[it] & 0xFF);
  #pragma unroll
      for (int it = 0; it < CITER; ++it)
        if ((kvr[it] >> 8) != 0 && lane == __ffs(pvr[it]) - 1) atomicAdd(&s_cnt[warp][kvr[it] & 0xFF], __popc(pvr[it]));
      __syncwarp();
      {
        const int c = lane < nbands ? s_cnt[warp][lane] : 0;
        const int cpad = (c + BPAD - 1) & ~(BPAD - 1);
        int incl = cpad;
  #pragma unroll
        for (int sh = 1; sh < 32; sh <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, sh);
          if (lane >= sh) incl += y;
        }
        // fillers at the end of each band: zero coefficient, the band's index
        for (int q = incl - cpad + c; q < incl; ++q) wrec[q] = make_int2(0, lane << 12);
        __syncwarp();
        if (lane < nbands) s_cnt[warp][lane] = incl - cpad;   // start of band `lane`
        nlist = __shfl_sync(0xffffffffu, incl, 31);
      }
      __syncwarp();
      // slots: each band group's leader reserves its records (the atomics of all
      // iterations in flight), then every member stores at its rank
      int oldv[CITER];
      if (KEEP) {
  #pragma unroll
        for (int it = 0; it < CITER; ++it) {
          const int bb = kvr[it] & 0xFF;
          oldv[it] = ((kvr[it] >> 8) != 0 && lane == __ffs(pvr[it]) - 1) ? atomicAdd(&s_cnt[warp][bb], __popc(pvr[it])) : 0;
        }
      }
  #pragma unroll
      for (int it = 0; it < CITER; ++it) {
        const int i = w0 + it * 32 + lane;
        const int kv = kvr[it], cv = kv >> 8, bb = kv & 0xFF;
        const unsigned peers = KEEP ? pvr[it] : __match_any_sync(0xffffffffu, bb);
        if (!KEEP) oldv[it] = (cv != 0 && lane == __ffs(peers) - 1) ? atomicAdd(&s_cnt[warp][bb], __popc(peers)) : 0;
        const int base = __shfl_sync(0xffffffffu, oldv[it], __ffs(peers) - 1);
        if (cv != 0) {
          const int k = base + __popc(peers & ((1u << lane) - 1u));
          wrec[k] = make_int2(__float_as_int(fvr[it]), i | (bb << 12) | (int)(__float_as_uint((float)cv) & 0xFFFF0000u));
        } else if (BWD && i < w1) {
          a.dX[item * a.n + v0 + i] = 0.f;
        }
      }
#endif
      __syncwarp();
      if (!BWD && a.recs) {   // kept for the backward
        int4* dst4 = reinterpret_cast<int4*>(a.recs + rbase * BREG);
        for (int q = lane; q < nlist / 2; q += 32) dst4[q] = reinterpret_cast<const int4*>(wrec)[q];
        if (lane == 0) a.rcnt[rbase] = nlist;
      }
    }
    if (chunk == c0) __syncthreads();   // the per-block tables of the prologue

    // fused G (backward): this chunk's first voxel in (z, y, x) and per-lane sums
    float gf0 = 0.f, gf1 = 0.f, gf2 = 0.f;
    int cx0 = 0, cy0 = 0, cz0 = 0;
    if (BWD && ECC_BAND_GFUSE) {
      const int64_t zq = v0 / (a.H * a.W), rq = v0 - zq * a.H * a.W, yq = rq / a.W;
      cz0 = (int)zq;
      cy0 = (int)yq;
      cx0 = (int)(rq - yq * a.W);
    }
    // ---- window loop: the warp's four slots walk its list together ---------
    // Slot g takes records kb + 2g and kb + 2g + 1 (one 16-byte load, the
    // next pair prefetched; the region has slack for the overrun): two
    // independent voxels per lane and iteration.
    auto walk = [&](auto prodtag) {
      constexpr bool PROD = decltype(prodtag)::value;
      int4 r = *reinterpret_cast<const int4*>(wrec + 2 * g);
      // one warp iteration: records kb + 2g, kb + 2g + 1 of each slot; w0 / w1
      // are this lane's partial w of the two voxels (backward)
      auto iter = [&](int kb, float& w0, float& w1) {
        const int4 cur = r;
        r = *reinterpret_cast<const int4*>(wrec + kb + BPAD + 2 * g);
        const int b = (cur.y >> 12) & 0xF;   // uniform over the warp (bands padded to BPAD)
        if (b != curb) {
          if (curb >= 0) flush();
          load_block(b);
          curb = b;
        }
        const float cf0 = __uint_as_float((uint32_t)cur.y & 0xFFFF0000u);
        const float cf1 = __uint_as_float((uint32_t)cur.w & 0xFFFF0000u);
        if (!BWD) csum += cf0 + cf1;
        const float kf0 = fminf(fmaxf(__fmaf_rn(a.kscale, __int_as_float(cur.x), koff), -bc), bc);
        const float kf1 = fminf(fmaxf(__fmaf_rn(a.kscale, __int_as_float(cur.z), koff), -bc), bc);
        if (PROD) {
          const float b0 = (!BWD && ECC_BAND_EX2_FMA) ? ex2_fma(kf0) : ex2_approx(kf0);
          const float b1 = (!BWD && ECC_BAND_EX2_FMA) ? ex2_fma(kf1) : ex2_approx(kf1);
          pair_loop_prod<BWD, BT, BWD ? ECC_PROD_UNP : 0>(nat2, up2, acc2, b0, cf0, w0);
          pair_loop_prod<BWD, BT, BWD ? ECC_PROD_UNP : 0>(nat2, up2, acc2, b1, cf1, w1);
        } else {
          pair_loop_fact2<BWD, BT>(nat2, up2, acc2, ex2_approx(kf0), cf0, w0);
          pair_loop_fact2<BWD, BT>(nat2, up2, acc2, ex2_approx(kf1), cf1, w1);
        }
      };
      if (!BWD) {
        for (int kb = 0; kb < nlist; kb += BPAD) {
          float w0 = 0.f, w1 = 0.f;
          iter(kb, w0, w1);
        }
      } else if (!ECC_BAND_DEFER) {
        float* dxp = a.dX + item * a.n + v0;
        for (int kb = 0; kb < nlist; kb += BPAD) {
          float w0 = 0.f, w1 = 0.f;
          iter(kb, w0, w1);
#pragma unroll
          for (int sh = NWB / 2; sh; sh >>= 1) {
            w0 += __shfl_xor_sync(0xffffffffu, w0, sh);
            w1 += __shfl_xor_sync(0xffffffffu, w1, sh);
          }
          const int ry0 = wrec[kb + 2 * g].y, ry1 = wrec[kb + 2 * g + 1].y;
          const float cf0 = __uint_as_float((uint32_t)ry0 & 0xFFFF0000u), cf1 = __uint_as_float((uint32_t)ry1 & 0xFFFF0000u);
          if (o == 0 && cf0 != 0.f) dxp[ry0 & 0xfff] = -cf0 * (lamf * w0);
          if (o == 1 && cf1 != 0.f) dxp[ry1 & 0xfff] = -cf1 * (lamf * w1);
        }
      } else {
        // w of 8 voxels (4 iterations) reduced at once: a reduce-scatter over
        // the slot's 8 lanes (7 shuffles instead of 24) leaves lane o with the
        // sum of voxel o of the group, which it writes
        float* dxp = a.dX + item * a.n + v0;
        for (int kb0 = 0; kb0 < nlist; kb0 += 4 * BPAD) {
          float wv[8];
#pragma unroll
          for (int gi = 0; gi < 4; ++gi) {
            wv[2 * gi] = wv[2 * gi + 1] = 0.f;
            if (kb0 + gi * BPAD < nlist) iter(kb0 + gi * BPAD, wv[2 * gi], wv[2 * gi + 1]);
          }
#pragma unroll
          for (int sh = 4, nn = 4; sh; sh >>= 1, nn >>= 1) {
            const bool upper = (o & sh) != 0;
#pragma unroll
            for (int i = 0; i < nn; ++i) {
              const float mine = upper ? wv[nn + i] : wv[i];
              const float give = upper ? wv[i] : wv[nn + i];
              wv[i] = mine + __shfl_xor_sync(0xffffffffu, give, sh);
            }
          }
          if (kb0 + (o >> 1) * BPAD < nlist) {
            const int ry = wrec[kb0 + (o >> 1) * BPAD + 2 * g + (o & 1)].y;
            const float cf = __uint_as_float((uint32_t)ry & 0xFFFF0000u);
            if (cf != 0.f) {
              const float d = -cf * (lamf * wv[0]);
              const int idx = ry & 0xfff;
              dxp[idx] = d;
              if (ECC_BAND_GFUSE) {
                // G -= d pos(voxel): coordinates from the chunk's first voxel
                // (quotient by W through a float estimate, corrected exactly)
                // (ints below 2^23 converted by the 2^23 magic add: no XU
                // instructions next to the reciprocals)
                const int t = cx0 + idx;
                int q = __float_as_int(__fmaf_rn(i2f23(t), invW, 8388608.f)) - 0x4B000000;
                int xx = t - q * Wi;
                if (xx < 0) { --q; xx += Wi; }
                if (xx >= Wi) { ++q; xx -= Wi; }
                int yy = cy0 + q, zz = cz0;
                while (yy >= Hi) { yy -= Hi; ++zz; }
                const float px = a.W > 1 ? __fmaf_rn(i2f23(xx), sWf, -1.f) : 0.f;
                const float py = a.H > 1 ? __fmaf_rn(i2f23(yy), sHf, -1.f) : 0.f;
                if (a.ndim == 2) {
                  gf0 = __fmaf_rn(-d, py, gf0);
                  gf1 = __fmaf_rn(-d, px, gf1);
                } else {
                  const float pz = a.D > 1 ? __fmaf_rn(i2f23(zz), sDf, -1.f) : 0.f;
                  gf0 = __fmaf_rn(-d, pz, gf0);
                  gf1 = __fmaf_rn(-d, py, gf1);
                  gf2 = __fmaf_rn(-d, px, gf2);
                }
              }
            }
          }
        }
      }
    };
    if (prod) walk(std::true_type{});
    else walk(std::false_type{});
    // flushed per chunk: the block registers are then dead during the next
    // chunk's compaction
    if (curb >= 0) flush();
    curb = -1;
    if (BWD && ECC_BAND_GFUSE) {
      gacc[0] += gf0;
      gacc[1] += gf1;
      gacc[2] += gf2;
    } else if (BWD && ECC_BAND_WARPG) {
      // G over this warp's slice: its dX were all written by this warp
      __syncwarp();
      const int i0 = w0 + 16 * lane;
      soft_run_G_acc(a, item, v0, i0, min(i0 + 16, w1), gacc);
    } else if (BWD) {
      __syncthreads();   // dX of this chunk is visible to the CTA
      soft_chunk_G_acc(a, item, v0, nvox, gacc);
    }
  }
  __syncthreads();

  // ---- fixed-order reduction over the CTA's slots ----------------------------
  if (!BWD && threadIdx.x < nblk) {
    // block J lies above the window of every band b <= J - NWB: sigma = 1
    int cs = 0;
    for (int b = 0; b <= (int)threadIdx.x - NWB; ++b) cs += s_csb[b];
    s_above[threadIdx.x] = (float)cs;
  }
  __syncthreads();
  double* out = a.part + (item * a.units + unit) * nb;
  for (int j = threadIdx.x; j < nb; j += SNT) {
    const int q = bq(j / BT, (j % BT) >> 2) + (j & 3);
    double sacc = BWD ? 0.0 : (double)s_above[j / BT];
    for (int sl = 0; sl < BSLOTS; ++sl) sacc += (double)red[sl * rowlen + q];
    out[j] = sacc;
  }
  if (BWD) soft_unit_G_write(a, item * a.units + unit, gacc, s_g);
}

static size_t band_smem(int nb) {
  const size_t rowlen = (size_t)((nb + BT - 1) / BT) * BT;
  return sizeof(int2) * SNW * BREG + sizeof(float) * ((size_t)BSLOTS + 2) * rowlen + (size_t)SNW * BSTAGE;
}

// K7: out[b][j] = scale_j * sum_c part[b][c][j] in a fixed order: stage 1
// sums contiguous groups of chunks (grid over bins x groups x items), stage 2
// sums the group partials; both orders are fixed, so runs are bit-identical.
constexpr int RGROUPS = 128;
__global__ void ecc_soft_reduce1(const double* __restrict__ part, int64_t chunks, int nb, int64_t per_group,
                                 double* __restrict__ gpart) {
  const int64_t item = blockIdx.z, grp = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nb) return;
  const int64_t c0 = grp * per_group, c1 = min(c0 + per_group, chunks);
  const double* p = part + item * chunks * nb + j;
  double s = 0.0;
  for (int64_t c = c0; c < c1; ++c) s += p[c * nb];
  gpart[(item * gridDim.y + grp) * nb + j] = s;
}

__global__ void ecc_soft_reduce2(const double* __restrict__ gpart, int groups, int nb, const double* __restrict__ up,
                                 double lam, const ecc_soft_params* __restrict__ pd, double* __restrict__ out) {
  if (pd) lam = pd->lam;
  const int64_t item = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nb) return;
  const double* p = gpart + item * groups * nb + j;
  double s = 0.0;
  for (int g = 0; g < groups; ++g) s += p[(int64_t)g * nb];
  if (up) s *= up[item * nb + j] * lam;
  out[item * nb + j] = s;
}

// G[item][0..ndim) = sum over chunks of gpart[item][chunk][0..ndim), fixed order:
// strided per-thread sums, then a fixed shared-memory tree
__global__ void ecc_soft_reduce_g(const double* __restrict__ gpart, int64_t chunks, int ndim, double* __restrict__ G) {
  __shared__ double sm[256][3];
  const int64_t item = blockIdx.x;
  double a[3] = {0.0, 0.0, 0.0};
  for (int64_t c = threadIdx.x; c < chunks; c += blockDim.x)
    for (int d = 0; d < 3; ++d) a[d] += gpart[(item * chunks + c) * 4 + d];
  for (int d = 0; d < 3; ++d) sm[threadIdx.x][d] = a[d];
  __syncthreads();
  for (int o = blockDim.x >> 1; o; o >>= 1) {
    if (threadIdx.x < o)
      for (int d = 0; d < 3; ++d) sm[threadIdx.x][d] += sm[threadIdx.x + o][d];
    __syncthreads();
  }
  if (threadIdx.x < ndim) G[item * ndim + threadIdx.x] = sm[0][threadIdx.x];
}

static size_t soft_smem(bool fact, int T) {
  const size_t chunk = CHUNK_BYTES + (fact ? sizeof(float) * MAXB_PASS
                                           : sizeof(float) * CH + sizeof(double) * MAXB_PASS);
  const size_t red = sizeof(float) * (size_t)SNT * T;   // nslots * rowlen = 8 * VW * Lv * T = 256 T
  return chunk > red ? chunk : red;
}

}  // namespace ecc

using namespace ecc;

static int soft_dims(int ndim, const int64_t* dims, int64_t d3[3]) {
  if (ndim == 2) { d3[0] = 1; d3[1] = dims[0]; d3[2] = dims[1]; }
  else if (ndim == 3) { d3[0] = dims[0]; d3[1] = dims[1]; d3[2] = dims[2]; }
  else return set_error(ECC_EINVAL, "grid must be 2D or 3D");
  for (int i = 0; i < 3; ++i) if (d3[i] < 1) return set_error(ECC_EINVAL, "grid extents must be positive");
  return ECC_OK;
}

extern "C" size_t ecc_soft_workspace_bytes(int ndim, const int64_t* dims, int64_t batch, int64_t nbins) {
  int64_t d3[3];
  if (soft_dims(ndim, dims, d3)) return 0;
  const int64_t n = d3[0] * d3[1] * d3[2];
  const int64_t chunks = (n + CH - 1) / CH;
  // per-CTA partials [batch][chunks][B], G partials [batch][chunks][4],
  // group partials [batch][RGROUPS][B]
  return sizeof(double) * ((size_t)(batch * chunks) * (size_t)(nbins + 4) + (size_t)batch * RGROUPS * (size_t)nbins);
}

// cudaFuncSetAttribute once per (kernel, smem size, device): the launchers
// stay free of per-call driver work besides the launches themselves
static bool soft_attr_done(const void* kfn, size_t smem) {
  // true when the kernel's attribute already covers smem; else the caller raises it
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> attr;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = attr[{kfn, dev}];
  if (smem <= cur) return true;
  cur = smem;
  return false;
}

// G chunks per CTA: the per-CTA tables and partial rows are amortised over G
// chunks while keeping ~6 waves of 3 CTAs per SM
static int64_t soft_units_G(int64_t batch, int64_t chunks) {
  int64_t G = variant_soft_g();
  if (G <= 0) G = std::max<int64_t>(1, std::min<int64_t>(16, batch * chunks / (148 * 3 * 6)));
  return std::max<int64_t>(1, std::min<int64_t>(G, chunks));
}

template <bool BWD>
static int soft_launch(const int8_t* coeffs, const float* fc, const float* fclo, int ndim, const int64_t* dims, int64_t batch,
                       const double* taus, int64_t nbins, const ecc_soft_params* p, const double* up, float* dX,
                       double* out_main, double* G_out, void* workspace, void* stream,
                       const ecc_soft_params* pd = nullptr, void* records = nullptr, int64_t unit_begin = 0,
                       int64_t unit_end = -1, bool finish = true, int64_t item_begin = 0, int64_t item_end = -1,
                       int64_t G_force = 0) {
  clear_error();
  int64_t d3[3];
  int rc = soft_dims(ndim, dims, d3);
  if (rc) return rc;
  if (!coeffs || !fc || !taus || !p || !out_main || !workspace) return set_error(ECC_EINVAL, "null pointer argument");
  if (BWD && (!up || !dX || !G_out)) return set_error(ECC_EINVAL, "null pointer argument");
  if (batch < 1 || nbins < 1) return set_error(ECC_EINVAL, "empty soft problem");
  if (nbins > MAXB_PASS) return set_error(ECC_EINVAL, "soft path supports at most 1024 thresholds per call");
  if (!pd && !(p->lam > 0)) return set_error(ECC_EINVAL, "sharpness must be positive");
  if ((pd || !p->factorized) && !fclo)
    return set_error(ECC_EINVAL, "direct mode needs the float32 field remainder");
  const int64_t n = d3[0] * d3[1] * d3[2];
  const int64_t chunks = (n + CH - 1) / CH;
  SoftArgs a;
  a.c = coeffs;
  a.fc = fc;
  a.fclo = fclo;
  a.n = n;
  a.chunks = chunks;
  a.D = d3[0];
  a.H = d3[1];
  a.W = d3[2];
  a.ndim = ndim;
  a.nb = (int)nbins;
  a.factorized = p->factorized;
  a.kscale = (float)(p->lam * LOG2E);
  a.lam = p->lam;
  a.m = p->center;
  a.taus = taus;
  a.up = up;
  a.part = (double*)workspace;
  a.gpart = a.part + (size_t)(batch * chunks) * (size_t)nbins;
  a.dX = dX;
  a.pd = pd;
  a.band = 0;
  if (((uintptr_t)records & 15) != 0) return set_error(ECC_EINVAL, "the records buffer must be 16-byte aligned");
  a.recs = reinterpret_cast<int2*>(records);
  a.rcnt = records ? reinterpret_cast<int*>(a.recs + (size_t)(batch * chunks) * SNW * BREG) : nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  // 16 thresholds per lane (~80 registers, 3 CTAs/SM): on 16 x 1024^2,
  // B = 256 the forward takes 522 vs 559 us and the backward 837 vs 868 us
  // compared with 32 per lane; ECC_SOFT_FWD_T / ECC_SOFT_BWD_T = 32 override
  const int tsel = variant_soft_t(BWD);
  const int T = (tsel == 8 && nbins <= 8 * 32) ? 8 : (tsel <= 16 && nbins <= 16 * 32) ? 16 : 32;
  // G chunks per CTA: the per-CTA tables and partial rows are amortised
  // over G chunks while keeping ~6 waves of 3 CTAs per SM
  const int64_t G = G_force > 0 ? std::min<int64_t>(G_force, chunks) : soft_units_G(batch, chunks);
  const int64_t units = (chunks + G - 1) / G;
  a.G = G;
  a.units = units;
  if (unit_end < 0) unit_end = units;
  if (unit_begin < 0 || unit_end > units || unit_begin > unit_end) return set_error(ECC_EINVAL, "unit range out of bounds");
  a.unit0 = unit_begin;
  a.lunits = unit_end - unit_begin;
  if (item_end < 0) item_end = batch;
  if (item_begin < 0 || item_end > batch || item_begin > item_end) return set_error(ECC_EINVAL, "item range out of bounds");
  a.item0 = item_begin;
  const int64_t grid = (item_end - item_begin) * a.lunits;
  if (grid > 0x7fffffff) return set_error(ECC_EINVAL, "soft problem too large");
  if (grid > 0) {
  // host parameters: the one mode they select; device parameters: both modes,
  // the kernel whose mode the device flag does not select exits at once
  // band kernel alongside the full factorised one (each CTA of both decides
  // band_ok identically; exactly one of them works)
  const int nblk = (int)((nbins + BT - 1) / BT);
  a.band = (T == BT && variant_soft_band() && nbins <= BAND_MAXB && nblk - NWB + 1 >= 2 && nblk - NWB + 1 <= BAND_MAXBANDS &&
            (pd || p->factorized)) ? 1 : 0;
  if (a.band) {
    auto kfn = ecc_soft_band_kernel<BWD>;
    const size_t smem = band_smem((int)nbins);
    if (!soft_attr_done(reinterpret_cast<const void*>(kfn), smem)) {
      cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(soft band)");
    }
    kfn<<<(unsigned)grid, SNT, smem, s>>>(a);
    rc = check_launch(BWD ? "ecc_soft_band_kernel<bwd>" : "ecc_soft_band_kernel<fwd>");
    if (rc) return rc;
  }
  for (int mode = 0; mode < 2; ++mode) {
    const bool fact = mode == 0;
    if (!pd && fact != (p->factorized != 0)) continue;
    auto kfn = fact ? (T == 8 ? ecc_soft_kernel<BWD, true, 8> : T == 16 ? ecc_soft_kernel<BWD, true, 16>
                                                                          : ecc_soft_kernel<BWD, true, 32>)
                    : (T == 8 ? ecc_soft_kernel<BWD, false, 8> : T == 16 ? ecc_soft_kernel<BWD, false, 16>
                                                                           : ecc_soft_kernel<BWD, false, 32>);
    const size_t smem = soft_smem(fact, T);
    if (!soft_attr_done(reinterpret_cast<const void*>(kfn), smem)) {
      cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(soft)");
    }
    kfn<<<(unsigned)grid, SNT, smem, s>>>(a);
    rc = check_launch(BWD ? "ecc_soft_kernel<bwd>" : "ecc_soft_kernel<fwd>");
    if (rc) return rc;
  }
  }
  if (!finish) return ECC_OK;
  const int groups = (int)(units < RGROUPS ? units : RGROUPS);
  const int64_t per_group = (units + groups - 1) / groups;
  double* grp = a.gpart + (size_t)(batch * chunks) * 4;
  dim3 g1((unsigned)((nbins + 127) / 128), (unsigned)groups, (unsigned)batch);
  ecc_soft_reduce1<<<g1, 128, 0, s>>>(a.part, units, (int)nbins, per_group, grp);
  rc = check_launch("ecc_soft_reduce1");
  if (rc) return rc;
  dim3 g2((unsigned)((nbins + 127) / 128), (unsigned)batch);
  ecc_soft_reduce2<<<g2, 128, 0, s>>>(grp, groups, (int)nbins, BWD ? up : nullptr, pd ? 0.0 : p->lam, pd, out_main);
  rc = check_launch("ecc_soft_reduce2");
  if (rc) return rc;
  if (BWD) {
    ecc_soft_reduce_g<<<(unsigned)batch, 256, 0, s>>>(a.gpart, units, ndim, G_out);
    rc = check_launch("ecc_soft_reduce_g");
  }
  return rc;
}

// band-sorted records kept from the forward for the backward (module path)
extern "C" size_t ecc_soft_records_bytes(int ndim, const int64_t* dims, int64_t batch) {
  int64_t d3[3];
  if (soft_dims(ndim, dims, d3)) return 0;
  const int64_t chunks = (d3[0] * d3[1] * d3[2] + CH - 1) / CH;
  return (size_t)(batch * chunks) * SNW * (sizeof(int2) * BREG + sizeof(int));
}

extern "C" int ecc_soft_forward(const int8_t* coeffs, const float* field_c, const float* field_lo, int ndim,
                                const int64_t* dims,
                                int64_t batch, const double* taus, int64_t nbins, const ecc_soft_params* p,
                                double* chi, void* workspace, void* stream) {
  return soft_launch<false>(coeffs, field_c, field_lo, ndim, dims, batch, taus, nbins, p, nullptr, nullptr, chi, nullptr,
                            workspace, stream);
}

extern "C" int ecc_soft_backward(const int8_t* coeffs, const float* field_c, const float* field_lo, int ndim,
                                 const int64_t* dims,
                                 int64_t batch, const double* taus, int64_t nbins, const ecc_soft_params* p,
                                 const double* upstream, float* d_values, double* d_tau, double* G, void* workspace,
                                 void* stream) {
  return soft_launch<true>(coeffs, field_c, field_lo, ndim, dims, batch, taus, nbins, p, upstream, d_values, d_tau, G,
                           workspace, stream);
}

// ---------------------------------------------------------------------------
// Device-resident soft parameters (the sync-free module path): one CTA
// derives what the host used to compute from tau / u / alpha
// (soft.py _params): the centre (tau_min + tau_max) / 2, the largest
// half-width of the 32-threshold blocks, the factorised-mode flag
// lam log2(e) halfwidth <= A_MAX, and copies lam, alpha, u.
// ---------------------------------------------------------------------------
namespace ecc {
__global__ void ecc_soft_setup_kernel(const double* __restrict__ taus, int nb, const double* __restrict__ u, int ndim,
                                      const double* __restrict__ alpha, double lam, ecc_soft_params* __restrict__ out) {
  __shared__ double smn[256], smx[256], shw[256];
  double mn = INFINITY, mx = -INFINITY, hw = 0.0;
  for (int b = threadIdx.x; b * TT < nb; b += blockDim.x) {   // block b: thresholds [32 b, 32 b + 32)
    double bmn = INFINITY, bmx = -INFINITY;
    for (int j = b * TT; j < min(nb, (b + 1) * TT); ++j) {
      bmn = fmin(bmn, taus[j]);
      bmx = fmax(bmx, taus[j]);
    }
    mn = fmin(mn, bmn);
    mx = fmax(mx, bmx);
    hw = fmax(hw, 0.5 * (bmx - bmn));
  }
  smn[threadIdx.x] = mn;
  smx[threadIdx.x] = mx;
  shw[threadIdx.x] = hw;
  __syncthreads();
  for (int o = blockDim.x >> 1; o; o >>= 1) {
    if (threadIdx.x < o) {
      smn[threadIdx.x] = fmin(smn[threadIdx.x], smn[threadIdx.x + o]);
      smx[threadIdx.x] = fmax(smx[threadIdx.x], smx[threadIdx.x + o]);
      shw[threadIdx.x] = fmax(shw[threadIdx.x], shw[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ecc_soft_params p;
    p.lam = lam;
    p.alpha = *alpha;
    for (int i = 0; i < 3; ++i) p.u[i] = i < ndim ? u[i] : 0.0;
    p.center = 0.5 * (smn[0] + smx[0]);
    p.factorized = lam * LOG2E * shw[0] <= (double)A_MAX ? 1 : 0;
    p.pad = 0;
    *out = p;
  }
}
}  // namespace ecc

extern "C" int ecc_soft_setup(const double* taus, int64_t nbins, const double* u, int ndim, const double* alpha,
                              double lam, ecc_soft_params* params_dev, void* stream) {
  clear_error();
  if (!taus || !u || !alpha || !params_dev) return set_error(ECC_EINVAL, "null pointer argument");
  if (nbins < 1 || nbins > MAXB_PASS) return set_error(ECC_EINVAL, "soft path takes 1 to 1024 thresholds");
  if (ndim != 2 && ndim != 3) return set_error(ECC_EINVAL, "grid must be 2D or 3D");
  if (!(lam > 0)) return set_error(ECC_EINVAL, "sharpness must be positive");
  ecc_soft_setup_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(taus, (int)nbins, u, ndim, alpha, lam, params_dev);
  return check_launch("ecc_soft_setup_kernel");
}

extern "C" int ecc_soft_forward_d(const int8_t* coeffs, const float* field_c, const float* field_lo, int ndim,
                                  const int64_t* dims, int64_t batch, const double* taus, int64_t nbins,
                                  const ecc_soft_params* params_dev, double* chi, void* workspace, void* records,
                                  void* stream) {
  if (!params_dev) return set_error(ECC_EINVAL, "null pointer argument");
  const ecc_soft_params placeholder{1.0, 0.0, {0.0, 0.0, 0.0}, 0.0, 1, 0};
  return soft_launch<false>(coeffs, field_c, field_lo, ndim, dims, batch, taus, nbins, &placeholder, nullptr, nullptr,
                            chi, nullptr, workspace, stream, params_dev, records);
}

extern "C" int ecc_soft_units(int ndim, const int64_t* dims, int64_t batch, int64_t* chunks_per_unit,
                              int64_t* units) {
  clear_error();
  int64_t d3[3];
  if (int rc = soft_dims(ndim, dims, d3)) return rc;
  if (!chunks_per_unit || !units) return set_error(ECC_EINVAL, "null pointer argument");
  const int64_t chunks = (d3[0] * d3[1] * d3[2] + CH - 1) / CH;
  const int64_t G = soft_units_G(batch, chunks);
  *chunks_per_unit = G;
  *units = (chunks + G - 1) / G;
  return ECC_OK;
}

extern "C" int ecc_soft_forward_range_d(const int8_t* coeffs, const float* field_c, const float* field_lo, int ndim,
                                        const int64_t* dims, int64_t batch, const double* taus, int64_t nbins,
                                        const ecc_soft_params* params_dev, double* chi, void* workspace, void* records,
                                        int64_t chunks_per_unit, int64_t item_begin, int64_t item_end,
                                        int64_t unit_begin, int64_t unit_end, int finish, void* stream) {
  if (!params_dev) return set_error(ECC_EINVAL, "null pointer argument");
  const ecc_soft_params placeholder{1.0, 0.0, {0.0, 0.0, 0.0}, 0.0, 1, 0};
  return soft_launch<false>(coeffs, field_c, field_lo, ndim, dims, batch, taus, nbins, &placeholder, nullptr, nullptr,
                            chi, nullptr, workspace, stream, params_dev, records, unit_begin, unit_end, finish != 0,
                            item_begin, item_end, chunks_per_unit);
}

extern "C" int ecc_soft_backward_d(const int8_t* coeffs, const float* field_c, const float* field_lo, int ndim,
                                   const int64_t* dims, int64_t batch, const double* taus, int64_t nbins,
                                   const ecc_soft_params* params_dev, const double* upstream, float* d_values,
                                   double* d_tau, double* G, void* workspace, const void* records, void* stream) {
  if (!params_dev) return set_error(ECC_EINVAL, "null pointer argument");
  const ecc_soft_params placeholder{1.0, 0.0, {0.0, 0.0, 0.0}, 0.0, 1, 0};
  return soft_launch<true>(coeffs, field_c, field_lo, ndim, dims, batch, taus, nbins, &placeholder, upstream, d_values,
                           d_tau, G, workspace, stream, params_dev, const_cast<void*>(records));
}

extern "C" int ecc_soft_backward_range_d(const int8_t* coeffs, const float* field_c, const float* field_lo, int ndim,
                                         const int64_t* dims, int64_t batch, const double* taus, int64_t nbins,
                                         const ecc_soft_params* params_dev, const double* upstream, float* d_values,
                                         double* d_tau, double* G, void* workspace, const void* records,
                                         int64_t chunks_per_unit, int64_t item_begin, int64_t item_end,
                                         int64_t unit_begin, int64_t unit_end, int finish, void* stream) {
  if (!params_dev) return set_error(ECC_EINVAL, "null pointer argument");
  const ecc_soft_params placeholder{1.0, 0.0, {0.0, 0.0, 0.0}, 0.0, 1, 0};
  return soft_launch<true>(coeffs, field_c, field_lo, ndim, dims, batch, taus, nbins, &placeholder, upstream, d_values,
                           d_tau, G, workspace, stream, params_dev, const_cast<void*>(records), unit_begin, unit_end,
                           finish != 0, item_begin, item_end, chunks_per_unit);
}
